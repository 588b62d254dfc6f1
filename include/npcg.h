/*
 * npcg.h -- C ABI of libnpcg.so, the B200 (sm_100a) NeuralPCG solve path.
 *
 * The reference (`pcgkit`, pure Python + numba) has no FFI: its boundary is
 * the duck-typed Python API listed next to each entry point below. This
 * header is the drop-in replacement a binding (ctypes / cffi / pybind) would
 * bind instead of those Python functions; INTEGRATION.md shows the binding.
 *
 * Conventions
 *  - Plain pointers and sizes only; no torch types. "host" pointers are
 *    ordinary CPU memory, "device" pointers are CUDA global memory on the
 *    current device. Streams are cudaStream_t passed as void*.
 *  - Batches: B systems (or B right-hand sides) that share one sparsity
 *    pattern. Vectors are laid out RHS-minor: v[i*B + b] (n x B, row major).
 *    Matrix / factor values are either shared ([nnz]) or per system
 *    ([nnz*B], value of system b for slot p at p*B + b); the `*_batched`
 *    flags select which.
 *  - Return codes map 1:1 onto pcgkit.errors (pkg/src/pcgkit/errors.py):
 *    see NPCG_ERR_*. npcg_last_error() gives the message (thread local).
 *  - No CPU fallback: every compute entry point launches CUDA kernels and
 *    fails with NPCG_ERR_CUDA when no sm_100a device is usable.
 */
#ifndef NPCG_H
#define NPCG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NPCG_ABI_VERSION 1

/* ---- status codes (pkg/src/pcgkit/errors.py:4-78) ---------------------- */
#define NPCG_OK                 0
#define NPCG_ERR_DIMENSION      1  /* DimensionMismatchError (errors.py:8)   */
#define NPCG_ERR_INVALID_FACTOR 2  /* InvalidFactorError     (errors.py:23)  */
#define NPCG_ERR_NOT_SPD        3  /* NotSpdError(pivot)     (errors.py:12)  */
#define NPCG_ERR_BREAKDOWN      4  /* BreakdownError         (errors.py:47)  */
#define NPCG_ERR_CUDA           5  /* device / launch failure                */
#define NPCG_ERR_DATA_FORMAT    6  /* DataFormatError        (errors.py:56)  */
#define NPCG_ERR_ARGUMENT       7  /* ValueError (bad handle / option)       */

/* per-system solve status written by npcg_pcg_solve */
#define NPCG_STATUS_ACTIVE     0
#define NPCG_STATUS_CONVERGED  1   /* SolveReport.converged = True           */
#define NPCG_STATUS_MAXITER    2   /* converged = False (pcg.py:171-176)     */
#define NPCG_STATUS_BREAKDOWN  3   /* pcg.py:136-140 would raise             */

typedef struct npcg_pattern npcg_pattern;   /* analysed sparsity pattern   */
typedef struct npcg_gnn npcg_gnn;           /* device-resident GNN weights */
typedef struct npcg_solver npcg_solver;     /* PCG workspace for (pattern, B) */

const char *npcg_last_error(void);
int npcg_abi_version(void);
/* 1 when a CUDA device with compute capability 10.0 is visible. */
int npcg_device_ok(void);

/* ---- patterns -----------------------------------------------------------
 * Replaces the pattern work of SparseMatrixCsr.__post_init__ (sparse.py:44-65),
 * has_full_diagonal / is_symmetric (sparse.py:133-147),
 * graph_from_system's edge_pair_index (gnn.py:83-88) and
 * A.strict_lower() (sparse.py:149-153), done once per mesh.
 *
 * Input: host CSR with int64 indices, exactly the reference layout.
 * flags: NPCG_PATTERN_FACTOR requests the triangular-solve schedules
 * (requires structural symmetry and a full diagonal; returns
 * NPCG_ERR_DATA_FORMAT otherwise, the error graph_from_system raises).
 */
#define NPCG_PATTERN_FACTOR 1
int npcg_pattern_create(int64_t n, const int64_t *row_ptr_host,
                        const int64_t *col_idx_host, int flags, npcg_pattern **out);
int npcg_pattern_destroy(npcg_pattern *p);

typedef struct {
    int64_t n, nnz, nnz_lower;
    int32_t full_diagonal, structurally_symmetric, has_factor_schedule;
    int32_t levels_lower, levels_upper;   /* global level-set depths */
    int32_t chunks;                       /* contiguous row chunks    */
    int32_t chunk_rows;                   /* rows per chunk           */
    int32_t window;                       /* smem ring depth (levels) */
    int32_t max_level_width;              /* rows per chunk-local level */
} npcg_pattern_info;
int npcg_pattern_get_info(const npcg_pattern *p, npcg_pattern_info *info);

/* The line-wavefront schedule of a factor pattern (built on first use;
 * pattern.h LineSched): grid lines, warps (32 lines each), wavefront steps,
 * and the CTAs per system (1, 2 or 4) a solve of `batch` systems launches
 * with. All zero when the pattern does not qualify and the triangular solves
 * run the level-set kernels. Any output may be NULL. */
int npcg_pattern_line_info(const npcg_pattern *p, int32_t *lines, int32_t *warps, int32_t *steps,
                           int32_t *cluster, int batch);

/* Device views owned by the pattern (int32). Any may be NULL. */
int npcg_pattern_device_arrays(const npcg_pattern *p, const int32_t **row_ptr,
                               const int32_t **col_idx, const int32_t **diag_pos,
                               const int32_t **pair, const int32_t **lower_slot);

/* Exact value-symmetry test on device for B systems (sparse.py:137-147):
 * writes ok[b] = 1 when vals[p] == vals[pair[p]] for every p (IEEE
 * equality like np.array_equal: -0.0 == 0.0, NaN never equal). */
int npcg_check_symmetric_values(const npcg_pattern *p, int B, const double *vals,
                                int vals_batched, int32_t *ok_host, void *stream);

/* ---- elementary kernels (unit parity) -----------------------------------
 * y = A x for a batch: spmv (sparse.py:213-219, 255-262). */
int npcg_spmv(const npcg_pattern *A, int B, const double *vals, int vals_batched,
              const double *x, double *y, void *stream);

/* Factor values on the pattern: S[p] for every off-diagonal slot p holds
 * L'_{ij} of the unit-lower factor with S symmetric (S[p] == S[pair[p]]).
 * From strict-lower values in A.strict_lower() slot order (gnn.py:299-311,
 * preconditioners.py:70-85): */
int npcg_factor_from_lower(const npcg_pattern *F, int B, const double *lower_vals,
                           int lower_batched, double *S, void *stream);
/* ... and back (for LowerFactor views): */
int npcg_factor_to_lower(const npcg_pattern *F, int B, const double *S,
                         double *lower_vals, void *stream);

/* z = P^{-1} r with P = (I+L') D (I+L')^T: forward unit solve, D^{-1} scale,
 * backward transpose solve (sparse.py:222-239, 265-275). D > 0 is the
 * caller's contract (LowerFactor validation, sparse.py:187-192). */
int npcg_ldlt_apply_inverse(const npcg_pattern *F, int B, const double *S, int S_batched,
                            const double *D, int D_batched, const double *r, double *z,
                            void *stream);

/* ---- GNN (gnn.py:106-318) ------------------------------------------------
 * Weights in the reference's checkpoint layout: for each layer of
 * _layer_specs order (gnn.py:130-147), W[fan_in][fan_out] row-major then
 * b[fan_out], concatenated. `width` is the latent F (FEATURE_WIDTH). */
typedef struct {
    int32_t width;        /* F: 16 or 64 */
    int32_t h, l;         /* encoder/decoder hidden width, hidden layers (l == 1) */
    int32_t h_mp, l_mp;   /* processor hidden width, hidden layers (l_mp == 1) */
    int32_t n_mp;         /* message-passing rounds */
    int32_t normalize;    /* GnnHyperParams.normalize */
    int32_t with_x0_head; /* node_dec present in the weight blob */
    /* BASELINE.json north_star extensions (0 = the reference network):
     * node inputs (b_i, boundary flag), edge inputs (A_ij, d_1..d_dim, |d|),
     * LayerNorm (gain, shift; appended to the blob after all layers, in the
     * order node_enc, edge_enc, mp0.node, mp0.edge, ...) after every encoder
     * and processor MLP, and the factor P = L L^T with L_ii = exp(M_ii). */
    int32_t north_star;
    int32_t dim;          /* mesh dimension of the edge geometry (2 or 3) */
} npcg_gnn_desc;
int npcg_gnn_create(const npcg_gnn_desc *desc, const double *weights_host,
                    int64_t n_weights, npcg_gnn **out);
int npcg_gnn_destroy(npcg_gnn *g);

/* build_learned (gnn.py:314-318) for B systems sharing A's pattern:
 * runs the GNN on (A_b, rhs_b), symmetrises (gnn.py:284-296) and writes the
 * factor values S ([nnz*B] or [nnz] when B == 1) and D = diag(A)
 * ([n*B], layout like vectors). edge_out (nullable) receives the raw edge
 * scalars M ([nnz*B]); x0_out (nullable) the node head (gnn.py:321-327).
 * Returns NPCG_ERR_NOT_SPD with *pivot set when some diag(A) <= 0. */
int npcg_gnn_build_factor(const npcg_gnn *g, const npcg_pattern *A, int B,
                          const double *A_vals, int A_batched, const double *rhs,
                          double *S, double *D, double *edge_out, double *x0_out,
                          int64_t *pivot, void *stream);

/* build_learned(model, A, b, mesh) in north_star mode (no reference
 * function: the extension of gnn.py:314-318 BASELINE.json names). pos
 * [n][dim] and boundary [n] (0 / 1) are device arrays shared by the batch
 * (one mesh). Writes the factor in the solver's unit-lower LDL^T form:
 * S = L diag(L)^-1 on the symmetric pattern, D = diag(L)^2, so
 * P = L L^T = (I + S) D (I + S)^T. NPCG_ERR_INVALID_FACTOR when L has
 * non-finite entries. */
int npcg_gnn_build_factor_mesh(const npcg_gnn *g, const npcg_pattern *A, int B,
                               const double *A_vals, int A_batched, const double *rhs,
                               const double *pos, const double *boundary,
                               double *S, double *D, double *edge_out, int64_t *pivot, void *stream);

/* ---- PCG (pcg.py:75-176) ---------------------------------------------------- */
typedef struct {
    int32_t n_thresholds;         /* SolveOptions.thresholds (strictly decreasing) */
    double thresholds[16];
    int64_t max_iter;             /* SolveOptions.max_iter or 10*n */
    int32_t absolute;             /* SolveOptions.absolute */
    int32_t check_every;          /* host polls convergence every k passes (0 = auto) */
    int32_t profile;              /* 1: time every kernel launch with CUDA events */
    int32_t history;              /* 1: keep ||r_k|| per system on the device (grown on
                                     demand) for npcg_solver_history; implied when
                                     report->history is given */
} npcg_solve_opts;

/* kernel classes reported by a profiled solve */
#define NPCG_PROF_SPMV_APDOT 0    /* Ap = A p, p.Ap, alpha            */
#define NPCG_PROF_TRSV_FWD   1    /* x,r update + forward unit solve  */
#define NPCG_PROF_SPMV_DRIFT 2    /* b - A x at threshold crossings   */
#define NPCG_PROF_TRSV_BWD   3    /* D^-1 + backward solve + r.z      */
#define NPCG_PROF_PUPD       4    /* p = z + beta p                   */
#define NPCG_PROF_OTHER      5    /* setup / polling / final residual */
#define NPCG_PROF_SLOTS      8

typedef struct {
    /* all host arrays, caller allocated */
    int32_t *status;              /* [B] NPCG_STATUS_* */
    int64_t *iterations;          /* [B] SolveReport.iterations */
    int64_t *iterations_to;       /* [B][n_thresholds], -1 = not crossed */
    double *seconds_to;           /* [B][n_thresholds] device-clock seconds */
    double *final_relative_residual; /* [B] */
    double *history;              /* [B][history_cap] ||r_k||, nullable */
    int64_t history_cap;          /* entries per system (>= max_iter+1 for full) */
    int64_t *breakdown_iteration; /* [B] k where p'Ap <= 0, else 0 */
    double *kernel_ms;            /* [NPCG_PROF_SLOTS] summed launch times (profile) */
    int64_t *kernel_launches;     /* [NPCG_PROF_SLOTS] launches per class (profile) */
    int64_t passes;               /* out: kernel-sequence passes executed */
} npcg_solve_report;

/* Kernel launches issued by this library since it was loaded (all entry
 * points), for launch accounting in benchmarks. */
int64_t npcg_launch_count(void);

/* Diagnostics: copies n entries of the line-solve timeline of block 0
 * (clock64 per pipeline batch and event, [16][2048]). All zeros unless the
 * library was built with -DNPCG_LINE_TRACE. Returns a cudaError_t code. */
int npcg_debug_line_trace(long long *out, int n);

/* Solver workspace for a (A pattern, factor pattern, B) triple. F may be
 * NULL (identity preconditioner, pcg.py:64-72) or equal A. */
int npcg_solver_create(const npcg_pattern *A, const npcg_pattern *F, int B,
                       npcg_solver **out);
int npcg_solver_destroy(npcg_solver *s);

/* Batched pcg_solve: all pointers except opts/report are device pointers.
 * x0 nullable (SolveOptions.x0). S/D ignored when the solver has F == NULL.
 * Per-system breakdown is reported in report->status; the function itself
 * returns NPCG_OK unless arguments / CUDA fail. Synchronises `stream`. */
int npcg_pcg_solve(npcg_solver *s, const double *A_vals, int A_batched,
                   const double *S, int S_batched, const double *D, int D_batched,
                   const double *b, double *x, const double *x0,
                   const npcg_solve_opts *opts, npcg_solve_report *report, void *stream);

/* SolveReport.history (pcg.py:113,145) of the last npcg_pcg_solve on `s`:
 * out[b*ld + k] = ||r_k|| for k < min(cols, max iterations + 1), host memory.
 * The device buffer grows with the iterations actually run, so callers can
 * size `out` from report->iterations instead of B x (max_iter + 1). */
int npcg_solver_history(const npcg_solver *s, double *out, int64_t ld, int64_t cols, void *stream);

/* ---- P1 FEM assembly (input side) --------------
 * Replaces pcgkit.fem.full_stiffness_and_mass / assemble's matrix part
 * (fem.py:42-69 element blocks, fem.py:116-134 COO in element order summed by
 * SparseMatrixCsr.from_coo after a stable (row, col) lexsort), for a fixed
 * triangle topology and any number of vertex sets / element coefficients.
 * Values are bit-identical to that host assembly (numpy add.reduceat order).
 *
 * npcg_fem_plan_create: host triangles int64 [nt][3] (counter-clockwise);
 * builds the lexsorted triplet plan once. NPCG_ERR_DATA_FORMAT for a vertex
 * index out of range or an empty mesh. */
typedef struct npcg_fem_plan npcg_fem_plan;
int npcg_fem_plan_create(int64_t n_vertices, int64_t n_triangles, const int64_t *triangles_host,
                         npcg_fem_plan **out);
/* The same for P1 elements with `verts_per_elem` vertices: 3 (triangles, 2-D
 * vertices) or 4 (positively oriented tetrahedra, 3-D vertices: configs 4 / 5;
 * pcgkit has no 3-D element, the host definition is inputs.tet_blocks:
 * K_ij = |T| grad l_i . grad l_j, M_ij = |T| (1 + d_ij) / 20). */
int npcg_fem_plan_create_p1(int64_t n_vertices, int64_t n_elements, int verts_per_elem, const int64_t *elements_host,
                            npcg_fem_plan **out);
int npcg_fem_plan_destroy(npcg_fem_plan *p);
/* The assembled CSR pattern: *nnz always; row_ptr [n_vertices + 1] and
 * col_idx [nnz] (host, int64, nullable) the reference's layout. */
int npcg_fem_plan_pattern(const npcg_fem_plan *p, int64_t *nnz, int64_t *row_ptr_host, int64_t *col_idx_host);

#define NPCG_FEM_K          0  /* sum of (coef_e * K_e)                    */
#define NPCG_FEM_M          1  /* sum of M_e                                */
#define NPCG_FEM_M_PLUS_SK  2  /* (sum M_e) + scale * (sum coef_e K_e)      */
/* Device assembly of B systems: vertices [n_vertices][dim][VB] (dim = 2 for
 * triangles, 3 for tetrahedra; VB = B when
 * vertices_batched, else 1), coef [nt][CB] nullable (CB = B when
 * coef_batched), values out [nnz][B]. bad_dev (device int, nullable) is set
 * to 1 when a triangle is degenerate or clockwise (fem.py raises there). */
int npcg_fem_assemble(const npcg_fem_plan *p, int B, const double *vertices, int vertices_batched,
                      const double *coef, int coef_batched, int mode, double scale, double *values,
                      int *bad_dev, void *stream);
/* Restriction of assembled values to a sub-pattern -- the Dirichlet
 * elimination of fem.py:209-215 (SparseMatrixCsr.submatrix, sparse.py:155-163)
 * on the device: dst[q] = src[sel[q]] for q < count (sel: device int32, the
 * kept slots in order), or rows of a column-minor (count, B) array when
 * `batched`. */
int npcg_gather_values(int64_t count, int B, int batched, const int32_t *sel, const double *src, double *dst,
                       void *stream);

/* ---- training step --------------------------------
 * Replaces, for one (A, b, x) tuple, train.tuple_loss + ad.backward
 * (train.py:189-205; loss_data / apply_learned_factor train.py:104-150; the
 * tape rules autodiff.py:113-253) and train.adam_step (train.py:164-185), in
 * fp64 like the reference, with a hand-written reverse pass; the reference
 * network only (l == l_mp == 1, no north_star extensions).
 *
 * npcg_trainer_create: weights in the checkpoint layout of npcg_gnn_create
 * (host); Adam moments start at zero.
 * npcg_trainer_tuple_grad: node_in [n] / edge_in [nnz] are the network inputs
 * AFTER the optional standardisation (gnn.py:239-245; the Python mirror forms
 * them with the reference's sorted statistics), A_vals [nnz], b, x [n]: all
 * device fp64. *loss_host receives the tuple loss; the parameter gradient is
 * ADDED to grad_accum [n_weights] (device; the caller sums a minibatch in
 * tuple-index order, train.py:208-226). Synchronises `stream`.
 * npcg_trainer_adam_step: one Adam update with g = grad * grad_scale (the
 * minibatch mean); *nonfinite = 1 and no update when g has a non-finite entry
 * (NonFiniteGradientError, train.py:175-176). */
typedef struct npcg_trainer npcg_trainer;
int npcg_trainer_create(const npcg_gnn_desc *desc, const double *weights_host, int64_t n_weights,
                        npcg_trainer **out);
int npcg_trainer_destroy(npcg_trainer *t);
int npcg_trainer_get_weights(const npcg_trainer *t, double *weights_host);
int npcg_trainer_set_weights(npcg_trainer *t, const double *weights_host, int reset_moments);
int npcg_trainer_tuple_grad(npcg_trainer *t, const npcg_pattern *A, const double *A_vals,
                            const double *node_in, const double *edge_in, const double *b, const double *x,
                            double x0_aux_weight, double *loss_host, double *grad_accum, void *stream);
int npcg_trainer_adam_step(npcg_trainer *t, const double *grad, double grad_scale, int64_t step,
                           double learning_rate, double beta1, double beta2, double eps, int32_t *nonfinite,
                           void *stream);

#ifdef __cplusplus
}
#endif
#endif /* NPCG_H */
