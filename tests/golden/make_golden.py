"""Golden vectors produced by the REFERENCE itself (pcgkit), for parity tests.

Runs only in the build container (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba \
        python tests/golden/make_golden.py

Inputs are generated with this repo's seeded vertex jitter / random fields
(paper_2305_16432_b200.inputs) but ASSEMBLED by the reference
(pcgkit.mesh.TriangleMesh + pcgkit.fem element formulas, fem.py:42-215),
so tests/test_inputs.py can pin our generator against the reference's
assembly. Everything downstream -- GNN edge scalars, L', PCG x / history /
iterations -- is pcgkit's own output (gnn.py:266-318, pcg.py:75-176).

Weight sets:
  trained   -- tests/golden/heat_trained.json (mint_checkpoint.py), F=16, 5 rounds
  perturbed -- create_model(hyper, seed) with processor output layers x10
               (cancels the 0.1 init gain), recorded in the file
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from pcgkit import fem, gnn, mesh as rmesh, pcg, sparse  # noqa: E402

from paper_2305_16432_b200 import inputs  # noqa: E402  (vertex jitter / random fields only)


def ref_mesh(m2d, dirichlet):
    marks = np.zeros(len(m2d.vertices), dtype=np.uint8)
    marks[m2d.boundary] = rmesh.DIRICHLET if dirichlet else rmesh.NEUMANN
    return rmesh.TriangleMesh(m2d.vertices, m2d.triangles, marks)


def ref_stiffness_mass(tm, coef=None):
    """fem.full_stiffness_and_mass (fem.py:116-134) with an optional
    per-element coefficient on K (the configs need it; fem.py has scalars)."""
    tris = tm.triangles
    rows = np.repeat(tris, 3, axis=1).ravel()
    cols = np.tile(tris, (1, 3)).ravel()
    kv = np.empty(9 * len(tris))
    mv = np.empty(9 * len(tris))
    for e, tri in enumerate(tris):
        ke = fem.element_stiffness(tm.vertices[tri])
        if coef is not None:
            ke = coef[e] * ke
        kv[9 * e:9 * e + 9] = ke.ravel()
        mv[9 * e:9 * e + 9] = fem.element_mass(tm.vertices[tri]).ravel()
    K = sparse.SparseMatrixCsr.from_coo(tm.n_vertices, rows, cols, kv)
    M = sparse.SparseMatrixCsr.from_coo(tm.n_vertices, rows, cols, mv)
    return K, M


def perturbed(hyper, seed):
    model = gnn.create_model(hyper, seed=seed)
    for r in range(hyper.n_mp):
        for s in ("node", "edge"):
            model.params[f"mp{r}.{s}.{hyper.l_mp}.w"] *= 10.0
    return model


def solve_record(A, b, P, thresholds, max_iter):
    x, rep = pcg.pcg_solve(A, b, P, pcg.SolveOptions(thresholds=thresholds, max_iter=max_iter))
    it_to = np.array([rep.iterations_to.get(t, -1) for t in thresholds], dtype=np.int64)
    return dict(x=x, iterations=rep.iterations, history=np.array(rep.history),
                iterations_to=it_to, converged=rep.converged,
                final_rel=rep.final_relative_residual)


def factor_record(model, A, b):
    g = gnn.graph_from_system(A, b)
    M, x0 = gnn.run(model, g)
    lower = gnn.symmetrize_triangulate(M, g)
    P = gnn.assemble_preconditioner(lower, A)
    return M, lower, x0, P


def save(name, A, rhs, cases, meta, model_params=None, extra=None):
    out = dict(n=A.n, row_ptr=A.row_ptr, col_idx=A.col_idx, values=A.values, rhs=rhs)
    for k, v in (extra or {}).items():
        out[k] = v
    for ci, c in enumerate(cases):
        for k, v in c.items():
            out[f"c{ci}_{k}"] = np.asarray(v)
    if model_params is not None:
        blob = np.concatenate([np.ravel(model_params[k]) for k in sorted(model_params)])
        meta = dict(meta, params_sha256=__import__("hashlib").sha256(blob.tobytes()).hexdigest())
        if blob.size <= 20000:  # small nets: store the weights themselves (pins create_model)
            for k, v in model_params.items():
                out["param:" + k] = v
    out["meta"] = np.array(json.dumps(meta))
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes", meta.get("summary", ""))


def heat_case(tag, model, hyper_meta, k=32, thresholds=(1e-8,), max_iter=2000):
    rng = inputs.streams(1, 1)[0]
    m2d = inputs.unit_square(k, 0.2, rng)
    tm = ref_mesh(m2d, dirichlet=False)
    K, M = ref_stiffness_mass(tm)
    dt, alpha = 1e-2, 1.0
    A = sparse.SparseMatrixCsr(tm.n_vertices, K.row_ptr, K.col_idx, M.values + (dt * alpha) * K.values)
    u0 = inputs.gaussian_bumps(m2d.vertices, rng)
    b = sparse.spmv(M, u0)
    Mv, lower, x0, P = factor_record(model, A, b)
    rec = solve_record(A, b, P, thresholds, max_iter)
    rec_all = solve_record(A, b, P, pcg.DEFAULT_THRESHOLDS, max_iter)
    rng2 = np.random.default_rng(99)
    r = rng2.standard_normal(A.n)
    cases = [dict(M=Mv, lower=lower, x0=x0 if x0 is not None else np.zeros(0), **rec,
                  all_iterations_to=rec_all["iterations_to"], all_history=rec_all["history"],
                  probe_r=r, probe_z=P.apply_inverse(r), probe_Ar=sparse.spmv(A, r))]
    meta = dict(kind="heat2d", k=k, jitter=0.2, dt=dt, cfg_stream=1, thresholds=list(thresholds),
                max_iter=max_iter, **hyper_meta,
                summary=f"n={A.n} it={rec['iterations']} |L'|max={np.abs(lower).max():.3g}")
    save(f"{tag}", A, b[:, None], cases, meta, model.params if "checkpoint" not in hyper_meta else None)


def poisson_case(tag, model, hyper_meta, k=64, nrhs=3, thresholds=(1e-8,)):
    rngs = inputs.streams(2, nrhs)
    m2d = inputs.unit_square(k, 0.2, rngs[0])
    tm = ref_mesh(m2d, dirichlet=True)
    cases = []
    rhs = []
    A = None
    for j, rng in enumerate(rngs):
        f = inputs.grf_2d(m2d.vertices, rng, rng.uniform(0.05, 0.3))
        sysj = fem.assemble(tm, fem.PdeProblem("poisson", source=f))
        A = sysj.A
        rhs.append(sysj.b)
    B = np.stack(rhs, axis=1)
    Mv, lower, _, P = factor_record(model, A, B[:, 0])  # one shared L' from RHS 0
    for j in range(nrhs):
        rec = solve_record(A, B[:, j], P, thresholds, None)
        cases.append(dict(**rec))
    meta = dict(kind="poisson2d", k=k, jitter=0.2, cfg_stream=2, nrhs=nrhs, thresholds=list(thresholds),
                **hyper_meta, summary=f"n={A.n} it={[c['iterations'] for c in cases]}")
    save(tag, A, B, cases, meta, model.params, extra=dict(M=Mv, lower=lower))


def wave_case(tag, model, hyper_meta, k=48, nsys=2, thresholds=(1e-8,)):
    rngs = inputs.streams(3, nsys)
    m2d = inputs.unit_square(k, 0.2, np.random.default_rng(np.random.SeedSequence(3017).entropy))
    tm = ref_mesh(m2d, dirichlet=False)
    cent = m2d.vertices[m2d.triangles].mean(axis=1)
    dt = 1e-3
    vals, rhs, cases = [], [], []
    A0 = None
    for rng in rngs:
        c = np.exp(0.5 * inputs.grf_2d(cent, rng, rng.uniform(0.05, 0.3)))
        K, M = ref_stiffness_mass(tm, coef=c)
        A = sparse.SparseMatrixCsr(tm.n_vertices, K.row_ptr, K.col_idx, M.values + (dt * dt) * K.values)
        b = sparse.spmv(M, inputs.grf_2d(m2d.vertices, rng, rng.uniform(0.05, 0.3)))
        Mv, lower, _, P = factor_record(model, A, b)
        rec = solve_record(A, b, P, thresholds, None)
        cases.append(dict(M=Mv, lower=lower, **rec))
        vals.append(A.values)
        rhs.append(b)
        A0 = A0 or A
    meta = dict(kind="wave2d", k=k, jitter=0.2, dt=dt, cfg_stream=3, nsys=nsys, thresholds=list(thresholds),
                **hyper_meta, summary=f"n={A0.n} it={[c['iterations'] for c in cases]}")
    save(tag, A0, np.stack(rhs, axis=1), cases, meta, model.params, extra=dict(values_batch=np.stack(vals, axis=1)))


def main():
    # 1. trained checkpoint (F=16, 5 rounds, x0 head) on the config-1 input
    model = gnn.load_model(os.path.join(HERE, "heat_trained.json"))
    heat_case("cfg1_trained", model, dict(weights="trained", checkpoint="heat_trained.json", width=16))
    # 2. config-1 network shape: F=16, 3 rounds, perturbed seeded weights
    hyper = gnn.GnnHyperParams(l=1, h=16, n_mp=3, l_mp=1, h_mp=16)
    heat_case("cfg1_perturbed", perturbed(hyper, 0),
              dict(weights="perturbed x10", seed=0, width=16, n_mp=3, h=16, h_mp=16))
    # 3./4. latent 64 (FEATURE_WIDTH monkeypatch)
    old = gnn.FEATURE_WIDTH
    gnn.FEATURE_WIDTH = 64
    try:
        hyper = gnn.GnnHyperParams(l=1, h=64, n_mp=5, l_mp=1, h_mp=64)
        seed = int(os.environ.get("GOLDEN_SEED64", "3"))
        poisson_case("cfg2_small_f64", perturbed(hyper, seed),
                     dict(weights="perturbed x10", seed=seed, width=64, n_mp=5, h=64, h_mp=64))
        wave_case("cfg3_small_f64", perturbed(hyper, seed),
                  dict(weights="perturbed x10", seed=seed, width=64, n_mp=5, h=64, h_mp=64))
    finally:
        gnn.FEATURE_WIDTH = old


if __name__ == "__main__":
    main()
