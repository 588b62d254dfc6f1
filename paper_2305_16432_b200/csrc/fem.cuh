// fem.cuh -- device P1 FEM assembly (fem.cu).
#pragma once
#include <cuda_runtime.h>

#include <string>
#include <vector>

namespace npcg {

enum FemMode : int { FEM_K = 0, FEM_M = 1, FEM_M_PLUS_SK = 2 };  // include/npcg.h NPCG_FEM_*

struct FemArgs {
    int nnz = 0, B = 1, nt = 0;
    int nper2 = 9;                // block entries per element: 9 (triangles) or 16 (tetrahedra)
    const int *starts = nullptr;  // [nnz + 1] runs of triplet ids per CSR slot
    const int *order = nullptr;   // [nper2 nt] triplet ids in lexsort order
    const int *tri = nullptr;     // [nt][3] or [nt][4]
    const double *V = nullptr;    // vertices [nv][dim][vb], dim = 2 or 3
    int vb = 1;                   // B when every system has its own vertices, else 1
    const double *coef = nullptr; // per-element stiffness coefficient [nt][cb] (nullable)
    int cb = 1;
    int mode = FEM_K;
    double scale = 1.0;           // s of M + s K
    double *out = nullptr;        // [nnz][B]
    double *kq = nullptr;         // plan scratch: unscaled stiffness entry per triplet [9 nt] (shared vertices)
    double *ms = nullptr;         // plan scratch: mass sum per slot [nnz]
    double *mq = nullptr;         // plan scratch: mass entry per triplet [9 nt]
};

struct FemPlanHost {
    std::vector<int> order, starts, col;
    std::vector<long long> row_ptr;
};

// stable (row, col) lexsort of the nper^2 nt triplets (fem.py:116-134); "" or an error
std::string fem_plan_build(long long nv, long long nt, int nper, const long long *elems, FemPlanHost &h);
cudaError_t launch_fem_assemble(const FemArgs &a, int *bad, cudaStream_t s);

}  // namespace npcg
