// microbench_chain.cu -- latency of the line solve's per-step dependency chain on one warp
// (nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mb tools/microbench_chain.cu)
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 4096;

template <int MODE, int KR>
__global__ void chain(double *out, long long *cyc, double f0, double f1, double f2) {
    const int t = threadIdx.x & 31;
    double h[KR], lp[KR];
    for (int c = 0; c < KR; ++c) h[c] = 1.0 + t * 1e-3 + c, lp[c] = 0.5;
    long long t0 = clock64();
#pragma unroll 8
    for (int i = 0; i < N; ++i) {
#pragma unroll
        for (int c = 0; c < KR; ++c) {
            if (MODE == 0) {  // DADD chain
                h[c] = __dadd_rn(h[c], f0);
            } else if (MODE == 1) {  // DMUL -> DADD
                h[c] = __dsub_rn(f0, __dmul_rn(f1, h[c]));
            } else if (MODE == 2) {  // SHFL.UP (64-bit) chain
                h[c] = __shfl_up_sync(0xffffffffu, h[c], 1);
            } else if (MODE == 3) {  // the solver's step: shfl, select, dmul, dsub, dsub
                const double pre = __dsub_rn(1.0, __dmul_rn(f0, lp[c]));
                const double p2 = __dmul_rn(f2, h[c]);
                double l1 = __shfl_up_sync(0xffffffffu, h[c], 1);
                if (t == 0) l1 = f0;
                double acc = __dsub_rn(pre, __dmul_rn(f1, l1));
                acc = __dsub_rn(acc, p2);
                h[c] = acc;
                lp[c] = l1;
            } else if (MODE == 4) {  // DFMA chain
                h[c] = __fma_rn(h[c], f1, f0);
            } else if (MODE == 5) {  // the step without the select
                const double pre = __dsub_rn(1.0, __dmul_rn(f0, lp[c]));
                const double p2 = __dmul_rn(f2, h[c]);
                double l1 = __shfl_up_sync(0xffffffffu, h[c], 1);
                double acc = __dsub_rn(pre, __dmul_rn(f1, l1));
                acc = __dsub_rn(acc, p2);
                h[c] = acc;
                lp[c] = l1;
            } else if (MODE == 6) {  // 32-bit shuffle chain
                float x = (float)h[c];
                x = __shfl_up_sync(0xffffffffu, x, 1);
                h[c] = x;
            }
        }
    }
    long long t1 = clock64();
    double s = 0;
    for (int c = 0; c < KR; ++c) s += h[c] + lp[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int MODE, int KR>
void run(const char *name, int warps) {
    double *out;
    long long *cyc, h;
    cudaMalloc(&out, 8 * 1024 * 32);
    cudaMalloc(&cyc, 8);
    chain<MODE, KR><<<1, 32 * warps>>>(out, cyc, 0.3, 0.2, 0.1);
    chain<MODE, KR><<<1, 32 * warps>>>(out, cyc, 0.3, 0.2, 0.1);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-44s KR=%d warps=%d  %.1f cycles/step\n", name, KR, warps, (double)h / N);
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    run<0, 1>("DADD chain", 1);
    run<4, 1>("DFMA chain", 1);
    run<1, 1>("DMUL->DSUB chain", 1);
    run<2, 1>("SHFL.UP 64-bit chain", 1);
    run<6, 1>("cvt + SHFL.UP 32-bit + cvt chain", 1);
    run<3, 1>("solver step (shfl, sel, dmul, dsub, dsub)", 1);
    run<5, 1>("solver step without select", 1);
    run<3, 2>("solver step", 1);
    run<3, 4>("solver step", 1);
    run<3, 1>("solver step", 4);
    run<3, 2>("solver step", 4);
    run<3, 4>("solver step", 4);
    run<3, 1>("solver step", 8);
    run<3, 2>("solver step", 8);
    run<3, 1>("solver step", 16);
    return 0;
}
