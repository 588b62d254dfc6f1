// microbench_step.cu -- the line solver's step loop on one warp, features toggled one by one
// (nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_step tools/microbench_step.cu)
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kStages = 256, G = 4, STEPS = 16, kTileSlots = 128, kKinds = 3;
enum { F_XL = 1, F_LDS = 2, F_STS = 4, F_RING = 8, F_GENERIC = 16, F_NOSEL = 32 };

__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void st_dsm(unsigned addr, double v) {
    asm volatile("st.relaxed.cluster.shared::cluster.b64 [%0], %1;" ::"r"(addr), "l"(__double_as_longlong(v)) : "memory");
}
__device__ __forceinline__ void st_gen(double *p, double v) {
    asm volatile("st.relaxed.cluster.b64 [%0], %1;" ::"l"(p), "l"(__double_as_longlong(v)) : "memory");
}
__device__ __forceinline__ int tile_elem(int q, int t) { return (q >> 1) * 64 + t * 2 + (q & 1); }

__device__ volatile int g_stop;

template <int FLAGS, int KR>
__global__ void __launch_bounds__(256, 1) step_kernel(double *out, long long *cyc, int Q0, int Q1, int R, int nline,
                                                      int noise_gap) {
    extern __shared__ __align__(128) double sm[];
    const int t = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (w >= nline) {  // helper-like traffic: 16-byte shared loads / stores, `noise_gap` idle cycles between bursts
        double2 *buf = reinterpret_cast<double2 *>(sm + (size_t)w * (G * (kKinds + 3 * KR) * kTileSlots + 64 * KR));
        double2 a = make_double2(1.0, 2.0);
        for (int it = 0; it < 20000; ++it) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                double2 v = buf[t + 32 * k];
                a.x += v.x;
                a.y += v.y;
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) buf[t + 32 * (8 + k)] = a;
            if (noise_gap) __nanosleep(noise_gap);
            if (g_stop) break;
        }
        out[blockIdx.x * blockDim.x + threadIdx.x] = a.x + a.y;
        return;
    }
    double *f = sm + (size_t)w * (G * (kKinds + 3 * KR) * kTileSlots + 64 * KR);
    double *vin = f + G * kKinds * kTileSlots;
    double *ring = f + G * (kKinds + 3 * KR) * kTileSlots;
    constexpr int kVec = G * kTileSlots;
    for (int i = t; i < G * (kKinds + 3 * KR) * kTileSlots; i += 32) f[i] = 1e-3 * (i % 17);
    __syncwarp();
    unsigned rout;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rout) : "r"(smem_u32(ring)), "r"(0));
    double *rgen = ring;
    asm volatile("mapa.u64 %0, %1, %2;" : "=l"(rgen) : "l"(ring), "r"(0));
    const bool prod = t == 31;
    double h0[KR], lp[KR], x[KR];
    for (int c = 0; c < KR; ++c) h0[c] = 1.0 + t * 1e-3, lp[c] = 0.5, x[c] = 0.25 + t;
    long long t0 = clock64();
    for (int j = 0; j < kStages; ++j) {
        const int sig = j * STEPS;
        auto pair_at = [&](int i) {
            const int tp = i / 4;
            const int e = tile_elem(i % 4, t);
            return make_int2(tp * kKinds * kTileSlots + e, tp * kTileSlots + e);
        };
        auto pair_ops = [&](int i, double2 &f0, double2 &f1, double2 &f2, double2 (&a0)[KR]) {
            if (FLAGS & F_LDS) {
                const int2 o = pair_at(i);
                f0 = *reinterpret_cast<const double2 *>(f + o.x);
                f1 = *reinterpret_cast<const double2 *>(f + o.x + kTileSlots);
                f2 = *reinterpret_cast<const double2 *>(f + o.x + 2 * kTileSlots);
#pragma unroll
                for (int c = 0; c < KR; ++c) a0[c] = *reinterpret_cast<const double2 *>(vin + 3 * c * kVec + o.y);
            } else {
                f0 = make_double2(0.01, 0.02), f1 = make_double2(0.03, 0.04), f2 = make_double2(0.05, 0.06);
#pragma unroll
                for (int c = 0; c < KR; ++c) a0[c] = make_double2(1.0, 2.0);
            }
        };
        double2 cf0, cf1, cf2, ca0[KR];
        pair_ops(0, cf0, cf1, cf2, ca0);
#pragma unroll
        for (int pi = 0; pi < STEPS / 2; ++pi) {
            const int i = 2 * pi;
            double2 nf0, nf1, nf2, na0[KR];
            if (pi + 1 < STEPS / 2) pair_ops(i + 2, nf0, nf1, nf2, na0);
            const double F0[2] = {cf0.x, cf0.y}, F1[2] = {cf1.x, cf1.y}, F2[2] = {cf2.x, cf2.y};
            double A[KR][2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int step = sig + i + h;
                const bool send = prod && step >= Q0 && step < Q1;
#pragma unroll
                for (int c = 0; c < KR; ++c) {
                    const double V = h == 0 ? ca0[c].x : ca0[c].y;
                    const double pre = __dsub_rn(V, __dmul_rn(F0[h], lp[c]));
                    const double p2 = __dmul_rn(F2[h], h0[c]);
                    double l1 = __shfl_up_sync(0xffffffffu, h0[c], 1);
                    if (FLAGS & F_XL) {
                        const double xl = __shfl_sync(0xffffffffu, x[c], i + h);
                        if (t == 0) l1 = xl;
                    } else if (!(FLAGS & F_NOSEL)) {
                        if (t == 0) l1 = x[c];
                    }
                    double acc = __dsub_rn(pre, __dmul_rn(F1[h], l1));
                    acc = __dsub_rn(acc, p2);
                    h0[c] = acc;
                    lp[c] = l1;
                    if (FLAGS & F_RING) {
                        if (FLAGS & F_GENERIC) {
                            if (send) st_gen(rgen + ((step & (R - 1)) * KR + c), acc);
                        } else {
                            if (send) st_dsm(rout + (unsigned)((step & (R - 1)) * KR + c) * 8u, acc);
                        }
                    }
                    A[c][h] = acc;
                }
            }
            if (FLAGS & F_STS) {
                const int2 o = pair_at(i);
#pragma unroll
                for (int c = 0; c < KR; ++c)
                    *reinterpret_cast<double2 *>(vin + (3 * c + 1) * kVec + o.y) = make_double2(A[c][0], A[c][1]);
            }
            if (pi + 1 < STEPS / 2) {
                cf0 = nf0, cf1 = nf1, cf2 = nf2;
#pragma unroll
                for (int c = 0; c < KR; ++c) ca0[c] = na0[c];
            }
        }
        __syncwarp();
    }
    long long t1 = clock64();
    double s = 0;
    for (int c = 0; c < KR; ++c) s += h0[c] + lp[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        *cyc = t1 - t0;
        g_stop = 1;
    }
}

template <int FLAGS, int KR>
void run(const char *name, int warps = 1, int noise = 0, int gap = 0) {
    double *out;
    long long *cyc, h;
    cudaMalloc(&out, 8 * 1024 * 32);
    cudaMalloc(&cyc, 8);
    auto k = step_kernel<FLAGS, KR>;
    const int smem = (warps + noise) * (G * (kKinds + 3 * KR) * kTileSlots + 64 * KR) * 8;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int r = 0; r < 2; ++r) {
        int zero = 0;
        cudaMemcpyToSymbol(g_stop, &zero, sizeof(int));
        k<<<1, 32 * (warps + noise), smem>>>(out, cyc, 64, 1 << 30, 64, warps, gap);
    }
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-58s KR=%d warps=%d noise=%d gap=%d  %.1f cycles/step  %s\n", name, KR, warps, noise, gap,
           (double)h / (kStages * STEPS),
           e == cudaSuccess ? "" : cudaGetErrorString(e));
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    run<0, 1>("chain only (select on t == 0)");
    run<F_NOSEL, 1>("chain only, no select");
    run<F_XL, 1>("+ xl shuffle");
    run<F_LDS, 1>("+ operand loads (LDS.128, one pair ahead)");
    run<F_LDS | F_STS, 1>("+ loads + result stores");
    run<F_LDS | F_STS | F_XL, 1>("+ loads + stores + xl");
    run<F_LDS | F_STS | F_XL | F_RING, 1>("+ loads + stores + xl + ring store (shared::cluster)");
    run<F_LDS | F_STS | F_XL | F_RING | F_GENERIC, 1>("+ loads + stores + xl + ring store (generic, hoisted)");
    run<F_LDS | F_STS | F_RING | F_GENERIC, 1>("+ loads + stores + ring (generic), no xl");
    run<F_LDS | F_STS | F_XL | F_RING, 2>("everything");
    run<F_LDS | F_STS | F_XL | F_RING | F_GENERIC, 2>("everything, generic ring store");
    run<F_LDS | F_STS | F_RING | F_GENERIC, 2>("no xl, generic ring store");
    run<F_LDS | F_STS | F_XL | F_RING, 1>("everything", 4);
    run<F_LDS | F_STS | F_XL | F_RING, 2>("everything", 4);
    run<F_LDS | F_STS | F_XL | F_RING, 4>("everything");
    // four line warps next to four warps of helper-like shared-memory traffic
    run<F_LDS | F_STS | F_XL | F_RING | F_GENERIC, 1>("everything + 4 noise warps, back to back", 4, 4, 0);
    run<F_LDS | F_STS | F_XL | F_RING | F_GENERIC, 1>("everything + 4 noise warps, 200 ns gaps", 4, 4, 200);
    run<F_LDS | F_STS | F_XL | F_RING | F_GENERIC, 1>("everything + 4 noise warps, 1 us gaps", 4, 4, 1000);
    run<F_LDS | F_STS | F_XL | F_RING | F_GENERIC, 1>("everything, no noise", 4, 0, 0);
    return 0;
}
