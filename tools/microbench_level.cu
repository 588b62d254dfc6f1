// microbench_level.cu -- cycles per "level step" for the ingredients of the
// triangular-solve loop on sm_100a (one thread walks a dependency chain).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_level tools/microbench_level.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

// FEAT bits: 1 global store, 2 cp.async pipeline (depth D), 4 syncthreads,
//            8 TMA bulk + mbarrier pipeline (depth D), 16 fence.proxy.async
template <int FEAT, int D>
__global__ void chain(double *gout, const double *gin, long long *cycles, int iters) {
    __shared__ double ring[64];
    __shared__ __align__(128) double stage[64][16];
    __shared__ __align__(8) unsigned long long bar[64];
    const int lane = threadIdx.x & 31;
    double acc = 1.0;
    if (threadIdx.x < 64) ring[threadIdx.x] = 0.5;
    if ((FEAT & 8) && threadIdx.x == 0) {
        for (int i = 0; i < 64; ++i)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[i])) : "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    auto tma = [&](int slot, int it) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 128;" ::"r"(smem_u32(&bar[slot])) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 128, [%2];" ::"r"(
                         smem_u32(&stage[slot][0])),
                     "l"(gin + ((it * 16 * 7) & 65535)), "r"(smem_u32(&bar[slot]))
                     : "memory");
    };
    if ((FEAT & 8) && threadIdx.x == 0)
        for (int s = 0; s < D; ++s) tma(s, s);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        if (FEAT & 2) asm volatile("cp.async.wait_group %0;" ::"n"(D - 1) : "memory");
        if (FEAT & 4) __syncthreads();
        else __syncwarp();
        if (FEAT & 8) {
            const unsigned slot = it % D, par = (it / D) & 1;
            asm volatile(
                "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(
                    smem_u32(&bar[slot])),
                "r"(par)
                : "memory");
        }
        if (threadIdx.x == 0) {
            double y = ring[it & 63];
            double s = (FEAT & 10) ? stage[it % D][0] + 0.25 : 0.25;
            acc = __dsub_rn(y, __dmul_rn(s, acc));
            ring[(it + 1) & 63] = acc;
            if (FEAT & 1)
                asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(gout + (it & 1023)),
                             "l"(__double_as_longlong(acc)) : "memory");
        }
        if (FEAT & 2) {
            if (lane == 0)
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(&stage[it % D][0])),
                             "l"(gin + ((it * 97) & 65535)) : "memory");
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
        if ((FEAT & 8) && threadIdx.x == 0) {
            if (FEAT & 16) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            if (it + D < iters) tma(it % D, it + D);
        }
        if (FEAT & 8) __syncwarp();
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) {
        cycles[blockIdx.x] = t1 - t0;
        gout[2000] = acc;
    }
}

int main() {
    double *gout, *gin;
    long long *cyc;
    cudaMalloc(&gout, 4096 * 8);
    cudaMalloc(&gin, 65536 * 8);
    cudaMemset(gin, 0, 65536 * 8);
    cudaMallocManaged(&cyc, 1024 * 8);
    const int iters = 4096;
    auto run = [&](const char *name, void (*k)(double *, const double *, long long *, int), int threads) {
        k<<<1, threads>>>(gout, gin, cyc, iters);
        cudaDeviceSynchronize();
        k<<<1, threads>>>(gout, gin, cyc, iters);
        cudaDeviceSynchronize();
        printf("%-52s %7.1f cycles/step\n", name, (double)cyc[0] / iters);
    };
    run("smem chain + syncwarp", chain<0, 4>, 32);
    run("+ relaxed global store", chain<1, 4>, 32);
    run("+ cp.async pipeline D=4", chain<3, 4>, 32);
    run("+ cp.async pipeline D=16", chain<3, 16>, 32);
    run("+ cp.async pipeline D=32", chain<3, 32>, 32);
    run("+ __syncthreads (8 warps), D=16", chain<7, 16>, 256);
    run("store + TMA/mbarrier pipeline D=4", chain<9, 4>, 32);
    run("store + TMA/mbarrier pipeline D=16", chain<9, 16>, 32);
    run("store + TMA/mbarrier D=16 + fence.proxy.async", chain<25, 16>, 32);
    run("store + cp.async D=16 + TMA D=16 + syncthreads(8w)", chain<15, 16>, 256);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
