// Microbenchmark of one "record" step of the level-set consumer in isolation:
// 128 threads: 12 LDS.128 + 3 LDS.64 (block values), 12 LDS.64 gathers,
// 27 DFMA in 3 chains, 3 STS, bar.sync -- repeated ITER times.
// Optional: a 5th warp streams HBM -> smem with cp.async.bulk concurrently.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <bool TMA>
__global__ void rec(const uint8_t *src, long long *out, int iters, int nbytes) {
    extern __shared__ __align__(128) uint8_t sm[];
    double *vec = (double *)sm;                  // 48 KB
    uint8_t *val = sm + 49152;                   // 32 KB of "record" data
    uint8_t *ring = sm + 49152 + 32768;          // 32 KB TMA target
    __shared__ uint64_t bar;
    const int t = threadIdx.x;
    for (int q = t; q < 6144; q += blockDim.x) vec[q] = 1.0 + q * 1e-7;
    for (int q = t; q < 4096; q += blockDim.x) ((double *)val)[q] = 1e-3 * (q & 7);
    if (t == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)));
    __syncthreads();
    if (t >= 128) {
        if (TMA && t == 128) {
            uint32_t ph = 0;
            for (int off = 0; off + 16384 <= nbytes; off += 16384) {
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar)), "r"(16384));
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             ::"r"(su(ring + (off & 16383))), "l"(src + off), "r"(16384), "r"(su(&bar)) : "memory");
                uint32_t ok = 0;
                while (!ok) asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }" : "=r"(ok) : "r"(su(&bar)), "r"(ph));
                ph ^= 1;
            }
        }
        return;
    }
    double a0 = 0, a1 = 0, a2 = 0;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const int row = (t * 13 + it * 7) & 2047;
        double B[3][9];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const uint8_t *b = val + k * 128 * 80 + 16 * t;
            double2 p0 = *(const double2 *)(b), p1 = *(const double2 *)(b + 2048), p2 = *(const double2 *)(b + 4096), p3 = *(const double2 *)(b + 6144);
            B[k][0] = p0.x; B[k][1] = p0.y; B[k][2] = p1.x; B[k][3] = p1.y; B[k][4] = p2.x; B[k][5] = p2.y; B[k][6] = p3.x; B[k][7] = p3.y;
            B[k][8] = *(const double *)(val + k * 128 * 80 + 8192 + 8 * t);
        }
        a0 = vec[3 * row]; a1 = vec[3 * row + 1]; a2 = vec[3 * row + 2];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const int j = (row + 1 + 16 * k) & 2047;
            const double x0 = vec[3 * j], x1 = vec[3 * j + 1], x2 = vec[3 * j + 2];
            a0 = __fma_rn(-B[k][0], x0, a0); a1 = __fma_rn(-B[k][3], x0, a1); a2 = __fma_rn(-B[k][6], x0, a2);
            a0 = __fma_rn(-B[k][1], x1, a0); a1 = __fma_rn(-B[k][4], x1, a1); a2 = __fma_rn(-B[k][7], x1, a2);
            a0 = __fma_rn(-B[k][2], x2, a0); a1 = __fma_rn(-B[k][5], x2, a1); a2 = __fma_rn(-B[k][8], x2, a2);
        }
        vec[3 * row] = a0 * 1e-9; vec[3 * row + 1] = a1 * 1e-9; vec[3 * row + 2] = a2 * 1e-9;
        asm volatile("bar.sync 1, 128;" ::: "memory");
    }
    long long t1 = clock64();
    if (t == 0) out[blockIdx.x] = (t1 - t0) / iters;
}
int main() {
    uint8_t *src; long long *out; cudaMalloc(&src, 1 << 30); cudaMalloc(&out, 8 * 4096);
    cudaMemset(src, 0, 1 << 30);
    int smem = 49152 + 65536;
    cudaFuncSetAttribute(rec<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(rec<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int tma = 0; tma < 2; ++tma)
        for (int grid : {1, 148, 296}) {
            if (tma) rec<true><<<grid, 160, smem>>>(src, out, 2000, 1 << 22);
            else rec<false><<<grid, 160, smem>>>(src, out, 2000, 1 << 22);
            cudaDeviceSynchronize();
            long long c[296]; cudaMemcpy(c, out, 8 * grid, cudaMemcpyDeviceToHost);
            double s = 0; for (int i = 0; i < grid; ++i) s += c[i];
            printf("tma=%d grid=%3d: %.0f cycles per record-step (%s)\n", tma, grid, s / grid, cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}
