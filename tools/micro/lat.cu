// Microbenchmark: dependent-chain latencies on sm_100a (DFMA, FFMA, LDS, IMAD)
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double *out, long long *cyc, int n, int mode) {
    __shared__ double sm[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = 1.0 + i * 1e-9;
    __syncthreads();
    double a = out[threadIdx.x], b = 1.0000001, c = 1e-9;
    float fa = (float)a, fb = 1.0001f, fc = 1e-5f;
    int idx = threadIdx.x & 7; unsigned ia = threadIdx.x;
    long long t0 = clock64();
    if (mode == 0) { for (int i = 0; i < n; ++i) a = __fma_rn(a, b, c); }
    else if (mode == 1) { for (int i = 0; i < n; ++i) fa = __fmaf_rn(fa, fb, fc); a = fa; }
    else if (mode == 2) { for (int i = 0; i < n; ++i) { idx = (int)sm[idx] & 7; } a = idx; }
    else if (mode == 3) { for (int i = 0; i < n; ++i) ia = ia * 3u + 7u; a = ia; }
    else if (mode == 4) { for (int i = 0; i < n; ++i) a = a * b; }
    else if (mode == 5) { for (int i = 0; i < n; ++i) a = a + c; }
    long long t1 = clock64();
    out[threadIdx.x] = a;
    if (threadIdx.x == 0) cyc[mode] = (t1 - t0);
}
__global__ void thr(double *out, long long *cyc, int n) {  // DFMA throughput: 8 independent chains per thread
    double a[8]; for (int q = 0; q < 8; ++q) a[q] = out[threadIdx.x] + q;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i)
#pragma unroll
        for (int q = 0; q < 8; ++q) a[q] = __fma_rn(a[q], 1.0000001, 1e-9);
    long long t1 = clock64();
    double s = 0; for (int q = 0; q < 8; ++q) s += a[q];
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
    double *out; long long *cyc; cudaMalloc(&out, 1 << 20); cudaMalloc(&cyc, 4096);
    cudaMemset(out, 0, 1 << 20);
    const char *names[] = {"DFMA", "FFMA", "LDS(dep)", "IMAD", "DMUL", "DADD"};
    for (int m = 0; m < 6; ++m) {
        int n = 4096;
        k<<<1, 32>>>(out, cyc, n, m); cudaDeviceSynchronize();
        long long c; cudaMemcpy(&c, cyc + m, 8, cudaMemcpyDeviceToHost);
        printf("%-9s latency %.2f cycles (1 warp)\n", names[m], (double)c / n);
    }
    for (int warps : {1, 2, 4, 8, 16, 32}) {
        int n = 1024;
        thr<<<1, 32 * warps>>>(out, cyc, n); cudaDeviceSynchronize();
        long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        printf("DFMA throughput, %2d warps x 8 chains: %.3f DFMA/cycle/SM\n", warps, 32.0 * warps * 8 * n / c);
    }
    return 0;
}
