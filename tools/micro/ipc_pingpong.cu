// Probe: cross-process device-flag ping-pong on one GPU through CUDA IPC.
// Two processes (server / client) each run ONE kernel that exchanges N
// ping/pong rounds through system-scope flags in the server's allocation.
// Bounded by %globaltimer (no hang): prints rounds done and us per round.
//   ipc_pingpong server <dir> N     ipc_pingpong client <dir> N
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <unistd.h>

__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ unsigned long long ld_acq(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_rel(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__global__ void k_pp(unsigned long long *f, int n, int server, int *out) {
    const unsigned long long t0 = gtime();
    int k = 1;
    for (; k <= n; ++k) {
        if (server) {
            st_rel(f, k);
            while (ld_acq(f + 1) < (unsigned long long)k)
                if (gtime() - t0 > 20000000000ull) { out[0] = k - 1; return; }
        } else {
            while (ld_acq(f) < (unsigned long long)k)
                if (gtime() - t0 > 20000000000ull) { out[0] = k - 1; return; }
            st_rel(f + 1, k);
        }
    }
    out[0] = n;
}
int main(int argc, char **argv) {
    if (argc < 4) return 2;
    const bool server = !strcmp(argv[1], "server");
    const std::string dir = argv[2];
    const int n = atoi(argv[3]);
    unsigned long long *f = nullptr;
    if (server) {
        cudaMalloc(&f, 64);
        cudaMemset(f, 0, 64);
        cudaIpcMemHandle_t h;
        if (cudaIpcGetMemHandle(&h, f) != cudaSuccess) { printf("get handle failed\n"); return 1; }
        FILE *o = fopen((dir + "/h.tmp").c_str(), "wb");
        fwrite(&h, sizeof h, 1, o);
        fclose(o);
        rename((dir + "/h.tmp").c_str(), (dir + "/h.bin").c_str());
    } else {
        cudaIpcMemHandle_t h;
        FILE *i = nullptr;
        for (int q = 0; q < 600 && !(i = fopen((dir + "/h.bin").c_str(), "rb")); ++q) usleep(100000);
        if (!i) { printf("no handle\n"); return 1; }
        fread(&h, sizeof h, 1, i);
        fclose(i);
        cudaError_t e = cudaIpcOpenMemHandle((void **)&f, h, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) { printf("open failed: %s\n", cudaGetErrorString(e)); return 1; }
    }
    int *out;
    cudaMallocManaged(&out, 4);
    *out = -1;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k_pp<<<1, 1>>>(f, n, server, out);
    cudaEventRecord(b);
    cudaError_t e = cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    printf("%s: %s rounds %d/%d in %.3f ms = %.2f us/round\n", argv[1], cudaGetErrorString(e), *out, n, ms,
           *out > 0 ? 1e3 * ms / *out : -1.0);
    if (server) { sleep(1); }
    return 0;
}
