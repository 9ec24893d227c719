// peer.cu -- signal / wait / put kernels of the peer-memory transport
// (DD_COMM_LOCAL, DD_COMM_IPC; see peer.cuh). One thread each, except the
// row put; the dot all-gather + finalize lives in krylov.cu next to the other
// finalizers.
#include <algorithm>

#include "peer.cuh"

namespace ddk {

namespace {

__device__ __forceinline__ bool skip_now(const int *skip) {
    return skip && *reinterpret_cast<const volatile int *>(skip) != 0;
}

__global__ void k_peer_signal(PeerDev d, int ch, const int32_t *peers, int n, const int *skip) {
    if (threadIdx.x != 0 || skip_now(skip)) return;
    const unsigned long long s = ++d.seq[ch];
    // the producer kernel before this one fenced its stores (system scope);
    // order this thread's view as well before publishing the count
    __threadfence_system();
    for (int e = 0; e < n; ++e) peer_st_release(peer_flags(d, peers[e]) + ch * d.world + d.rank, s);
}

__global__ void k_peer_wait(PeerDev d, int ch, const int32_t *peers, int n, int free_mode, const int *skip) {
    if (threadIdx.x != 0 || skip_now(skip)) return;
    const unsigned long long target = free_mode ? d.seq[PCH_HALO] : ++d.seq[PCH_COUNT + ch];
    for (int e = 0; e < n; ++e)
        if (!peer_spin(d, ch, peers[e], target)) return;
}

template <int BS>
__global__ void k_put_rows(int64_t n, const int32_t *__restrict__ rows, double *const *__restrict__ dst,
                           const double *__restrict__ x) {
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t li = rows[e];
        double *o = dst[e];
#pragma unroll
        for (int c = 0; c < BS; ++c) o[c] = x[BS * li + c];
    }
    __threadfence_system();  // before the signal kernel publishes the count
}

}  // namespace

void launch_peer_signal(const PeerDev &d, int ch, const int32_t *peers, int n, const int *skip, cudaStream_t st) {
    k_peer_signal<<<1, 32, 0, st>>>(d, ch, peers, n, skip);
}

void launch_peer_wait(const PeerDev &d, int ch, const int32_t *peers, int n, int free_mode, const int *skip,
                      cudaStream_t st) {
    k_peer_wait<<<1, 32, 0, st>>>(d, ch, peers, n, free_mode, skip);
}

void launch_put_rows(int bs, int64_t n, const int32_t *rows, double *const *dst, const double *x, cudaStream_t st) {
    if (n <= 0) return;
    const int g = (int)std::min<int64_t>(1024, (n + 255) / 256);
    if (bs == 3)
        k_put_rows<3><<<g, 256, 0, st>>>(n, rows, dst, x);
    else
        k_put_rows<1><<<g, 256, 0, st>>>(n, rows, dst, x);
}

}  // namespace ddk
