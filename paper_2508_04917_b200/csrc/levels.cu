// levels.cu -- Alg. 5 on the device: per-subdomain parallel
// level assignment by fixpoint marking, one CTA per subdomain (sec. 8(f2)).
//
// Iteration `lev`: every unmarked row all of whose dependencies were marked
// in EARLIER iterations gets hmap = lev. A dependency marked in the current
// iteration reads as -1 or lev and never satisfies "0 <= hmap[j] < lev", so
// the concurrent writes need no extra barrier. The loop ends when an
// iteration adds nothing (the paper's `added` flag). The result is the
// longest-path level of every row (R16), i.e. equal to the host's.
#include <cuda_runtime.h>

#include <cstdint>

#include "levels.cuh"

namespace ddk {

// dir = 0: lower (deps = strictly-lower blocks); 1: upper (strictly upper).
// rp/ci are the rank-local factor patterns (Lrp/Lci or Urp/Uci); sub[s] and
// sub[s+1] bound subdomain s's rank-local rows; hmap is rank-local.
__global__ void __launch_bounds__(256) k_levels(const int64_t *__restrict__ sub, const int64_t *__restrict__ rp,
                                                const int32_t *__restrict__ ci, int32_t *__restrict__ hmap) {
    extern __shared__ int32_t h[];
    __shared__ int added;
    const int64_t a = sub[blockIdx.x], e = sub[blockIdx.x + 1];
    const int P = (int)(e - a);
    for (int i = threadIdx.x; i < P; i += blockDim.x) h[i] = -1;
    __syncthreads();
    for (int lev = 0;; ++lev) {
        if (threadIdx.x == 0) added = 0;
        __syncthreads();
        int mine = 0;
        for (int i = threadIdx.x; i < P; i += blockDim.x) {
            if (h[i] >= 0) continue;
            bool ready = true;
            for (int64_t q = rp[a + i]; q < rp[a + i + 1] && ready; ++q) {
                const int hj = *reinterpret_cast<volatile int32_t *>(&h[ci[q] - a]);
                ready = hj >= 0 && hj < lev;
            }
            if (ready) {
                h[i] = lev;
                mine = 1;
            }
        }
        if (mine) added = 1;
        __syncthreads();
        if (!added) break;
        __syncthreads();
    }
    for (int i = threadIdx.x; i < P; i += blockDim.x) hmap[a + i] = h[i];
}

void launch_levels(int nsl, const int64_t *sub, const int64_t *rp, const int32_t *ci, int32_t *hmap, int max_p,
                   cudaStream_t st) {
    cudaFuncSetAttribute(k_levels, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * max_p);
    k_levels<<<nsl, 256, 4 * max_p, st>>>(sub, rp, ci, hmap);
}

}  // namespace ddk
