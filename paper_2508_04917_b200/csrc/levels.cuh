// levels.cuh -- device Alg. 5 level assignment (product-internal).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace ddk {
void launch_levels(int nsl, const int64_t *sub, const int64_t *rp, const int32_t *ci, int32_t *hmap, int max_p,
                   cudaStream_t st);
}
