// Binning helpers: the identity permutation the depth sort starts from.
// (The per-tile lists themselves are built by the span binning, vg_span.cu.)
#include "vg_kernels.cuh"

namespace vg {

__global__ void k_iota(int64_t n, uint32_t* ids) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) ids[i] = (uint32_t)i;
}

void launch_iota(int64_t n, uint32_t* ids, cudaStream_t st) {
  if (n > 0) k_iota<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, ids);
}

}  // namespace vg
