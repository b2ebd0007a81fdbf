// Depth sort of the Gaussians by float32 view depth with CUB's onesweep
// device radix sort (library; the hand-written onesweep of vg_radix.cu is
// selectable with VG_RADIX=1).  Positive floats sort as their bit patterns;
// the values start as the identity so equal depths keep index order.
#include <cub/device/device_radix_sort.cuh>

#include "vg_kernels.cuh"

namespace vg {

cudaError_t depth_sort_temp_bytes(int64_t n, size_t* bytes) {
  return cub::DeviceRadixSort::SortPairs(nullptr, *bytes, (const uint32_t*)nullptr,
                                         (uint32_t*)nullptr, (const uint32_t*)nullptr,
                                         (uint32_t*)nullptr, (int)n);
}
cudaError_t depth_sort(void* tmp, size_t tmp_bytes, const uint32_t* keys_in, uint32_t* keys_out,
                       const uint32_t* ids_in, uint32_t* ids_out, int64_t n, cudaStream_t st) {
  return cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys_in, keys_out, ids_in, ids_out,
                                         (int)n, 0, 32, st);
}

}  // namespace vg
