// K3 radix sorts + the count scan.  Round 1 uses CUB's onesweep device radix
// sort / scan (library, like cuBLAS for a GEMM): the 32-bit depth sort of the
// Gaussians, the 16/32-bit stable tile sort of the pairs, and the tiny
// heavy-tiles-first order sort.  See DESIGN.md for the planned hand-written
// replacement.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "vg_kernels.cuh"

namespace vg {

cudaError_t scan_temp_bytes(int64_t n, size_t* bytes) {
  return cub::DeviceScan::ExclusiveSum(nullptr, *bytes, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                       (int)n);
}

cudaError_t exclusive_scan(void* tmp, size_t tmp_bytes, const uint32_t* in, uint32_t* out,
                           int64_t n, cudaStream_t st) {
  return cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, in, out, (int)n, st);
}

int sort_launches(int end_bit) { return 1 + (end_bit + 7) / 8; }

// Gaussians by float32 view depth (positive floats sort as their bit
// patterns); values start as the identity so equal depths keep index order.
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

// Stable sort of the depth-ordered pairs by their tile id: 16-bit keys up to
// 65536 tiles (two 8-bit passes at 1080p), 32-bit keys beyond (e.g. 8K).
template <typename K>
static cudaError_t tile_sort_t(void* tmp, size_t* tmp_bytes, K* k0, K* k1, uint32_t* v0,
                               uint32_t* v1, int64_t n, int end_bit, int* which, cudaStream_t st) {
  cub::DoubleBuffer<K> k(k0, k1);
  cub::DoubleBuffer<uint32_t> v(v0, v1);
  cudaError_t e = cub::DeviceRadixSort::SortPairs(tmp, *tmp_bytes, k, v, (int)n, 0, end_bit, st);
  if (which) *which = k.selector;
  return e;
}
cudaError_t tile_sort_temp_bytes(int64_t n, int end_bit, bool wide, size_t* bytes) {
  if (wide)
    return tile_sort_t<uint32_t>(nullptr, bytes, nullptr, nullptr, nullptr, nullptr, n, end_bit,
                                 nullptr, 0);
  return tile_sort_t<uint16_t>(nullptr, bytes, nullptr, nullptr, nullptr, nullptr, n, end_bit,
                               nullptr, 0);
}
cudaError_t tile_sort(void* tmp, size_t tmp_bytes, void* k0, void* k1, uint32_t* v0, uint32_t* v1,
                      int64_t n, int end_bit, bool wide, int* which, cudaStream_t st) {
  if (wide)
    return tile_sort_t<uint32_t>(tmp, &tmp_bytes, (uint32_t*)k0, (uint32_t*)k1, v0, v1, n,
                                 end_bit, which, st);
  return tile_sort_t<uint16_t>(tmp, &tmp_bytes, (uint16_t*)k0, (uint16_t*)k1, v0, v1, n, end_bit,
                               which, st);
}

// Heavy-tiles-first launch order: tiles sorted by descending list length, so
// the longest tiles start in the first wave (longest-processing-time first).
__global__ void k_tile_len(const uint2* ranges, uint32_t* len, uint32_t* ids, int n) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) {
    uint2 r = ranges[t];
    len[t] = r.y - r.x;
    ids[t] = (uint32_t)t;
  }
}

cudaError_t tile_order_temp_bytes(int n_tiles, size_t* bytes) {
  return cub::DeviceRadixSort::SortPairsDescending(nullptr, *bytes, (const uint32_t*)nullptr,
                                                   (uint32_t*)nullptr, (const uint32_t*)nullptr,
                                                   (uint32_t*)nullptr, n_tiles);
}

cudaError_t tile_order(void* tmp, size_t tmp_bytes, const uint2* ranges, uint32_t* len_in,
                       uint32_t* len_out, uint32_t* ids_in, uint32_t* ids_out, int n_tiles,
                       cudaStream_t st) {
  k_tile_len<<<(n_tiles + 255) / 256, 256, 0, st>>>(ranges, len_in, ids_in, n_tiles);
  return cub::DeviceRadixSort::SortPairsDescending(tmp, tmp_bytes, len_in, len_out, ids_in,
                                                   ids_out, n_tiles, 0, 32, st);
}

}  // namespace vg
