// K2 duplicate + K4 tile ranges (raster._build_grid, raster.py:222-260).
//
// The Gaussians are first sorted by float32 view depth (IEEE bits of a
// positive float sort as unsigned; the sort is stable over the identity
// permutation, so equal depths keep index order).  Pairs are then emitted in
// that order, each Gaussian's tiles row-major over its rectangle, with the
// tile id as key; a stable sort by tile alone yields the reference's
// lexsort((prim, depth, tile)) order with float32 depth keys.
#include "vg_kernels.cuh"

namespace vg {

__global__ void k_total(int64_t n, const uint32_t* count, const uint32_t* offset, uint64_t* total) {
  total[0] = n > 0 ? (uint64_t)offset[n - 1] + count[n - 1] : 0;
}

// --- depth-presorted binning: Gaussians are first sorted by float32 depth,
// pairs are emitted in that order with 16-bit tile keys, and a stable sort by
// tile alone then yields (tile, depth, index) order.

__global__ void k_iota(int64_t n, uint32_t* ids) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) ids[i] = (uint32_t)i;
}

__global__ void k_gather_counts(int64_t n, const uint32_t* __restrict__ perm,
                                const uint32_t* __restrict__ count, uint32_t* __restrict__ out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = count[perm[i]];
}

// One thread per Gaussian in depth order writes its pairs; rectangles of more
// than 8 tiles are written by the whole warp (coalesced, load-balanced).
template <typename KeyT>
__global__ void __launch_bounds__(256) k_duplicate_sorted(int64_t n, const uint32_t* __restrict__ perm,
                                                          const uint32_t* __restrict__ offset,
                                                          const uint32_t* __restrict__ count_sorted,
                                                          const int4* __restrict__ rect, int ntx,
                                                          KeyT* __restrict__ keys,
                                                          uint32_t* __restrict__ vals) {
  const unsigned FULLM = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t cnt = i < n ? count_sorted[i] : 0u;
  uint32_t g = 0, o = 0;
  int4 r = make_int4(0, 0, -1, -1);
  if (cnt) {
    g = perm[i];
    o = offset[i];
    r = rect[g];
  }
  if (cnt && cnt <= 8) {
    for (int y = r.y; y <= r.w; ++y)
      for (int x = r.x; x <= r.z; ++x) {
        keys[o] = (KeyT)(y * ntx + x);
        vals[o] = g;
        ++o;
      }
  }
  unsigned big = __ballot_sync(FULLM, cnt > 8);
  while (big) {
    const int src = __ffs(big) - 1;
    big &= big - 1;
    const uint32_t bc = __shfl_sync(FULLM, cnt, src), bo = __shfl_sync(FULLM, o, src);
    const uint32_t bg = __shfl_sync(FULLM, g, src);
    const int x0 = __shfl_sync(FULLM, r.x, src), y0 = __shfl_sync(FULLM, r.y, src);
    const int w = __shfl_sync(FULLM, r.z, src) - x0 + 1;
    const float inv_w = 1.0f / (float)w;
    for (uint32_t idx = lane; idx < bc; idx += 32) {
      // floor((idx + 0.5) / w) is exact in float for idx < 2^21
      const int dy = (int)((float)idx * inv_w + 0.5f * inv_w);
      const int dx = (int)idx - dy * w;
      keys[bo + idx] = (KeyT)((y0 + dy) * ntx + x0 + dx);
      vals[bo + idx] = bg;
    }
  }
}

template <typename KeyT>
__global__ void __launch_bounds__(256) k_tile_ranges(int64_t P, const KeyT* __restrict__ keys,
                                                     uint2* __restrict__ ranges) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P) return;
  uint32_t t = keys[i];
  if (i == 0 || keys[i - 1] != t) ranges[t].x = (uint32_t)i;
  if (i == P - 1 || keys[i + 1] != t) ranges[t].y = (uint32_t)(i + 1);
}

void launch_iota(int64_t n, uint32_t* ids, cudaStream_t st) {
  if (n > 0) k_iota<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, ids);
}
void launch_gather_counts(int64_t n, const uint32_t* perm, const uint32_t* count, uint32_t* out,
                          cudaStream_t st) {
  if (n > 0) k_gather_counts<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, perm, count, out);
}
void launch_duplicate_sorted(int64_t n, const uint32_t* perm, const uint32_t* offset,
                             const uint32_t* count_sorted, const int4* rect, int ntx, void* keys,
                             bool wide, uint32_t* vals, cudaStream_t st) {
  if (n <= 0) return;
  const unsigned g = (unsigned)((n + 255) / 256);
  if (wide)
    k_duplicate_sorted<uint32_t><<<g, 256, 0, st>>>(n, perm, offset, count_sorted, rect, ntx,
                                                    (uint32_t*)keys, vals);
  else
    k_duplicate_sorted<uint16_t><<<g, 256, 0, st>>>(n, perm, offset, count_sorted, rect, ntx,
                                                    (uint16_t*)keys, vals);
}
void launch_tile_ranges(int64_t P, const void* keys, bool wide, uint2* ranges, cudaStream_t st) {
  if (P <= 0) return;
  const unsigned g = (unsigned)((P + 255) / 256);
  if (wide) k_tile_ranges<uint32_t><<<g, 256, 0, st>>>(P, (const uint32_t*)keys, ranges);
  else k_tile_ranges<uint16_t><<<g, 256, 0, st>>>(P, (const uint16_t*)keys, ranges);
}

void launch_total(int64_t n, const uint32_t* count, const uint32_t* offset, uint64_t* total,
                  cudaStream_t st) {
  k_total<<<1, 1, 0, st>>>(n, count, offset, total);
}

}  // namespace vg
