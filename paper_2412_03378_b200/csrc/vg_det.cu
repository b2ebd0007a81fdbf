// Deterministic-gradient mode: the reference's backward
// is bitwise identical across thread counts (fixed tile-order reduction,
// grad.py:188-204); the default device backward adds per-warp partial sums
// into the per-Gaussian accumulators with float atomics, whose order varies
// from run to run.  With vg_options.deterministic the backward blend instead
// stores every (list entry, warp) partial into its own slot, and a reduction
// sums each Gaussian's slots in a fixed order (its tiles row-major over its
// tile rectangle, then warps combined as (w0 + w1) + (w2 + w3)) into the
// accumulator; k_det_tiles sums the per-tile d_background / loss partials in
// tile order.  Every output is a fixed-order float sum: bitwise reproducible.
//
// Render backward (a forward visibility mask exists): slots are
// Gaussian-major -- slot 4 (off[g] + k) + w holds warp w's partial of g's
// k-th tile, and a byte per (Gaussian, tile) holds the four warp bits -- so
// k_det_reduce_g reads each Gaussian's slots as one contiguous run, with no
// dependent gathers (its fixed order: DET_LANES interleaved lanes, then a
// fixed shuffle tree); the blend's staging thread derives the index from the
// Gaussian's tile rectangle.  Tomography / splat: slots are pair-major (4 per
// list entry) and k_pair_slots maps each Gaussian's k-th tile to its list
// position for k_det_reduce.
#include "vg_kernels.cuh"

namespace vg {

constexpr int DET_WARPS = 4;    // warps per tile CTA (vg_blend.cu NT / 32)
constexpr int DET_STRIDE = 16;  // floats per (entry, warp) slot (13 used)

__global__ void k_rect_counts(int64_t n, const ushort4* __restrict__ rect, uint32_t* __restrict__ cnt) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const ushort4 r = rect[i];
  cnt[i] = r.z >= r.x ? (uint32_t)(r.z - r.x + 1) * (uint32_t)(r.w - r.y + 1) : 0u;
}

// one CTA per tile: list position p of Gaussian g in tile (tx, ty) ->
// slot[off[g] + (ty - y0) * w + (tx - x0)]
__global__ void k_pair_slots(const uint2* __restrict__ ranges, const uint32_t* __restrict__ vals,
                             const ushort4* __restrict__ rect, const uint32_t* __restrict__ off,
                             int ntx, uint32_t* __restrict__ slot) {
  const int t = blockIdx.x;
  const int ty = t / ntx, tx = t - ty * ntx;
  const uint2 r = ranges[t];
  for (uint32_t p = r.x + threadIdx.x; p < r.y; p += blockDim.x) {
    const uint32_t g = vals[p];
    const ushort4 q = rect[g];
    const uint32_t w = (uint32_t)(q.z - q.x + 1);
    slot[off[g] + (uint32_t)(ty - q.y) * w + (uint32_t)(tx - q.x)] = p;
  }
}

// Pair-major slots: four lanes per Gaussian; lane w sums warp slot w of each
// of the Gaussian's tiles in tile order, then the four partials are combined
// as (w0 + w1) + (w2 + w3).
__global__ void __launch_bounds__(256) k_det_reduce(int64_t n, const uint32_t* __restrict__ cnt,
                                                    const uint32_t* __restrict__ off,
                                                    const uint32_t* __restrict__ slot,
                                                    const float* __restrict__ part, float* __restrict__ acc) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t g = t >> 2;
  const int w = (int)(t & 3);
  const uint32_t c = g < n ? cnt[g] : 0u;
  float s[13];
#pragma unroll
  for (int q = 0; q < 13; ++q) s[q] = 0.f;
  const uint32_t o = g < n ? off[g] : 0u;
  for (uint32_t k = 0; k < c; ++k) {
    const size_t idx = (size_t)slot[o + k] * DET_WARPS + w;
    const float4* p4 = reinterpret_cast<const float4*>(part + idx * DET_STRIDE);
    const float4 a = p4[0], b = p4[1], d = p4[2], e = p4[3];
    s[0] += a.x; s[1] += a.y; s[2] += a.z; s[3] += a.w;
    s[4] += b.x; s[5] += b.y; s[6] += b.z; s[7] += b.w;
    s[8] += d.x; s[9] += d.y; s[10] += d.z; s[11] += d.w;
    s[12] += e.x;
  }
#pragma unroll
  for (int q = 0; q < 13; ++q) {
    s[q] += __shfl_xor_sync(0xffffffffu, s[q], 1);
    s[q] += __shfl_xor_sync(0xffffffffu, s[q], 2);
  }
  if (g < n && w == 0 && c) {
    float* a = acc + 16 * g;
#pragma unroll
    for (int q = 0; q < 13; ++q) a[q] += s[q];
  }
}

// Gaussian-major slots: a Gaussian's 4 c slots (c = tiles of its rectangle)
// are one contiguous run, slot 4 k + w = warp w of its k-th tile, written
// only where the forward saw warp w visible (gvis4).  Each Gaussian is summed
// by ONE group of threads in a fixed order -- lane j of the group sums, in
// increasing order, the visible slots j, j + L, j + 2L, ..., then the L
// partials are combined by a fixed tree -- so the result is bitwise
// reproducible whichever group takes it.  Small Gaussians (c <= DET_BIG):
// DET_LANES lanes (k_det_reduce_g); large ones are queued and summed by a
// whole CTA each (k_det_reduce_big), so a Gaussian covering thousands of
// tiles does not leave its warp as the kernel's tail.
#ifndef VG_DET_LANES
#define VG_DET_LANES 2  // A/B (16 views of config 3, serial, det step): 1: 41.0, 2: 40.1, 4: 40.3, 8: 40.8, 16: 42.2, 32: 46.5 ms
#endif
constexpr int DET_LANES = VG_DET_LANES;
constexpr uint32_t DET_BIG = 32;
constexpr int DET_BIG_NT = 256;

__device__ __forceinline__ void det_add_slot(const float4* p4, float (&s)[13]) {
  const float4 a = __ldg(p4), b = __ldg(p4 + 1), d = __ldg(p4 + 2), e = __ldg(p4 + 3);
  s[0] += a.x; s[1] += a.y; s[2] += a.z; s[3] += a.w;
  s[4] += b.x; s[5] += b.y; s[6] += b.z; s[7] += b.w;
  s[8] += d.x; s[9] += d.y; s[10] += d.z; s[11] += d.w;
  s[12] += e.x;
}

__global__ void __launch_bounds__(256) k_det_reduce_g(int64_t n, const uint32_t* __restrict__ cnt,
                                                      const uint32_t* __restrict__ off,
                                                      const uint8_t* __restrict__ gvis4,
                                                      const float* __restrict__ part,
                                                      float* __restrict__ acc, uint32_t* __restrict__ big,
                                                      uint32_t* __restrict__ n_big) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t g = t / DET_LANES;
  const int j = (int)(t % DET_LANES);
  uint32_t c = g < n ? cnt[g] : 0u;
  if (c > DET_BIG) {
    if (j == 0) big[atomicAdd(n_big, 1u)] = (uint32_t)g;  // summed by k_det_reduce_big
    c = 0;
  }
  float s[13];
#pragma unroll
  for (int q = 0; q < 13; ++q) s[q] = 0.f;
  const uint32_t o = g < n ? off[g] : 0u;
  const float4* base = reinterpret_cast<const float4*>(part + (size_t)o * DET_WARPS * DET_STRIDE);
  // the visibility bytes of 16 consecutive slots of this lane are loaded at
  // once (independent loads) into a bit mask, then only the visible slots are
  // read, in increasing order (85 % of the slots are invisible: a serial
  // byte test per slot made the loop one L1/L2 latency per slot)
  const uint32_t ns = DET_WARPS * c;
  for (uint32_t i0 = 0; (uint32_t)j + DET_LANES * i0 < ns; i0 += 16) {
    uint32_t m = 0;
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const uint32_t sl = (uint32_t)j + DET_LANES * (i0 + u);
      if (sl < ns) m |= ((__ldg(gvis4 + o + sl / DET_WARPS) >> (sl % DET_WARPS)) & 1u) << u;
    }
    while (m) {
      const int u = __ffs(m) - 1;
      m &= m - 1;
      det_add_slot(base + (size_t)((uint32_t)j + DET_LANES * (i0 + u)) * (DET_STRIDE / 4), s);
    }
  }
#pragma unroll
  for (int q = 0; q < 13; ++q) {
#pragma unroll
    for (int mk = DET_LANES / 2; mk >= 1; mk >>= 1) s[q] += __shfl_xor_sync(0xffffffffu, s[q], mk);
  }
  if (g < n && j == 0 && c) {
    float* a = acc + 16 * g;
#pragma unroll
    for (int q = 0; q < 13; ++q) a[q] += s[q];
  }
}

// One CTA per queued large Gaussian (grid-stride over the queue): thread j
// sums the visible slots j, j + 256, ... in order, then a fixed shared-memory
// tree (warp xor-shuffles, then warps 0..7 in order).
__global__ void __launch_bounds__(DET_BIG_NT) k_det_reduce_big(const uint32_t* __restrict__ cnt,
                                                               const uint32_t* __restrict__ off,
                                                               const uint8_t* __restrict__ gvis4,
                                                               const float* __restrict__ part,
                                                               float* __restrict__ acc,
                                                               const uint32_t* __restrict__ big,
                                                               const uint32_t* __restrict__ n_big) {
  __shared__ float red[DET_BIG_NT / 32][13];
  const uint32_t nb = *n_big;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint32_t b = blockIdx.x; b < nb; b += gridDim.x) {
    const uint32_t g = big[b];
    const uint32_t c = cnt[g], o = off[g];
    const float4* base = reinterpret_cast<const float4*>(part + (size_t)o * DET_WARPS * DET_STRIDE);
    float s[13];
#pragma unroll
    for (int q = 0; q < 13; ++q) s[q] = 0.f;
    for (uint32_t sl = threadIdx.x; sl < DET_WARPS * c; sl += DET_BIG_NT)
      if ((__ldg(gvis4 + o + sl / DET_WARPS) >> (sl % DET_WARPS)) & 1u)
        det_add_slot(base + (size_t)sl * (DET_STRIDE / 4), s);
#pragma unroll
    for (int q = 0; q < 13; ++q) {
#pragma unroll
      for (int m = 16; m >= 1; m >>= 1) s[q] += __shfl_xor_sync(0xffffffffu, s[q], m);
    }
    if (lane == 0)
      for (int q = 0; q < 13; ++q) red[warp][q] = s[q];
    __syncthreads();
    if (threadIdx.x < 13) {
      float v = 0.f;
      for (int w = 0; w < DET_BIG_NT / 32; ++w) v += red[w][threadIdx.x];
      acc[16 * (size_t)g + threadIdx.x] += v;
    }
    __syncthreads();
  }
}

// Fixed-order sum of the per-tile d_background (3 floats) and loss (double)
// partials: thread i sums tiles i, i + 256, ... in order, then thread 0 the
// 256 thread sums in order.
__global__ void __launch_bounds__(256) k_det_tiles(int n_tiles, const float* __restrict__ bg,
                                                   const double* __restrict__ loss,
                                                   float* __restrict__ d_background,
                                                   double* __restrict__ loss_sum) {
  __shared__ float sb[256][3];
  __shared__ double sl[256];
  float b0 = 0.f, b1 = 0.f, b2 = 0.f;
  double l = 0.0;
  for (int t = threadIdx.x; t < n_tiles; t += 256) {
    b0 += bg[3 * t]; b1 += bg[3 * t + 1]; b2 += bg[3 * t + 2];
    if (loss) l += loss[t];
  }
  sb[threadIdx.x][0] = b0; sb[threadIdx.x][1] = b1; sb[threadIdx.x][2] = b2;
  sl[threadIdx.x] = l;
  __syncthreads();
  if (threadIdx.x == 0) {
    float s0 = 0.f, s1 = 0.f, s2 = 0.f;
    double sll = 0.0;
    for (int i = 0; i < 256; ++i) { s0 += sb[i][0]; s1 += sb[i][1]; s2 += sb[i][2]; sll += sl[i]; }
    if (d_background) { d_background[0] += s0; d_background[1] += s1; d_background[2] += s2; }
    if (loss_sum && loss) *loss_sum += sll;
  }
}

// out += the deferred sums (when out is given); the sums are cleared
__global__ void k_det_flush(float* __restrict__ bg, double* __restrict__ loss, float* __restrict__ bg_out,
                            double* __restrict__ loss_out) {
  if (threadIdx.x != 0) return;
  if (bg_out) { bg_out[0] += bg[0]; bg_out[1] += bg[1]; bg_out[2] += bg[2]; }
  if (loss_out) *loss_out += *loss;
  bg[0] = bg[1] = bg[2] = 0.f;
  *loss = 0.0;
}

void launch_det_flush(float* bg, double* loss, float* bg_out, double* loss_out, cudaStream_t st) {
  k_det_flush<<<1, 32, 0, st>>>(bg, loss, bg_out, loss_out);
}

size_t det_part_bytes(int64_t pairs) {
  return sizeof(float) * (size_t)pairs * DET_WARPS * DET_STRIDE;
}

cudaError_t det_prepare(int64_t n, const ushort4* rect, const uint2* ranges, const uint32_t* vals,
                        int n_tiles, int ntx, uint32_t* cnt, uint32_t* off, uint32_t* slot,
                        void* scan_scratch, uint32_t* total, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  k_rect_counts<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, rect, cnt);
  cudaError_t e = scan_u32(cnt, off, scan_scratch, total, n, st);
  if (e != cudaSuccess) return e;
  if (slot) k_pair_slots<<<n_tiles, 128, 0, st>>>(ranges, vals, rect, off, ntx, slot);
  return cudaGetLastError();
}

cudaError_t det_reduce(int64_t n, const uint32_t* cnt, const uint32_t* off, const uint32_t* slot,
                       const float* part, float* acc, int n_tiles, const float* bg_part,
                       const double* loss_part, float* d_background, double* loss_sum,
                       cudaStream_t st, const uint8_t* gvis4, uint32_t* big_scratch) {
  const unsigned blocks = (unsigned)((4 * n + 255) / 256);
  if (n > 0 && gvis4) {
    // queue of large Gaussians: n entries after the counter in big_scratch
    uint32_t* n_big = big_scratch;
    uint32_t* big = big_scratch + 1;
    cudaMemsetAsync(n_big, 0, sizeof(uint32_t), st);
    k_det_reduce_g<<<(unsigned)((DET_LANES * n + 255) / 256), 256, 0, st>>>(n, cnt, off, gvis4, part, acc,
                                                                          big, n_big);
    k_det_reduce_big<<<4 * 148, DET_BIG_NT, 0, st>>>(cnt, off, gvis4, part, acc, big, n_big);
  }
  else if (n > 0 && slot)
    k_det_reduce<<<blocks, 256, 0, st>>>(n, cnt, off, slot, part, acc);
  k_det_tiles<<<1, 256, 0, st>>>(n_tiles, bg_part, loss_part, d_background, loss_sum);
  return cudaGetLastError();
}

}  // namespace vg
