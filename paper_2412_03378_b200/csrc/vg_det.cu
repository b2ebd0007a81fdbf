// Deterministic-gradient mode: the reference's backward
// is bitwise identical across thread counts (fixed tile-order reduction,
// grad.py:188-204); the default device backward adds per-warp partial sums
// into the per-Gaussian accumulators with float atomics, whose order varies
// from run to run.  With vg_options.deterministic the backward blend instead
// stores every (list entry, warp) partial into its own slot, and
//   k_pair_slots  maps each Gaussian's k-th tile (row-major over its tile
//                 rectangle) to its list position in that tile,
//   k_det_reduce  sums, per Gaussian, its slots in that fixed order (tiles
//                 row-major, then warps 0..3) into the accumulator,
//   k_det_tiles   sums the per-tile d_background / loss partials in tile
//                 order,
// so every output is a fixed-order float sum: bitwise reproducible.
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

// Four lanes per Gaussian: lane w sums warp slot w of each of the Gaussian's
// tiles in tile order, then the four partials are combined as
// (w0 + w1) + (w2 + w3) -- a fixed order.  COMPACT: only the (entry, warp)
// pairs set in the forward's visibility mask have slots, numbered pair-major
// (the others contributed nothing).
template <bool COMPACT>
__global__ void __launch_bounds__(256) k_det_reduce(int64_t n, const uint32_t* __restrict__ cnt,
                                                    const uint32_t* __restrict__ off,
                                                    const uint32_t* __restrict__ slot,
                                                    const float* __restrict__ part, float* __restrict__ acc,
                                                    const uint32_t* __restrict__ pbase,
                                                    const uint8_t* __restrict__ vis4) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t g = t >> 2;
  const int w = (int)(t & 3);
  const uint32_t c = g < n ? cnt[g] : 0u;
  float s[13];
#pragma unroll
  for (int q = 0; q < 13; ++q) s[q] = 0.f;
  const uint32_t o = g < n ? off[g] : 0u;
  for (uint32_t k = 0; k < c; ++k) {
    const uint32_t p = slot[o + k];
    size_t idx;
    if (COMPACT) {
      const uint32_t v = vis4[p];
      if (!((v >> w) & 1u)) continue;
      idx = pbase[p] + __popc(v & ((1u << w) - 1u));
    } else {
      idx = (size_t)p * DET_WARPS + w;
    }
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

__global__ void k_pair_vis(int64_t pairs, const uint32_t* __restrict__ vm, int vm_words,
                           uint8_t* __restrict__ vis4, uint32_t* __restrict__ cnt) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= pairs) return;
  const size_t wi = (size_t)(p >> 5);
  const uint32_t sh = (uint32_t)(p & 31);
  uint32_t v = 0;
#pragma unroll
  for (int w = 0; w < DET_WARPS; ++w) v |= ((vm[(size_t)w * vm_words + wi] >> sh) & 1u) << w;
  vis4[p] = (uint8_t)v;
  cnt[p] = __popc(v);
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

size_t det_pairs_scratch_bytes(int64_t pairs) { return scan_u32_scratch_bytes(pairs) + 16; }

cudaError_t det_pairs(const uint32_t* vm, int vm_words, int64_t pairs, uint8_t* vis4, uint32_t* cnt_tmp,
                      uint32_t* pbase, void* scratch, cudaStream_t st) {
  k_pair_vis<<<(unsigned)((pairs + 255) / 256), 256, 0, st>>>(pairs, vm, vm_words, vis4, cnt_tmp);
  return scan_u32(cnt_tmp, pbase, scratch, pbase + pairs, pairs, st);
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
  k_pair_slots<<<n_tiles, 128, 0, st>>>(ranges, vals, rect, off, ntx, slot);
  return cudaGetLastError();
}

cudaError_t det_reduce(int64_t n, const uint32_t* cnt, const uint32_t* off, const uint32_t* slot,
                       const float* part, float* acc, int n_tiles, const float* bg_part,
                       const double* loss_part, float* d_background, double* loss_sum,
                       cudaStream_t st, const uint32_t* pbase, const uint8_t* vis4) {
  const unsigned blocks = (unsigned)((4 * n + 255) / 256);
  if (n > 0 && pbase)
    k_det_reduce<true><<<blocks, 256, 0, st>>>(n, cnt, off, slot, part, acc, pbase, vis4);
  else if (n > 0)
    k_det_reduce<false><<<blocks, 256, 0, st>>>(n, cnt, off, slot, part, acc, nullptr, nullptr);
  k_det_tiles<<<1, 256, 0, st>>>(n_tiles, bg_part, loss_part, d_background, loss_sum);
  return cudaGetLastError();
}

}  // namespace vg
