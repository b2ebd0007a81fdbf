// Shared device helpers of the tile kernels (vg_blend.cu: analytic render
// and tomography; vg_splat.cu: the EWA comparator): packed FP32x2
// arithmetic, lane geometry, warp reductions and gradient flushes, and the
// per-pixel backward prologue.
#pragma once

#include "vg_kernels.cuh"

namespace vg {

constexpr unsigned FULL = 0xffffffffu;
constexpr float C_HALF_LOG2E = 0.72134752044448170f;  // 0.5 * log2(e)
constexpr int ACC_STRIDE = 16;                         // floats per Gaussian accumulator
constexpr int NT = 128;                                // threads per tile CTA
#ifndef VG_BATCH
#define VG_BATCH 256
#endif
constexpr int BATCH = VG_BATCH;                        // staged records per batch

// ---------------------------------------------------------------------------
// packed FP32x2 helpers (sm_100a FFMA2 / FMUL2 / FADD2)

struct F2 {
  unsigned long long v;
};
__device__ __forceinline__ F2 f2(float a, float b) {
  F2 r;
  asm("mov.b64 %0, {%1,%2};" : "=l"(r.v) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ F2 f2s(float a) { return f2(a, a); }
__device__ __forceinline__ float lo(F2 x) { return __uint_as_float((unsigned)(x.v & 0xffffffffull)); }
__device__ __forceinline__ float hi(F2 x) { return __uint_as_float((unsigned)(x.v >> 32)); }
__device__ __forceinline__ F2 fma2(F2 a, F2 b, F2 c) {
  F2 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d.v) : "l"(a.v), "l"(b.v), "l"(c.v));
  return d;
}
__device__ __forceinline__ F2 mul2(F2 a, F2 b) {
  F2 d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d.v) : "l"(a.v), "l"(b.v));
  return d;
}
__device__ __forceinline__ F2 add2(F2 a, F2 b) {
  F2 d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d.v) : "l"(a.v), "l"(b.v));
  return d;
}
__device__ __forceinline__ F2 sub2(F2 a, F2 b) {
  F2 d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d.v) : "l"(a.v), "l"(b.v));
  return d;
}
__device__ __forceinline__ F2 ex2_2(F2 x) { return f2(ex2f(lo(x)), ex2f(hi(x))); }
__device__ __forceinline__ F2 rsq_2(F2 x) { return f2(rsqf(lo(x)), rsqf(hi(x))); }
__device__ __forceinline__ F2 neg2(F2 x) { return f2(-lo(x), -hi(x)); }
__device__ __forceinline__ F2 sel2(bool p0, bool p1, F2 a, F2 b) {
  return f2(p0 ? lo(a) : lo(b), p1 ? hi(a) : hi(b));
}
__device__ __forceinline__ float hsum(F2 x) { return lo(x) + hi(x); }

// ---------------------------------------------------------------------------
// staging + culling

__device__ __forceinline__ float d0(float lo_, float hi_) {
  // distance of the interval [lo_, hi_] from 0
  return fmaxf(fmaxf(lo_, -hi_), 0.f);
}

// Lane geometry: warp w owns the 8x8 block (8(w&1), 8(w>>1)); lane l owns
// column 8(w&1) + (l&7) and rows 8(w>>1) + (l>>3) and +4.
struct LaneGeo {
  int lxi, ly0, col, row0, row1;
  bool in0, in1;
};
__device__ __forceinline__ LaneGeo lane_geo(const BlendParams& p, int tx, int ty) {
  LaneGeo g;
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  g.lxi = 8 * (w & 1) + (l & 7);
  g.ly0 = 8 * (w >> 1) + (l >> 3);
  g.col = tx * TILE + g.lxi;
  g.row0 = ty * TILE + g.ly0;
  g.row1 = g.row0 + 4;
  g.in0 = g.col < p.width && g.row0 < p.height;
  g.in1 = g.col < p.width && g.row1 < p.height;
  return g;
}

// Reduce 16 per-lane values over the warp; lane l ends with the warp total of
// value index ((l>>4&1)*8 + (l>>3&1)*4 + (l>>2&1)*2 + (l>>1&1)).
__device__ __forceinline__ float transpose_reduce16(float (&v)[16], int lane) {
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    bool h = lane & 16;
    float send = h ? v[i] : v[i + 8];
    float keep = h ? v[i + 8] : v[i];
    v[i] = keep + __shfl_xor_sync(FULL, send, 16);
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    bool h = lane & 8;
    float send = h ? v[i] : v[i + 4];
    float keep = h ? v[i + 4] : v[i];
    v[i] = keep + __shfl_xor_sync(FULL, send, 8);
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    bool h = lane & 4;
    float send = h ? v[i] : v[i + 2];
    float keep = h ? v[i + 2] : v[i];
    v[i] = keep + __shfl_xor_sync(FULL, send, 4);
  }
  {
    bool h = lane & 2;
    float send = h ? v[0] : v[1];
    float keep = h ? v[1] : v[0];
    v[0] = keep + __shfl_xor_sync(FULL, send, 2);
  }
  return v[0] + __shfl_xor_sync(FULL, v[0], 1);
}

__device__ __forceinline__ void flush_acc(float (&v)[16], int lane, uint32_t gid, float* acc) {
  float s = transpose_reduce16(v, lane);
  int idx = ((lane >> 4) & 1) * 8 + ((lane >> 3) & 1) * 4 + ((lane >> 2) & 1) * 2 + ((lane >> 1) & 1);
  if (!(lane & 1) && idx < 13 && s != 0.f) atomicAdd(acc + (size_t)gid * ACC_STRIDE + idx, s);
}

// Warp sum of 13 per-lane values through shared memory (wb: RED_WORDS floats
// per warp, 16-byte aligned): each lane stores its 13 values as column `lane`
// of a 13 x 36 array (conflict-free), lanes 2q and 2q+1 each sum one half
// row of value q with four 128-bit loads (the 4-float row padding spreads
// the eight rows a quarter-warp reads over all 32 banks) and packed adds,
// and one shuffle joins the halves: lane 2q (q < 13) returns the sum of
// value q.  About 30 instructions against the 62 of transpose_reduce16.
constexpr int RED_ROW = 36;
constexpr int RED_WORDS = 13 * RED_ROW;
__device__ __forceinline__ float smem_reduce13(const float (&v)[16], int lane, float* wb) {
#pragma unroll
  for (int q = 0; q < 13; ++q) wb[q * RED_ROW + lane] = v[q];
  __syncwarp();
  float s = 0.f;
  if (lane < 26) {
    const float4* src = reinterpret_cast<const float4*>(wb + (lane >> 1) * RED_ROW + (lane & 1) * 16);
    const float4 x0 = src[0], x1 = src[1], x2 = src[2], x3 = src[3];
    const F2 a = add2(add2(f2(x0.x, x0.y), f2(x1.x, x1.y)), add2(f2(x2.x, x2.y), f2(x3.x, x3.y)));
    const F2 b = add2(add2(f2(x0.z, x0.w), f2(x1.z, x1.w)), add2(f2(x2.z, x2.w), f2(x3.z, x3.w)));
    s = hsum(add2(a, b));
  }
  s += __shfl_xor_sync(FULL, s, 1);
  __syncwarp();  // the buffer is rewritten by the warp's next entry
  return s;
}

// Packed variant for two entries: value q of both entries is stored as one
// 8-byte pair per lane in row q (68 floats: 64 data + 4 pad, so that the 8
// rows a quarter-warp reads start in distinct bank groups); lanes 0..12 sum
// the lower half row of q = lane, lanes 16..28 the upper half of q = lane-16,
// both entries at once in packed FP32x2 adds, and one exchange joins the
// halves: lane q (< 13) returns (sum_a[q], sum_b[q]).  13 STS.64 instead of
// 26 STS.32.
constexpr int REDP_ROW = 68;
constexpr int REDP_WORDS = 13 * REDP_ROW;
__device__ __forceinline__ F2 smem_reduce13x2p(const float (&va)[16], const float (&vb)[16], int lane,
                                               float* wb) {
#pragma unroll
  for (int q = 0; q < 13; ++q)
    *reinterpret_cast<unsigned long long*>(wb + q * REDP_ROW + 2 * lane) = f2(va[q], vb[q]).v;
  __syncwarp();
  F2 acc = f2s(0.f);
  const int q = lane & 15;
  if (q < 13) {
    const float4* src = reinterpret_cast<const float4*>(wb + q * REDP_ROW + (lane & 16) * 2);
    F2 t[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float4 x = src[k];
      t[k] = add2(f2(x.x, x.y), f2(x.z, x.w));
    }
    acc = add2(add2(add2(t[0], t[1]), add2(t[2], t[3])), add2(add2(t[4], t[5]), add2(t[6], t[7])));
  }
  F2 o;
  o.v = __shfl_xor_sync(FULL, acc.v, 16);
  __syncwarp();
  return add2(acc, o);
}

__device__ __forceinline__ void flush_acc_smem(const float (&v)[16], int lane, uint32_t gid, float* acc,
                                               float* wb) {
  const float s = smem_reduce13(v, lane, wb);
  if (!(lane & 1) && lane < 26) atomicAdd(acc + (size_t)gid * ACC_STRIDE + (lane >> 1), s);
}

__device__ __forceinline__ void flush_det_smem(const float (&v)[16], int lane, float* slot, float* wb) {
  const float s = smem_reduce13(v, lane, wb);
  // all 16 floats of the slot (3 zero pads): whole sectors
  if (!(lane & 1)) slot[lane >> 1] = lane < 26 ? s : 0.f;
}

// Deterministic mode: the warp's 13 sums go to the (entry, warp) slot (no
// atomics); vg_det.cu reduces the slots per Gaussian in a fixed order.
__device__ __forceinline__ void flush_det(float (&v)[16], int lane, float* slot) {
  float s = transpose_reduce16(v, lane);
  int idx = ((lane >> 4) & 1) * 8 + ((lane >> 3) & 1) * 4 + ((lane >> 2) & 1) * 2 + ((lane >> 1) & 1);
  if (!(lane & 1) && idx < 13) slot[idx] = s;
}

// Block sum of 3 floats + 1 double into global (d_background, loss).
__device__ __forceinline__ void block_flush(float a0, float a1, float a2, double l, float* out3,
                                            double* outl, bool store = false) {
  __shared__ float r3[NT / 32][3];
  __shared__ double rl[NT / 32];
  for (int o = 16; o; o >>= 1) {
    a0 += __shfl_xor_sync(FULL, a0, o);
    a1 += __shfl_xor_sync(FULL, a1, o);
    a2 += __shfl_xor_sync(FULL, a2, o);
    l += __shfl_xor_sync(FULL, l, o);
  }
  int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) { r3[w][0] = a0; r3[w][1] = a1; r3[w][2] = a2; rl[w] = l; }
  __syncthreads();
  if (threadIdx.x == 0) {
    float s0 = 0, s1 = 0, s2 = 0;
    double sl = 0;
    for (int i = 0; i < NT / 32; ++i) { s0 += r3[i][0]; s1 += r3[i][1]; s2 += r3[i][2]; sl += rl[i]; }
    if (store) {  // deterministic mode: this tile's partial, reduced in tile order later
      if (out3) { out3[0] = s0; out3[1] = s1; out3[2] = s2; }
      if (outl) *outl = sl;
    } else {
      if (out3) {
        if (s0 != 0.f) atomicAdd(out3 + 0, s0);
        if (s1 != 0.f) atomicAdd(out3 + 1, s1);
        if (s2 != 0.f) atomicAdd(out3 + 2, s2);
      }
      if (outl && sl != 0.0) atomicAdd(outl, sl);
    }
  }
}

// Per-pixel prologue of the backward: upstream gradient (explicit or fused
// L2), total = dc . color + dT T_final, n_act; d_background and loss sums.
template <int LOSS, bool DET>
__device__ __forceinline__ void bwd_prologue(const BlendParams& p, const LaneGeo& G, const BwdIO& io,
                                             float (&dcv)[2][3], float (&totv)[2], int tile,
                                             bool sums = true) {
  float Tfv[2] = {1.f, 1.f};
  double lossv = 0.0;
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    dcv[q][0] = dcv[q][1] = dcv[q][2] = 0.f;
    totv[q] = 0.f;
    const bool in = q ? G.in1 : G.in0;
    if (!in) continue;
    const int pix = (q ? G.row1 : G.row0) * p.width + G.col;
    const float cc0 = io.color[3 * pix], cc1 = io.color[3 * pix + 1], cc2 = io.color[3 * pix + 2];
    Tfv[q] = io.final_t[pix];
    float dT = 0.f;
    if (LOSS == 0) {
      dcv[q][0] = io.d_color[3 * pix];
      dcv[q][1] = io.d_color[3 * pix + 1];
      dcv[q][2] = io.d_color[3 * pix + 2];
      if (io.d_t) dT = io.d_t[pix];
    } else {
      const float r0 = cc0 - io.target[3 * pix], r1 = cc1 - io.target[3 * pix + 1],
                  r2 = cc2 - io.target[3 * pix + 2];
      lossv += (double)r0 * r0 + (double)r1 * r1 + (double)r2 * r2;
      dcv[q][0] = io.loss_scale * r0;
      dcv[q][1] = io.loss_scale * r1;
      dcv[q][2] = io.loss_scale * r2;
    }
    totv[q] = fmaf(dcv[q][0], cc0, fmaf(dcv[q][1], cc1, fmaf(dcv[q][2], cc2, dT * Tfv[q])));
  }
  if (!sums) return;  // (CTA-uniform) a later segment of a segmented tile
  __syncthreads();
  if (DET)
    block_flush(dcv[0][0] * Tfv[0] + dcv[1][0] * Tfv[1], dcv[0][1] * Tfv[0] + dcv[1][1] * Tfv[1],
                dcv[0][2] * Tfv[0] + dcv[1][2] * Tfv[1], lossv, io.det_bg + 3 * tile,
                LOSS ? io.det_loss + tile : nullptr, true);
  else
    block_flush(dcv[0][0] * Tfv[0] + dcv[1][0] * Tfv[1], dcv[0][1] * Tfv[0] + dcv[1][1] * Tfv[1],
                dcv[0][2] * Tfv[0] + dcv[1][2] * Tfv[1], lossv, io.d_background,
                LOSS ? io.loss_sum : nullptr);
  __syncthreads();
}

}  // namespace vg
