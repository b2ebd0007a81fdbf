// K5 forward blend, K6 backward blend, K8 tomography projector + adjoint.
//
// One 256-thread CTA per 16x16 tile (raster.py:322-329), one pixel per
// thread.  The tile's sorted Gaussian list is staged through shared memory
// in batches of 256: each thread gathers one 64-byte record and derives the
// tile-relative coefficients (c1, c2, c3) once, so the per-pair cost is the
// float32 evaluation in vg_common.cuh plus 4 broadcast LDS.128.
//
// Semantics reproduced exactly (raster.py:332-395, grad.py:135-178):
//   alpha_raw = 1 - exp(-e), alpha = min(alpha_raw, clamp), alpha < cut -> 0;
//   an entry is composited iff the transmittance IN FRONT of it is >= stop;
//   T_final is the transmittance after the last active entry; n_contrib
//   counts active entries with alpha > 0.
// The backward runs front to back and needs no division: with
//   total = dc . color + dT * T_final  (= sum over active of dot*contrib
//                                         + (dc . bg + dT) T_final),
//   suffix_i = total - sum_{j<=i} dot_j contrib_j, and for live entries
//   dL/de_i = dL/dalpha_i (1 - alpha_i) = dot_i T_after_i - suffix_i.
// Per-Gaussian accumulators (13 floats, whitened e-frame, see vg_finalize.cu)
// are warp-reduced with a transpose-reduce (16 shuffles) and one vector of
// 13 red.global.add per warp.
#include "vg_kernels.cuh"

namespace vg {

constexpr unsigned FULL = 0xffffffffu;
constexpr float C_HALF_LOG2E = 0.72134752044448170f;  // 0.5 * log2(e)
constexpr int ACC_STRIDE = 16;                         // floats per Gaussian accumulator

struct __align__(16) SRec {
  float4 a;  // c1, c2, c3, cD2
  float4 b;  // P11, P21, P22, kap2
  float4 c;  // n1, n2, D|beta, gid (bits)
  float4 d;  // r, g, b, 0
};



__device__ __forceinline__ void stage(SRec* sm, int slot, const GRec* __restrict__ rec, uint32_t gid,
                                      int x0, int y0) {
  const GRec g = rec[gid];
  float bu = (float)((double)x0 + 0.5 - g.u);
  float bv = (float)((double)y0 + 0.5 - g.v);
  SRec s;
  s.a = make_float4(g.P11 * bu, fmaf(g.P22, bv, g.P21 * bu), fmaf(g.n2, bv, fmaf(g.n1, bu, g.wm)),
                    g.cD2);
  s.b = make_float4(g.P11, g.P21, g.P22, g.kap2);
  s.c = make_float4(g.n1, g.n2, g.D, __uint_as_float(gid));
  s.d = make_float4(g.cr, g.cg, g.cb, 0.f);
  sm[slot] = s;
}

struct Pair {
  float q1, q2, wp, X, rs, G, E2;
};

// Pinhole ray: the shared (forward == backward) float32 evaluation.  Explicit
// fmaf / __fmul_rn keep the rounding identical in every kernel.
__device__ __forceinline__ Pair eval_pinhole(const SRec& s, float lx, float ly, float Lp) {
  Pair o;
  o.q1 = fmaf(s.b.x, lx, s.a.x);
  o.q2 = fmaf(s.b.y, lx, fmaf(s.b.z, ly, s.a.y));
  o.wp = fmaf(s.c.x, lx, fmaf(s.c.y, ly, s.a.z));
  o.X = fmaf(o.q1, o.q1, __fmul_rn(o.q2, o.q2));
  float W2 = fmaf(o.wp, o.wp, o.X);
  o.rs = rsqf(W2);
  float ri = __fmul_rn(o.rs, o.rs);
  float arg = fmaf(-s.a.w, __fmul_rn(o.X, ri), Lp);
  o.G = __fmul_rn(o.rs, ex2f(arg));
  o.E2 = __fmul_rn(s.b.w, o.G);
  return o;
}

// Parallel ray: beta is per Gaussian (slot c.z), expo = X.
__device__ __forceinline__ Pair eval_parallel(const SRec& s, float lx, float ly) {
  Pair o;
  o.q1 = fmaf(s.b.x, lx, s.a.x);
  o.q2 = fmaf(s.b.y, lx, fmaf(s.b.z, ly, s.a.y));
  o.wp = 0.f;
  o.X = fmaf(o.q1, o.q1, __fmul_rn(o.q2, o.q2));
  o.rs = 0.f;
  o.G = __fmul_rn(s.c.z, ex2f(__fmul_rn(-C_HALF_LOG2E, o.X)));
  o.E2 = __fmul_rn(s.b.w, o.G);
  return o;
}

__device__ __forceinline__ float pixel_lp(const BlendParams& p, int col, int row) {
  float X = ((float)col + 0.5f - p.cx) / p.fx;
  float Y = ((float)row + 0.5f - p.cy) / p.fy;
  return 0.5f * lg2f(fmaf(X, X, fmaf(Y, Y, 1.f)));
}

// Reduce 16 per-lane values over the warp; returns, in every lane, the
// warp total of value index ((l>>4&1)*8 + (l>>3&1)*4 + (l>>2&1)*2 + (l>>1&1)).
__device__ __forceinline__ float transpose_reduce16(float (&v)[16], int lane) {
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    bool hi = lane & 16;
    float send = hi ? v[i] : v[i + 8];
    float keep = hi ? v[i + 8] : v[i];
    v[i] = keep + __shfl_xor_sync(FULL, send, 16);
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    bool hi = lane & 8;
    float send = hi ? v[i] : v[i + 4];
    float keep = hi ? v[i + 4] : v[i];
    v[i] = keep + __shfl_xor_sync(FULL, send, 8);
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    bool hi = lane & 4;
    float send = hi ? v[i] : v[i + 2];
    float keep = hi ? v[i + 2] : v[i];
    v[i] = keep + __shfl_xor_sync(FULL, send, 4);
  }
  {
    bool hi = lane & 2;
    float send = hi ? v[0] : v[1];
    float keep = hi ? v[1] : v[0];
    v[0] = keep + __shfl_xor_sync(FULL, send, 2);
  }
  return v[0] + __shfl_xor_sync(FULL, v[0], 1);
}

__device__ __forceinline__ void flush_acc(float (&v)[16], int lane, uint32_t gid, float* acc) {
  float s = transpose_reduce16(v, lane);
  int idx = ((lane >> 4) & 1) * 8 + ((lane >> 3) & 1) * 4 + ((lane >> 2) & 1) * 2 + ((lane >> 1) & 1);
  if (!(lane & 1) && idx < 13 && s != 0.f) atomicAdd(acc + (size_t)gid * ACC_STRIDE + idx, s);
}

// Block sum of 3 floats + 1 double into global (d_background, loss).
__device__ __forceinline__ void block_flush(float a0, float a1, float a2, double l, float* out3,
                                            double* outl) {
  __shared__ float r3[8][3];
  __shared__ double rl[8];
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
    for (int i = 0; i < 8; ++i) { s0 += r3[i][0]; s1 += r3[i][1]; s2 += r3[i][2]; sl += rl[i]; }
    if (out3) {
      if (s0 != 0.f) atomicAdd(out3 + 0, s0);
      if (s1 != 0.f) atomicAdd(out3 + 1, s1);
      if (s2 != 0.f) atomicAdd(out3 + 2, s2);
    }
    if (outl && sl != 0.0) atomicAdd(outl, sl);
  }
}

// ---------------------------------------------------------------------------
// K5 forward blend (raster.render)

template <bool STOP, bool CUT>
__global__ void __launch_bounds__(256) k_render_fwd(const GRec* __restrict__ rec,
                                                    const uint32_t* __restrict__ vals,
                                                    const uint2* __restrict__ ranges,
                                                    BlendParams p, float* __restrict__ color,
                                                    float* __restrict__ final_t,
                                                    int* __restrict__ n_contrib,
                                                    int* __restrict__ n_act) {
  __shared__ SRec sm[TILE_PIX];
  const int tile = blockIdx.x;
  const int tx = tile % p.ntx, ty = tile / p.ntx;
  const int lxi = threadIdx.x & 15, lyi = threadIdx.x >> 4;
  const int col = tx * TILE + lxi, row = ty * TILE + lyi;
  const bool inside = col < p.width && row < p.height;
  const float lx = (float)lxi, ly = (float)lyi;
  const float Lp = pixel_lp(p, col, row);
  const uint2 r = ranges[tile];
  float T = 1.f, c0 = 0.f, c1 = 0.f, c2 = 0.f;
  int nc = 0, na = 0;
  bool done = !inside;
  for (uint32_t base = r.x; base < r.y; base += TILE_PIX) {
    if (__syncthreads_count(done) == TILE_PIX) break;
    uint32_t i = base + threadIdx.x;
    if (i < r.y) stage(sm, threadIdx.x, rec, vals[i], tx * TILE, ty * TILE);
    __syncthreads();
    const int nb = min((uint32_t)TILE_PIX, r.y - base);
    if (!done) {
      for (int k = 0; k < nb; ++k) {
        if (STOP && T < p.stop) { done = true; break; }
        const SRec s = sm[k];
        Pair e = eval_pinhole(s, lx, ly, Lp);
        float a = fminf(1.f - ex2f(-e.E2), p.clamp);
        if (CUT && a < p.cut) a = 0.f;
        float w = __fmul_rn(a, T);
        c0 = fmaf(w, s.d.x, c0);
        c1 = fmaf(w, s.d.y, c1);
        c2 = fmaf(w, s.d.z, c2);
        nc += (a > 0.f);
        T = fmaf(-a, T, T);
        ++na;
      }
    }
  }
  if (inside) {
    int pix = row * p.width + col;
    color[3 * pix + 0] = fmaf(T, p.bg[0], c0);
    color[3 * pix + 1] = fmaf(T, p.bg[1], c1);
    color[3 * pix + 2] = fmaf(T, p.bg[2], c2);
    final_t[pix] = T;
    n_contrib[pix] = nc;
    n_act[pix] = na;
  }
}

// ---------------------------------------------------------------------------
// K6 backward blend (grad.backward tile_job + e_chain)



template <bool CUT, int LOSS>
__global__ void __launch_bounds__(256) k_render_bwd(const GRec* __restrict__ rec,
                                                    const uint32_t* __restrict__ vals,
                                                    const uint2* __restrict__ ranges,
                                                    BlendParams p, BwdIO io) {
  __shared__ SRec sm[TILE_PIX];
  __shared__ int s_maxna;
  const int tile = blockIdx.x;
  const int tx = tile % p.ntx, ty = tile / p.ntx;
  const int lxi = threadIdx.x & 15, lyi = threadIdx.x >> 4;
  const int lane = threadIdx.x & 31;
  const int col = tx * TILE + lxi, row = ty * TILE + lyi;
  const bool inside = col < p.width && row < p.height;
  const float lx = (float)lxi, ly = (float)lyi;
  const float Lp = pixel_lp(p, col, row);
  const uint2 r = ranges[tile];
  float dc0 = 0.f, dc1 = 0.f, dc2 = 0.f, tot = 0.f, Tf = 1.f;
  double lossv = 0.0;
  int na = 0;
  if (threadIdx.x == 0) s_maxna = 0;
  if (inside) {
    int pix = row * p.width + col;
    float cc0 = io.color[3 * pix], cc1 = io.color[3 * pix + 1], cc2 = io.color[3 * pix + 2];
    Tf = io.final_t[pix];
    na = io.n_act[pix];
    float dT = 0.f;
    if (LOSS == 0) {
      dc0 = io.d_color[3 * pix]; dc1 = io.d_color[3 * pix + 1]; dc2 = io.d_color[3 * pix + 2];
      if (io.d_t) dT = io.d_t[pix];
    } else {
      float r0 = cc0 - io.target[3 * pix], r1 = cc1 - io.target[3 * pix + 1],
            r2 = cc2 - io.target[3 * pix + 2];
      lossv = (double)r0 * r0 + (double)r1 * r1 + (double)r2 * r2;
      dc0 = io.loss_scale * r0; dc1 = io.loss_scale * r1; dc2 = io.loss_scale * r2;
    }
    tot = fmaf(dc0, cc0, fmaf(dc1, cc1, fmaf(dc2, cc2, dT * Tf)));
  }
  __syncthreads();
  if (na) atomicMax(&s_maxna, na);
  block_flush(dc0 * Tf, dc1 * Tf, dc2 * Tf, lossv, io.d_background, LOSS ? io.loss_sum : nullptr);
  __syncthreads();
  const uint32_t end = r.x + (uint32_t)s_maxna;
  float T = 1.f, P = 0.f;
  for (uint32_t base = r.x; base < end; base += TILE_PIX) {
    __syncthreads();
    uint32_t i = base + threadIdx.x;
    if (i < end) stage(sm, threadIdx.x, rec, vals[i], tx * TILE, ty * TILE);
    __syncthreads();
    const int nb = min((uint32_t)TILE_PIX, end - base);
    for (int k = 0; k < nb; ++k) {
      const int j = (int)(base - r.x) + k;
      const SRec s = sm[k];
      float v[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) v[q] = 0.f;
      bool nz = false, vis = false;
      if (j < na) {
        Pair e = eval_pinhole(s, lx, ly, Lp);
        float araw = 1.f - ex2f(-e.E2);
        float a = fminf(araw, p.clamp);
        bool cut = CUT && a < p.cut;
        if (cut) a = 0.f;
        float contrib = __fmul_rn(a, T);
        float Tn = fmaf(-a, T, T);
        float dot = fmaf(dc0, s.d.x, fmaf(dc1, s.d.y, dc2 * s.d.z));
        P = fmaf(dot, contrib, P);
        bool live = !cut && araw < p.clamp;
        float de = live ? fmaf(dot, Tn, P - tot) : 0.f;
        float h = de * e.G;
        float ri = e.rs * e.rs;
        float dr = s.c.z * ri;
        float t = dr * e.wp;
        float r1 = -t * e.q1, r2 = -t * e.q2, r3 = dr * e.X;
        float w1 = e.rs * e.q1, w2 = e.rs * e.q2, w3 = e.rs * e.wp;
        float hr1 = h * r1, hr2 = h * r2, hr3 = h * r3;
        float hw1 = h * w1, hw2 = h * w2, hw3 = h * w3;
        v[0] = fmaf(hr1, r1, hw1 * w1);
        v[1] = fmaf(hr1, r2, hw1 * w2);
        v[2] = fmaf(hr1, r3, hw1 * w3);
        v[3] = fmaf(hr2, r2, hw2 * w2);
        v[4] = fmaf(hr2, r3, hw2 * w3);
        v[5] = fmaf(hr3, r3, hw3 * w3);
        v[6] = hr1; v[7] = hr2; v[8] = hr3;
        v[9] = h;
        v[10] = contrib * dc0; v[11] = contrib * dc1; v[12] = contrib * dc2;
        vis = a > 0.f;
        nz = vis || h != 0.f;
        T = Tn;
      }
      const unsigned any_nz = __ballot_sync(FULL, nz);
      if (any_nz) {
        uint32_t gid = __float_as_uint(s.c.w);
        const bool any_vis = __any_sync(FULL, vis);
        if (lane == 0 && any_vis) io.visible[gid] = 1;
        flush_acc(v, lane, gid, io.acc);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// K8 tomography (tomo.tomo_forward / tomo_backward): order-independent sum
// of e over every binned pair; no cut, clamp or early stop (tomo.py:43-47).

template <int RAY>
__global__ void __launch_bounds__(256) k_tomo_fwd(const GRec* __restrict__ rec,
                                                  const uint32_t* __restrict__ vals,
                                                  const uint2* __restrict__ ranges, BlendParams p,
                                                  float* __restrict__ image,
                                                  float* __restrict__ intensity) {
  __shared__ SRec sm[TILE_PIX];
  const int tile = blockIdx.x;
  const int tx = tile % p.ntx, ty = tile / p.ntx;
  const int lxi = threadIdx.x & 15, lyi = threadIdx.x >> 4;
  const int col = tx * TILE + lxi, row = ty * TILE + lyi;
  const bool inside = col < p.width && row < p.height;
  const float lx = (float)lxi, ly = (float)lyi;
  const float Lp = RAY == VG_PINHOLE ? pixel_lp(p, col, row) : 0.f;
  const uint2 r = ranges[tile];
  float sum = 0.f;
  for (uint32_t base = r.x; base < r.y; base += TILE_PIX) {
    __syncthreads();
    uint32_t i = base + threadIdx.x;
    if (i < r.y) stage(sm, threadIdx.x, rec, vals[i], tx * TILE, ty * TILE);
    __syncthreads();
    const int nb = min((uint32_t)TILE_PIX, r.y - base);
    for (int k = 0; k < nb; ++k) {
      const SRec s = sm[k];
      Pair e = RAY == VG_PINHOLE ? eval_pinhole(s, lx, ly, Lp) : eval_parallel(s, lx, ly);
      sum += e.E2;
    }
  }
  if (inside) {
    int pix = row * p.width + col;
    float I = sum * (float)LN2;
    image[pix] = I;
    if (intensity) intensity[pix] = __expf(-I);
  }
}

template <int RAY, int LOSS>
__global__ void __launch_bounds__(256) k_tomo_bwd(const GRec* __restrict__ rec,
                                                  const uint32_t* __restrict__ vals,
                                                  const uint2* __restrict__ ranges, BlendParams p,
                                                  const float* __restrict__ d_image,
                                                  const float* __restrict__ image,
                                                  const float* __restrict__ target,
                                                  float loss_scale, double* loss_sum,
                                                  float* __restrict__ acc,
                                                  uint8_t* __restrict__ visible) {
  __shared__ SRec sm[TILE_PIX];
  const int tile = blockIdx.x;
  const int tx = tile % p.ntx, ty = tile / p.ntx;
  const int lxi = threadIdx.x & 15, lyi = threadIdx.x >> 4;
  const int lane = threadIdx.x & 31;
  const int col = tx * TILE + lxi, row = ty * TILE + lyi;
  const bool inside = col < p.width && row < p.height;
  const float lx = (float)lxi, ly = (float)lyi;
  const float Lp = RAY == VG_PINHOLE ? pixel_lp(p, col, row) : 0.f;
  const uint2 r = ranges[tile];
  float de = 0.f;
  double lossv = 0.0;
  if (inside) {
    int pix = row * p.width + col;
    if (LOSS == 0) {
      de = d_image[pix];
    } else {
      float rr = image[pix] - target[pix];
      lossv = (double)rr * rr;
      de = loss_scale * rr;
    }
  }
  if (LOSS) block_flush(0.f, 0.f, 0.f, lossv, nullptr, loss_sum);
  for (uint32_t base = r.x; base < r.y; base += TILE_PIX) {
    __syncthreads();
    uint32_t i = base + threadIdx.x;
    if (i < r.y) stage(sm, threadIdx.x, rec, vals[i], tx * TILE, ty * TILE);
    __syncthreads();
    const int nb = min((uint32_t)TILE_PIX, r.y - base);
    for (int k = 0; k < nb; ++k) {
      const SRec s = sm[k];
      float v[16];
#pragma unroll
      for (int q = 0; q < 16; ++q) v[q] = 0.f;
      bool nz = false;
      if (inside) {
        Pair e = RAY == VG_PINHOLE ? eval_pinhole(s, lx, ly, Lp) : eval_parallel(s, lx, ly);
        float h = de * e.G;
        if (RAY == VG_PINHOLE) {
          float ri = e.rs * e.rs;
          float dr = s.c.z * ri;
          float t = dr * e.wp;
          float r1 = -t * e.q1, r2 = -t * e.q2, r3 = dr * e.X;
          float w1 = e.rs * e.q1, w2 = e.rs * e.q2, w3 = e.rs * e.wp;
          float hr1 = h * r1, hr2 = h * r2, hr3 = h * r3;
          float hw1 = h * w1, hw2 = h * w2, hw3 = h * w3;
          v[0] = fmaf(hr1, r1, hw1 * w1);
          v[1] = fmaf(hr1, r2, hw1 * w2);
          v[2] = fmaf(hr1, r3, hw1 * w3);
          v[3] = fmaf(hr2, r2, hw2 * w2);
          v[4] = fmaf(hr2, r3, hw2 * w3);
          v[5] = fmaf(hr3, r3, hw3 * w3);
          v[6] = hr1; v[7] = hr2; v[8] = hr3;
        } else {
          // rho = -(q1, q2, 0), w_hat = (0, 0, 1)
          float hq1 = h * e.q1, hq2 = h * e.q2;
          v[0] = hq1 * e.q1;
          v[1] = hq1 * e.q2;
          v[3] = hq2 * e.q2;
          v[5] = h;
          v[6] = -hq1; v[7] = -hq2;
        }
        v[9] = h;
        nz = e.E2 > 0.f;
      }
      if (__any_sync(FULL, nz)) {
        uint32_t gid = __float_as_uint(s.c.w);
        if (lane == 0) visible[gid] = 1;
        flush_acc(v, lane, gid, acc);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// launchers

void launch_render_fwd(int n_tiles, const GRec* rec, const uint32_t* vals, const uint2* ranges,
                       const BlendParams& p, bool stop, bool cut, float* color, float* final_t,
                       int* n_contrib, int* n_act, cudaStream_t st) {
  if (stop && cut)
    k_render_fwd<true, true><<<n_tiles, 256, 0, st>>>(rec, vals, ranges, p, color, final_t, n_contrib, n_act);
  else if (stop)
    k_render_fwd<true, false><<<n_tiles, 256, 0, st>>>(rec, vals, ranges, p, color, final_t, n_contrib, n_act);
  else if (cut)
    k_render_fwd<false, true><<<n_tiles, 256, 0, st>>>(rec, vals, ranges, p, color, final_t, n_contrib, n_act);
  else
    k_render_fwd<false, false><<<n_tiles, 256, 0, st>>>(rec, vals, ranges, p, color, final_t, n_contrib, n_act);
}

void launch_render_bwd(int n_tiles, const GRec* rec, const uint32_t* vals, const uint2* ranges,
                       const BlendParams& p, bool cut, int loss, const BwdIO& io, cudaStream_t st) {
  if (cut) {
    if (loss) k_render_bwd<true, 1><<<n_tiles, 256, 0, st>>>(rec, vals, ranges, p, io);
    else k_render_bwd<true, 0><<<n_tiles, 256, 0, st>>>(rec, vals, ranges, p, io);
  } else {
    if (loss) k_render_bwd<false, 1><<<n_tiles, 256, 0, st>>>(rec, vals, ranges, p, io);
    else k_render_bwd<false, 0><<<n_tiles, 256, 0, st>>>(rec, vals, ranges, p, io);
  }
}

void launch_tomo_fwd(int n_tiles, int ray, const GRec* rec, const uint32_t* vals,
                     const uint2* ranges, const BlendParams& p, float* image, float* intensity,
                     cudaStream_t st) {
  if (ray == VG_PINHOLE)
    k_tomo_fwd<VG_PINHOLE><<<n_tiles, 256, 0, st>>>(rec, vals, ranges, p, image, intensity);
  else
    k_tomo_fwd<VG_PARALLEL><<<n_tiles, 256, 0, st>>>(rec, vals, ranges, p, image, intensity);
}

void launch_tomo_bwd(int n_tiles, int ray, int loss, const GRec* rec, const uint32_t* vals,
                     const uint2* ranges, const BlendParams& p, const float* d_image,
                     const float* image, const float* target, float loss_scale, double* loss_sum,
                     float* acc, uint8_t* visible, cudaStream_t st) {
#define VG_TB(R, L)                                                                           \
  k_tomo_bwd<R, L><<<n_tiles, 256, 0, st>>>(rec, vals, ranges, p, d_image, image, target,     \
                                            loss_scale, loss_sum, acc, visible)
  if (ray == VG_PINHOLE) {
    if (loss) VG_TB(VG_PINHOLE, 1); else VG_TB(VG_PINHOLE, 0);
  } else {
    if (loss) VG_TB(VG_PARALLEL, 1); else VG_TB(VG_PARALLEL, 0);
  }
#undef VG_TB
}

}  // namespace vg
