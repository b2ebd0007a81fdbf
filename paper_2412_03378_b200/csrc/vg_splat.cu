// mode="splat": the EWA 3DGS comparator of the reference (
// raster.py:353-361 forward, grad.py:170-177 backward).  Same tile layout,
// list order, compositing semantics and culling structure as the analytic
// kernels of vg_blend.cu; only the per-pair alpha differs:
//   alpha_raw = opacity * exp(-maha / 2),  maha = dlt^T conic dlt,
//   dlt = pixel centre - projected mean, conic = (dilated EWA cov2d)^-1.
// The backward leaves, per Gaussian and view, dL/dopacity, dL/dconic (3) and
// dL/dmean2d (2) in accumulator slots 0..5 (colour in 10..12 as in the
// analytic path); vg_finalize.cu chains them through the EWA projection
// (grad.py:262-302).
//
// Culling is result-preserving: maha >= lambda_min(conic) * dist^2 with dist
// the distance from the projected mean to the 8x8 block, so a block is
// skipped only when opacity * exp(-lambda_min dist^2 / 2) < alpha_cut
// (1e-3 margin).
#include "vg_blend.cuh"

namespace vg {

struct __align__(16) SplatRec {
  float4 a;  // bu, bv (tile-relative offsets of the pixel-(0,0) centre), l00, l01
  float4 b;  // l11, opacity, 0, gid (bits)
  float4 d;  // r, g, b, 0
};

// GRec fields in splat mode (vg_preprocess.cu): P11/P21/P22 = conic,
// kap2 = amp = opacity, n1 = lambda_min(conic).
__device__ __forceinline__ uint32_t stage_splat(SplatRec* sm, int slot, const GRec* __restrict__ rec,
                                                uint32_t gid, int x0, int y0, bool cull, float cut) {
  const GRec g = rec[gid];
  const float bu = (float)((double)x0 + 0.5 - g.u);
  const float bv = (float)((double)y0 + 0.5 - g.v);
  SplatRec s;
  s.a = make_float4(bu, bv, g.P11, g.P21);
  s.b = make_float4(g.P22, g.kap2, 0.f, __uint_as_float(gid));
  s.d = make_float4(g.cr, g.cg, g.cb, 0.f);
  sm[slot] = s;
  if (!cull) return 0xFu;
  if (!(g.kap2 > cut)) return 0u;
  const float lnr = __logf(g.kap2 / cut * 1.001f);  // alpha >= cut needs lmin d^2 / 2 <= lnr
  uint32_t m = 0;
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    const float xa = (float)(8 * (b & 1)), ya = (float)(8 * (b >> 1));
    const float dx = d0(bu + xa, bu + xa + 7.f), dy = d0(bv + ya, bv + ya + 7.f);
    if (0.5f * g.n1 * (dx * dx + dy * dy) * 0.999f <= lnr) m |= 1u << b;
  }
  return m;
}

struct SplatPair {
  float dx;
  F2 dy, fall, raw;
};

__device__ __forceinline__ SplatPair eval_splat2(const SplatRec& s, float lx, F2 ly) {
  SplatPair o;
  o.dx = s.a.x + lx;
  o.dy = add2(f2s(s.a.y), ly);
  // maha = l00 dx^2 + 2 l01 dx dy + l11 dy^2
  const F2 t = fma2(f2s(s.b.x), o.dy, f2s(2.f * s.a.w * o.dx));
  const F2 maha = fma2(t, o.dy, f2s(s.a.z * o.dx * o.dx));
  o.fall = ex2_2(mul2(f2s(-C_HALF_LOG2E), maha));
  o.raw = mul2(f2s(s.b.y), o.fall);
  return o;
}

// transmittance factor of one pixel: 1 when cut or inactive, else
// max(1 - alpha_raw, 1 - clamp) (the analytic path's floor, see vg_blend.cu)
__device__ __forceinline__ float splat_om(float raw, bool act, const BlendParams& p, bool& cut) {
  cut = p.cut > 0.f && raw < p.cut;
  return (cut || !act) ? 1.f : fmaxf(1.f - raw, p.cc);
}

template <bool COUNTS>
__global__ void __launch_bounds__(NT) k_splat_fwd(const GRec* __restrict__ rec,
                                                  const uint32_t* __restrict__ vals,
                                                  const uint2* __restrict__ ranges,
                                                  const uint32_t* __restrict__ order,
                                                  BlendParams p, float* __restrict__ color,
                                                  float* __restrict__ final_t,
                                                  int* __restrict__ n_contrib,
                                                  int* __restrict__ n_act) {
  __shared__ SplatRec sm[BATCH];
  __shared__ uint8_t smask[BATCH];
  const int tile = order[blockIdx.x];
  const int tx = tile % p.ntx, ty = tile / p.ntx;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const LaneGeo G = lane_geo(p, tx, ty);
  const float lx = (float)G.lxi;
  const F2 ly = f2((float)G.ly0, (float)(G.ly0 + 4));
  const uint2 r = ranges[tile];
  float T0 = G.in0 ? 1.f : 0.f, T1 = G.in1 ? 1.f : 0.f;
  float C0[3] = {0.f, 0.f, 0.f}, C1[3] = {0.f, 0.f, 0.f};
  int nc0 = 0, nc1 = 0, na0 = 0, na1 = 0;
  bool done = !(G.in0 || G.in1);
  for (uint32_t base = r.x; base < r.y; base += BATCH) {
    if (__syncthreads_count(done) == NT) break;
    for (int sidx = threadIdx.x; sidx < BATCH; sidx += NT) {
      const uint32_t i = base + sidx;
      if (i < r.y) smask[sidx] = (uint8_t)stage_splat(sm, sidx, rec, vals[i], tx * TILE, ty * TILE,
                                                      p.cut > 0.f, p.cut);
    }
    __syncthreads();
    const int nb = min((uint32_t)BATCH, r.y - base);
    const int jb = (int)(base - r.x) + 1;
    for (int c = 0; c < nb && !__all_sync(FULL, done); c += 32) {
      const bool vb = (c + lane < nb) && ((smask[c + lane] >> warp) & 1);
      unsigned bits = __ballot_sync(FULL, vb);
      while (bits) {
        const int k = c + __ffs(bits) - 1;
        bits &= bits - 1;
        const SplatRec s = sm[k];
        const SplatPair e = eval_splat2(s, lx, ly);
        const bool a0 = T0 >= p.stop, a1 = T1 >= p.stop;
        bool cut0, cut1;
        const float om0 = splat_om(lo(e.raw), a0, p, cut0), om1 = splat_om(hi(e.raw), a1, p, cut1);
        const float w0 = (1.f - om0) * T0, w1 = (1.f - om1) * T1;
        C0[0] = fmaf(w0, s.d.x, C0[0]); C0[1] = fmaf(w0, s.d.y, C0[1]); C0[2] = fmaf(w0, s.d.z, C0[2]);
        C1[0] = fmaf(w1, s.d.x, C1[0]); C1[1] = fmaf(w1, s.d.y, C1[1]); C1[2] = fmaf(w1, s.d.z, C1[2]);
        T0 *= om0;
        T1 *= om1;
        if (COUNTS) {
          na0 = a0 ? jb + k : na0;
          na1 = a1 ? jb + k : na1;
          nc0 += om0 < 1.f;
          nc1 += om1 < 1.f;
        }
      }
      done = !(T0 >= p.stop) && !(T1 >= p.stop);
    }
  }
  const int len = (int)(r.y - r.x);
  if (T0 >= p.stop) na0 = len;
  if (T1 >= p.stop) na1 = len;
  if (G.in0) {
    const int pix = G.row0 * p.width + G.col;
    for (int q = 0; q < 3; ++q) color[3 * pix + q] = fmaf(T0, p.bg[q], C0[q]);
    final_t[pix] = T0;
    if (COUNTS) { n_contrib[pix] = nc0; n_act[pix] = na0; }
  }
  if (G.in1) {
    const int pix = G.row1 * p.width + G.col;
    for (int q = 0; q < 3; ++q) color[3 * pix + q] = fmaf(T1, p.bg[q], C1[q]);
    final_t[pix] = T1;
    if (COUNTS) { n_contrib[pix] = nc1; n_act[pix] = na1; }
  }
}

template <int LOSS, bool DET>
__global__ void __launch_bounds__(NT) k_splat_bwd(const GRec* __restrict__ rec,
                                                  const uint32_t* __restrict__ vals,
                                                  const uint2* __restrict__ ranges,
                                                  const uint32_t* __restrict__ order,
                                                  BlendParams p, BwdIO io) {
  __shared__ SplatRec sm[BATCH];
  __shared__ uint8_t smask[BATCH];
  const int tile = order[blockIdx.x];
  const int tx = tile % p.ntx, ty = tile / p.ntx;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const LaneGeo G = lane_geo(p, tx, ty);
  const float lx = (float)G.lxi;
  const F2 ly = f2((float)G.ly0, (float)(G.ly0 + 4));
  const uint2 r = ranges[tile];
  float dcv[2][3], totv[2];
  bwd_prologue<LOSS, DET>(p, G, io, dcv, totv, tile);
  float T[2] = {G.in0 ? 1.f : 0.f, G.in1 ? 1.f : 0.f}, P[2] = {0.f, 0.f};
  const bool in[2] = {G.in0, G.in1};
  bool done = !(G.in0 || G.in1);
  for (uint32_t base = r.x; base < r.y; base += BATCH) {
    if (__syncthreads_count(done) == NT) break;
    for (int sidx = threadIdx.x; sidx < BATCH; sidx += NT) {
      const uint32_t i = base + sidx;
      if (i < r.y) smask[sidx] = (uint8_t)stage_splat(sm, sidx, rec, vals[i], tx * TILE, ty * TILE,
                                                      p.cut > 0.f, p.cut);
    }
    __syncthreads();
    const int nb = min((uint32_t)BATCH, r.y - base);
    for (int c = 0; c < nb && !__all_sync(FULL, done); c += 32) {
      const bool vb = (c + lane < nb) && ((smask[c + lane] >> warp) & 1);
      unsigned bits = __ballot_sync(FULL, vb);
      while (bits) {
        const int k = c + __ffs(bits) - 1;
        bits &= bits - 1;
        const SplatRec s = sm[k];
        const SplatPair e = eval_splat2(s, lx, ly);
        float v[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) v[q] = 0.f;
        bool any_vis = false, any_live = false;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const float raw = q ? hi(e.raw) : lo(e.raw), fall = q ? hi(e.fall) : lo(e.fall);
          const float dy = q ? hi(e.dy) : lo(e.dy), dx = e.dx;
          const bool act = in[q] && T[q] >= p.stop;
          bool cut;
          const float om = splat_om(raw, act, p, cut);
          const float contrib = (1.f - om) * T[q];
          const float Tn = T[q] * om;
          const float dot = fmaf(dcv[q][0], s.d.x, fmaf(dcv[q][1], s.d.y, dcv[q][2] * s.d.z));
          P[q] = fmaf(dot, contrib, P[q]);
          T[q] = Tn;
          any_vis |= om < 1.f;
          // live: not cut, active and not clamped; dL/dalpha_raw = dL/dalpha
          if (!cut && act && raw < p.clamp) {
            any_live = true;
            const float dar = (dot * Tn - (totv[q] - P[q])) / om;
            const float dm = -0.5f * fall * dar * s.b.y;
            v[0] += dar * fall;
            v[1] += dm * dx * dx;
            v[2] += dm * dx * dy;
            v[3] += dm * dy * dy;
            v[4] += -2.f * dm * (s.a.z * dx + s.a.w * dy);
            v[5] += -2.f * dm * (s.a.w * dx + s.b.x * dy);
          }
          v[10] += contrib * dcv[q][0];
          v[11] += contrib * dcv[q][1];
          v[12] += contrib * dcv[q][2];
        }
        const bool wvis = __any_sync(FULL, any_vis);
        const bool wlive = __any_sync(FULL, any_live);
        if (wvis || wlive) {
          const uint32_t gid = __float_as_uint(s.b.w);
          if (lane == 0 && wvis) io.visible[gid] = 1;
          if (DET)
            flush_det(v, lane, io.det_part + ((size_t)(base + k) * (NT / 32) + warp) * ACC_STRIDE);
          else
            flush_acc(v, lane, gid, io.acc);
        }
      }
      done = !(G.in0 && T[0] >= p.stop) && !(G.in1 && T[1] >= p.stop);
    }
  }
}

void launch_splat_fwd(int n_tiles, const GRec* rec, const uint32_t* vals, const uint2* ranges,
                      const uint32_t* order, const BlendParams& p, float* color, float* final_t,
                      int* n_contrib, int* n_act, cudaStream_t st) {
  if (n_contrib)
    k_splat_fwd<true><<<n_tiles, NT, 0, st>>>(rec, vals, ranges, order, p, color, final_t,
                                              n_contrib, n_act);
  else
    k_splat_fwd<false><<<n_tiles, NT, 0, st>>>(rec, vals, ranges, order, p, color, final_t,
                                               nullptr, nullptr);
}

void launch_splat_bwd(int n_tiles, const GRec* rec, const uint32_t* vals, const uint2* ranges,
                      const uint32_t* order, const BlendParams& p, int loss, const BwdIO& io,
                      cudaStream_t st) {
  const bool det = io.det_part != nullptr;
#define VG_SB(L, D) k_splat_bwd<L, D><<<n_tiles, NT, 0, st>>>(rec, vals, ranges, order, p, io)
  if (det) {
    if (loss) VG_SB(1, true); else VG_SB(0, true);
  } else {
    if (loss) VG_SB(1, false); else VG_SB(0, false);
  }
#undef VG_SB
}

}  // namespace vg
