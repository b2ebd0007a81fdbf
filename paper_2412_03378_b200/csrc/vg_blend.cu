// K5 forward blend, K6 backward blend, K8 tomography projector + adjoint.
//
// Layout: one 128-thread CTA per 16x16 tile (raster.py:322-329), launched in
// heavy-tiles-first order.  Each warp owns an 8x8 pixel block; each lane owns
// two pixels of one column (rows r and r+4) and evaluates both with packed
// FP32x2 instructions (FFMA2/FMUL2/FADD2); exp2 / rsqrt run on the SFU.
// The tile's depth-sorted list is staged through shared memory in batches of
// 256 records; the staging thread derives the tile-relative coefficients once
// and a 4-bit mask of the warp blocks the Gaussian can reach.
//
// Culling (result-preserving): e = kappa sqrt(2pi) beta peak with
// beta <= s_max and expo = D^2 X / (w_par^2 + X), so alpha >= alpha_cut at
// some pixel of a block needs X (D^2 - R^2) <= R^2 w_par^2 there, with
// R^2 = 2 ln(kappa sqrt(2pi) s_max / e_cut).  A block is skipped only when the
// interval lower bound of X and upper bound of w_par^2 over the block violate
// it (with a 1e-3 margin on e_cut); every skipped pair would have been cut to
// alpha = 0, so images, n_contrib and gradients are unchanged.
//
// Semantics reproduced exactly (raster.py:332-395, grad.py:135-178):
//   alpha_raw = 1 - exp(-e), alpha = min(alpha_raw, clamp), alpha < cut -> 0;
//   an entry is composited iff the transmittance IN FRONT of it is >= stop;
//   T_final is the transmittance after the last active entry; n_contrib
//   counts active entries with alpha > 0.
// The transmittance factor is carried directly: om = max(exp(-e), 1-clamp)
// (1 if cut), T <- T * om, alpha = 1 - om.
// The backward runs front to back and needs no division: with
//   total = dc . color + dT * T_final  (= sum over active of dot*contrib
//                                         + (dc . bg + dT) T_final),
//   suffix_i = total - sum_{j<=i} dot_j contrib_j, and for live entries
//   dL/de_i = dL/dalpha_i (1 - alpha_i) = dot_i T_after_i - suffix_i.
// Per-Gaussian accumulators (13 floats, whitened e-frame, see vg_finalize.cu)
// are summed over the lane's two pixels, warp-reduced through shared memory
// (smem_reduce13x2p: two entries per pass, packed) and added with one 13-lane
// red.global.add per warp and entry.
#include "vg_blend.cuh"

// The file is compiled twice (build.py): VG_TU=1 holds the forward kernel
// (built with ptxas -regUsageLevel=6: forward -2.3 % on config 3, -4.3 % on
// config 4; the same level makes the backward 0.8 % slower), VG_TU=2 the rest.
// Without VG_TU everything is built (tools, A/B builds).
#if !defined(VG_TU) || VG_TU == 1
#define VG_TU_FWD 1
#else
#define VG_TU_FWD 0
#endif
#if !defined(VG_TU) || VG_TU == 2
#define VG_TU_REST 1
#else
#define VG_TU_REST 0
#endif

// minimum resident CTAs per SM requested from ptxas (register budget); A/B knobs
#ifndef VG_FWD_MINB
// 8: <= 64 registers.  With the branch-free entry pairs, 8 CTAs / 63 registers
// beat 10 / 48 (config 3 step 121.5 -> 120.3 ms, config 2 3.86 -> 3.77 ms);
// 6, 7, 9 and 12 were slower
#define VG_FWD_MINB 8
#endif
#ifndef VG_DEEP_ILP
// deep-tile forward: entries evaluated ahead (4 and 8 measured the same; the
// deepest config-4 tile alone on an SM: 521 -> 391 us)
#define VG_DEEP_ILP 4
#endif
#ifndef VG_SEEN_REDUX
#define VG_SEEN_REDUX 1  // forward: per-lane visibility bits, one warp OR per chunk
#endif
#ifndef VG_BWD_PAIR
// two visible entries per step: 1 = both replays, then both entries' gradient
// terms, two reductions; 2 = the same with one shared-memory pass for both,
// packed 8-byte stores (A/B on config 3, 16 views: backward 21.1 -> 20.0 ->
// 18.9 ms; packed pass 17.65 -> 17.28 ms)
#define VG_BWD_PAIR 2
#endif
#ifndef VG_TOMO_SKIP
// projector: (entry, column) pairs whose peak in the column is below 2^-60 of
// the Gaussian's peak (< 1e-18 relative; far below float32 resolution) are not
// summed (-40: another 3.5 %, but that is the size of the reference's own
// binning cut and is left alone)
#define VG_TOMO_SKIP -60.f
#endif
#ifndef VG_TOMO_MOM
#define VG_TOMO_MOM 1   // parallel-beam adjoint in moment form (-18 % on config 5)
#endif
#ifndef VG_TOMO_REC
#define VG_TOMO_REC 1   // parallel-beam projector: row recurrence (k_tomo_fwd_rec), -21 % on config 5
#endif
#ifndef VG_SMEM_RED
#define VG_SMEM_RED 1   // backward warp sums through shared memory (smem_reduce13)
#endif

namespace vg {

// debug builds: a list entry must name a scene primitive
__device__ __forceinline__ uint32_t chk_gid(const BlendParams& p, uint32_t gid) {
  VG_ASSERT((int64_t)gid < p.dbg_n);
  return gid;
}

struct __align__(16) SRec {
  float4 a;  // c1, c2, c3, cD2
  float4 b;  // P11, P21, P22, kap2
  float4 c;  // n1, n2, D|beta, gid (bits)
  float4 d;  // r, g, b, 0
};

// Tile-relative record of Gaussian gid for the tile at pixel origin (x0, y0).
__device__ __forceinline__ SRec make_srec(const GRec& g, uint32_t gid, int x0, int y0) {
  const float bu = (float)((double)x0 + 0.5 - g.u);
  const float bv = (float)((double)y0 + 0.5 - g.v);
  SRec s;
  s.a = make_float4(g.P11 * bu, fmaf(g.P22, bv, g.P21 * bu), fmaf(g.n2, bv, fmaf(g.n1, bu, g.wm)), g.cD2);
  s.b = make_float4(g.P11, g.P21, g.P22, g.kap2);
  s.c = make_float4(g.n1, g.n2, g.D, __uint_as_float(gid));
  s.d = make_float4(g.cr, g.cg, g.cb, 0.f);
  return s;
}

// Stage one record for the tile at pixel origin (x0, y0); return the 4-bit
// mask of 8x8 warp blocks the Gaussian may reach with alpha >= cut.
// Bound per block: e = K beta exp(-expo/2) with K = kappa sqrt(2pi),
//   beta = |d'| / |w| <= min(s_max, dmax / sqrt(w_par_min^2 + X_min)),
//   expo = D^2 X / (w_par^2 + X) >= D^2 X_min / (w_par_max^2 + X_min),
// X_min / w_par ranges from interval arithmetic over the block (q1, q2, w_par
// are affine in the pixel offset), dmax = max |d'| over the block's corners.
__device__ __forceinline__ uint32_t stage_rec(SRec* sm, int slot, const GRec& g, uint32_t gid,
                                              int x0, int y0, bool cull, float ecut,
                                              const float* __restrict__ dmax4 = nullptr) {
  const SRec s = make_srec(g, gid, x0, y0);
  const float c1 = s.a.x, c2 = s.a.y, c3 = s.a.z;
  sm[slot] = s;
  if (!cull) return 0xFu;
  if (!(g.amp > ecut)) return 0u;  // alpha < cut at every pixel
  const float K = g.kap2 * 0.69314718f;  // kappa sqrt(2 pi)
  const float D2 = g.D * g.D;
  const float inv_ecut = 1.f / ecut;
  uint32_t m = 0;
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    const float xa = (float)(8 * (b & 1)), xb = xa + 7.f;
    const float ya = (float)(8 * (b >> 1)), yb = ya + 7.f;
    float q1a = fmaf(g.P11, xa, c1), q1b = fmaf(g.P11, xb, c1);
    float pxa = g.P21 * xa, pxb = g.P21 * xb, pya = g.P22 * ya, pyb = g.P22 * yb;
    float q2lo = c2 + fminf(pxa, pxb) + fminf(pya, pyb);
    float q2hi = c2 + fmaxf(pxa, pxb) + fmaxf(pya, pyb);
    float nxa = g.n1 * xa, nxb = g.n1 * xb, nya = g.n2 * ya, nyb = g.n2 * yb;
    float wlo = c3 + fminf(nxa, nxb) + fminf(nya, nyb);
    float whi = c3 + fmaxf(nxa, nxb) + fmaxf(nya, nyb);
    float t1 = d0(fminf(q1a, q1b), fmaxf(q1a, q1b));
    float t2 = d0(q2lo, q2hi);
    const float Xmin = (t1 * t1 + t2 * t2) * 0.999f;
    const float wmax2 = fmaxf(wlo * wlo, whi * whi) * 1.001f;
    const float wd = d0(wlo, whi);
    const float wmin2 = wd * wd * 0.999f;
    float A = g.amp;
    if (dmax4) A = fminf(A, K * dmax4[b] * rsqf(fmaxf(wmin2 + Xmin, 1e-30f)));
    A *= 1.001f;
    if (!(A > ecut)) continue;
    const float L = __logf(A * inv_ecut);
    if (D2 * Xmin <= 2.f * L * (wmax2 + Xmin)) m |= 1u << b;
  }
  return m;
}

__device__ __forceinline__ uint32_t stage(SRec* sm, int slot, const GRec* __restrict__ rec,
                                          uint32_t gid, int x0, int y0, bool cull, float ecut,
                                          const float* __restrict__ dmax4 = nullptr) {
  const GRec g = rec[gid];
  return stage_rec(sm, slot, g, gid, x0, y0, cull, ecut, dmax4);
}

// max |d'| = max sqrt(1 + X^2 + Y^2) over the corners of each 8x8 block of a tile
__device__ __forceinline__ void block_dmax(const BlendParams& p, int tx, int ty, float* out4) {
  if (threadIdx.x < 4) {
    const int b = threadIdx.x;
    float best = 0.f;
    for (int cy = 0; cy < 2; ++cy)
      for (int cx = 0; cx < 2; ++cx) {
        const float col = (float)(tx * TILE + 8 * (b & 1) + 7 * cx) + 0.5f;
        const float row = (float)(ty * TILE + 8 * (b >> 1) + 7 * cy) + 0.5f;
        const float X = (col - p.cx) / p.fx, Y = (row - p.cy) / p.fy;
        best = fmaxf(best, fmaf(X, X, fmaf(Y, Y, 1.f)));
      }
    out4[b] = sqrtf(best) * 1.0001f;
  }
}

struct Pair2 {
  float q1;
  F2 q2, wp, X, rs, G, E2, ex;
};

// Pinhole rays, two pixels (same column lx, rows ly.x / ly.y).  The single
// shared evaluation for forward and backward (identical rounding).
// CUT: entries with alpha_raw < alpha_cut get the transmittance factor
// ex = 1 exactly, so the callers need no separate cut test: om = max(ex,
// floor) is 1 for cut and inactive entries alike, and every other factor is
// exp(-e) < 1 in float32 (alpha_cut >= 6e-8).  The decision is taken on E2 = e log2(e),
// which carries full float32 relative precision: testing exp(-e) ~ 0.996
// against 1 - cut would quantise alpha to 1.5e-5 relative and flip ~0.3 %
// of the pixels of a dense view against the float64 reference.
template <bool CUT = false>
__device__ __forceinline__ Pair2 eval_pinhole2(const SRec& s, float lx, F2 ly, F2 Lp, float e2cut = 0.f) {
  Pair2 o;
  o.q1 = fmaf(s.b.x, lx, s.a.x);
  const float t2 = fmaf(s.b.y, lx, s.a.y);
  o.q2 = fma2(f2s(s.b.z), ly, f2s(t2));
  const float tw = fmaf(s.c.x, lx, s.a.z);
  o.wp = fma2(f2s(s.c.y), ly, f2s(tw));
  o.X = fma2(o.q2, o.q2, f2s(__fmul_rn(o.q1, o.q1)));
  const F2 W2 = fma2(o.wp, o.wp, o.X);
  o.rs = rsq_2(W2);
  const F2 ri = mul2(o.rs, o.rs);
  const F2 arg = fma2(f2s(-s.a.w), mul2(o.X, ri), Lp);
  o.G = mul2(o.rs, ex2_2(arg));
  o.E2 = mul2(f2s(s.b.w), o.G);
  o.ex = ex2_2(neg2(o.E2));
  if (CUT) o.ex = sel2(lo(o.E2) < e2cut, hi(o.E2) < e2cut, f2s(1.f), o.ex);
  return o;
}

// Parallel rays: beta is per Gaussian (slot c.z), expo = X.
__device__ __forceinline__ Pair2 eval_parallel2(const SRec& s, float lx, F2 ly) {
  Pair2 o;
  o.q1 = fmaf(s.b.x, lx, s.a.x);
  const float t2 = fmaf(s.b.y, lx, s.a.y);
  o.q2 = fma2(f2s(s.b.z), ly, f2s(t2));
  o.wp = f2s(0.f);
  o.X = fma2(o.q2, o.q2, f2s(__fmul_rn(o.q1, o.q1)));
  o.rs = f2s(0.f);
  o.G = mul2(f2s(s.c.z), ex2_2(mul2(f2s(-C_HALF_LOG2E), o.X)));
  o.E2 = mul2(f2s(s.b.w), o.G);
  o.ex = f2s(1.f);
  return o;
}

__device__ __forceinline__ float pixel_lp(const BlendParams& p, int col, int row) {
  float X = ((float)col + 0.5f - p.cx) / p.fx;
  float Y = ((float)row + 0.5f - p.cy) / p.fy;
  return 0.5f * lg2f(fmaf(X, X, fmaf(Y, Y, 1.f)));
}

#if VG_TU_FWD
// ---------------------------------------------------------------------------
// K5 forward blend (raster.render)

__device__ unsigned long long g_vg_stats[4];  // debug: processed / visible warp-entries, list entries

// COUNTS: also produce n_contrib and n_active (the render API and the
// roofline statistics); the training step's forward skips them -- the
// backward re-derives activity from its own transmittance replay.
// DEEP: the latency-bound variant for the few very deep tiles of a tail-bound
// view (run beside the regular launch): VG_DEEP_ILP visible entries' alpha
// factors evaluated ahead of their (sequential) compositing, at low occupancy
template <bool STOP, bool CUT, bool STATS = false, bool COUNTS = true, bool DEEP = false>
__global__ void __launch_bounds__(NT, DEEP ? 2 : VG_FWD_MINB) k_render_fwd(const GRec* __restrict__ rec,
                                                   const uint32_t* __restrict__ vals,
                                                   const uint2* __restrict__ ranges,
                                                   const uint32_t* __restrict__ order,
                                                   BlendParams p, float* __restrict__ color,
                                                   float* __restrict__ final_t,
                                                   int* __restrict__ n_contrib,
                                                   int* __restrict__ n_act,
                                                   uint32_t* __restrict__ vmask, int vm_words,
                                                   SegIO seg) {
  unsigned long long st_proc = 0, st_vis = 0, st_tot = 0;
  cta_log_begin(p);
  __shared__ SRec sm[BATCH];
  __shared__ uint8_t smask[BATCH];
  __shared__ float sdmax[4];
  const int tile = order[blockIdx.x];
  const int tx = tile % p.ntx, ty = tile / p.ntx;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const LaneGeo G = lane_geo(p, tx, ty);
  const float lx = (float)G.lxi;
  const F2 ly = f2((float)G.ly0, (float)(G.ly0 + 4));
  const F2 Lp = f2(pixel_lp(p, G.col, G.row0), pixel_lp(p, G.col, G.row1));
  const uint2 r = ranges[tile];
  block_dmax(p, tx, ty, sdmax);
  // Pixels outside the image start (and stay) at T = 0: never active.
  F2 T = f2(G.in0 ? 1.f : 0.f, G.in1 ? 1.f : 0.f);
  F2 Cr = f2s(0.f), Cg = f2s(0.f), Cb = f2s(0.f);
  // floor of the transmittance factor: 1 - clamp while active, 1 once stopped
  float fl0 = G.in0 ? p.cc : 1.f, fl1 = G.in1 ? p.cc : 1.f;
  int nc0 = 0, nc1 = 0, na0 = 0, na1 = 0;
  bool done = !(G.in0 || G.in1);
  VG_ASSERT(r.x <= r.y && (int64_t)r.y <= p.dbg_pairs);
  // after the loop, min(base, r.y) is the end of the last batch walked (the
  // tile's depth)
  uint32_t base = r.x;
#if VG_CTA_LOG
  unsigned long long w_walk = 0, w_stage = 0;  // this warp's cycles: chunk walk, staging + its barrier
#endif
  for (; base < r.y; base += BATCH) {
    VG_JITTER(p.dbg_jitter, base);
    if (__syncthreads_count(done) == NT) break;
#if VG_CTA_LOG
    const unsigned long long c0 = clock64();
#endif
    if (seg.on && base != r.x && ((base - r.x) & (VG_SEG - 1)) == 0) {
      // a segment boundary: the state the backward's replay of the next segment starts from
      float4* o = seg.state + ((size_t)(base / VG_SEG) * NT + threadIdx.x) * 2;
      o[0] = make_float4(lo(T), hi(T), lo(Cr), hi(Cr));
      o[1] = make_float4(lo(Cg), hi(Cg), lo(Cb), hi(Cb));
    }
    if constexpr (DEEP) {
      // both of this thread's entries: list values, then both records, in
      // flight together (a missing entry re-reads the batch's first; in the
      // regular kernel the two records spill: forward +13 % at 48 and at 63
      // registers)
      static_assert(BATCH == 2 * NT, "two staged entries per thread");
      const uint32_t i0 = base + threadIdx.x, i1 = i0 + NT;
      const bool v0 = i0 < r.y, v1 = i1 < r.y;
      const uint32_t g0 = chk_gid(p, vals[v0 ? i0 : base]), g1 = chk_gid(p, vals[v1 ? i1 : base]);
      const GRec R0 = rec[g0], R1 = rec[g1];
      if (v0) smask[threadIdx.x] = (uint8_t)stage_rec(sm, threadIdx.x, R0, g0, tx * TILE, ty * TILE, CUT, p.ecut, sdmax);
      if (v1) smask[threadIdx.x + NT] = (uint8_t)stage_rec(sm, threadIdx.x + NT, R1, g1, tx * TILE, ty * TILE, CUT, p.ecut, sdmax);
    } else
    for (int sidx = threadIdx.x; sidx < BATCH; sidx += NT) {
      uint32_t i = base + sidx;
      if (i < r.y)
        smask[sidx] = (uint8_t)stage(sm, sidx, rec, chk_gid(p, vals[i]), tx * TILE, ty * TILE, CUT, p.ecut, sdmax);
    }
    __syncthreads();
#if VG_CTA_LOG
    const unsigned long long c1 = clock64();
    w_stage += c1 - c0;
#endif
    const int nb = min((uint32_t)BATCH, r.y - base);
    const int jb = (int)(base - r.x) + 1;
    for (int c = 0; c < nb && !__all_sync(FULL, done); c += 32) {
      VG_JITTER(p.dbg_jitter, base + c + 1);
      const bool vb = (c + lane < nb) && ((smask[c + lane] >> warp) & 1);
      unsigned bits = __ballot_sync(FULL, vb);
      unsigned seen = 0;  // entries of this chunk with a visible pixel in this warp's block
      // composite one evaluated entry (front to back; T carries the order)
      auto composite_ex = [&](int k, const float4& d, F2 ex) {
        if (STOP) {
          // active iff the transmittance in front is >= stop (raster.py:384-385);
          // n_act = 1 + index of the last active processed entry
          const bool a0 = lo(T) >= p.stop, a1 = hi(T) >= p.stop;
          fl0 = a0 ? p.cc : 1.f;
          fl1 = a1 ? p.cc : 1.f;
          if (COUNTS) {
            na0 = a0 ? jb + k : na0;
            na1 = a1 ? jb + k : na1;
          }
        }
        // cut entries carry the factor 1 (eval_pinhole2), inactive ones the
        // floor 1: either way om = 1, no contribution, no count
        const float om0 = fmaxf(lo(ex), fl0), om1 = fmaxf(hi(ex), fl1);
        if (COUNTS) {
          nc0 += om0 < 1.f;
          nc1 += om1 < 1.f;
        }
        const F2 om = f2(om0, om1);
        const F2 w = mul2(sub2(f2s(1.f), om), T);
        Cr = fma2(w, f2s(d.x), Cr);
        Cg = fma2(w, f2s(d.y), Cg);
        Cb = fma2(w, f2s(d.z), Cb);
        T = mul2(T, om);
#if VG_SEEN_REDUX
        // per-lane bits, OR-reduced over the warp once per chunk
        if (vmask) seen |= (om0 < 1.f || om1 < 1.f ? 1u : 0u) << (k - c);
#else
        if (vmask && __any_sync(FULL, om0 < 1.f || om1 < 1.f)) seen |= 1u << (k - c);
#endif
        if (STATS) {
          st_proc++;
          st_vis += __any_sync(FULL, om0 < 1.f || om1 < 1.f) ? 1 : 0;
        }
      };
      if constexpr (DEEP) {
        // up to VG_DEEP_ILP visible entries evaluated, then composited in order
        constexpr int ILP = VG_DEEP_ILP;
        // (branch-free: missing entries repeat the last one, so the
        // evaluations are straight-line code the scheduler interleaves)
        while (bits) {
          int kk[ILP];
          F2 xe[ILP];
          int m = 0;
#pragma unroll
          for (int j = 0; j < ILP; ++j) {
            const bool v = bits != 0u;
            kk[j] = v ? c + __ffs(bits) - 1 : kk[j > 0 ? j - 1 : 0];
            m = v ? j + 1 : m;
            bits &= bits - 1u;
          }
#pragma unroll
          for (int j = 0; j < ILP; ++j) xe[j] = eval_pinhole2<CUT>(sm[kk[j]], lx, ly, Lp, p.e2cut).ex;
#pragma unroll
          for (int j = 0; j < ILP; ++j)
            if (j < m) composite_ex(kk[j], sm[kk[j]].d, xe[j]);
        }
      } else {
        // two visible entries per iteration, evaluated branch-free (the second
        // repeats the first when the chunk has no second entry) so that both
        // evaluations are straight-line code the scheduler interleaves before
        // the short compositing chain (forward -5.7 % on config 3 against
        // evaluating the second entry under its own branch)
        while (bits) {
          const int k = c + __ffs(bits) - 1;
          bits &= bits - 1;
          const bool two = bits != 0u;
          const int kb = two ? c + __ffs(bits) - 1 : k;
          bits &= bits - 1;
          VG_ASSERT(k < nb && kb < nb);
          const F2 ea = eval_pinhole2<CUT>(sm[k], lx, ly, Lp, p.e2cut).ex;
          const F2 eb = eval_pinhole2<CUT>(sm[kb], lx, ly, Lp, p.e2cut).ex;
          composite_ex(k, sm[k].d, ea);
          if (two) composite_ex(kb, sm[kb].d, eb);
        }
      }
#if VG_SEEN_REDUX
      if (vmask) seen = __reduce_or_sync(FULL, seen);
#endif
      if (vmask && seen && lane == 0) {
        // record (entry, warp) visibility for the backward: bit g of this warp's row
        const uint32_t g = base + c;
        uint32_t* row = vmask + (size_t)warp * vm_words + (g >> 5);
        const uint32_t sh = g & 31u;
        VG_ASSERT((int)(g >> 5) + (sh ? 1 : 0) < vm_words);
        atomicOr(row, seen << sh);
        if (sh) atomicOr(row + 1, seen >> (32u - sh));
      }
      if (STATS) st_tot += min(32, nb - c);
      if (STOP) done = !(lo(T) >= p.stop) && !(hi(T) >= p.stop);
    }
#if VG_CTA_LOG
    w_walk += clock64() - c1;
#endif
  }
#if VG_CTA_LOG
  if (p.dbg_cta && lane == 0 && (int)blockIdx.x < p.dbg_cta_n) {
    p.dbg_cta[VG_CTA_LOG_STRIDE * (size_t)blockIdx.x + 3 + warp] = w_walk;
    p.dbg_cta[VG_CTA_LOG_STRIDE * (size_t)blockIdx.x + 7 + warp] = w_stage;
  }
#endif
  if (STATS && lane == 0) {
    atomicAdd(&g_vg_stats[0], st_proc);
    atomicAdd(&g_vg_stats[1], st_vis);
    atomicAdd(&g_vg_stats[2], st_tot);
  }
  if (VG_CTA_LOG) cta_log_end(p, tile);
  if (seg.counts && threadIdx.x == 0) {
    // this view's depth statistics (the next view's decision: seg_publish)
    const uint32_t d = min(base, r.y) - r.x;
    unsigned long long* st = reinterpret_cast<unsigned long long*>(seg.counts + SEG_STATS);
    atomicAdd(st, (unsigned long long)d);
    atomicMax(st + 1, (unsigned long long)d);
  }
  if (seg.on && threadIdx.x == 0) {
    // this tile's backward items (a tile that walked nothing still gets its
    // item: the pixel terms)
    const uint32_t d = min(base, r.y) - r.x;
    const uint32_t t = order[blockIdx.x];
    uint32_t ns = d > seg.thr ? (d + VG_SEG - 1) / VG_SEG : 1u;
    if (ns > 1 && atomicAdd(seg.counts + SEG_BINS, ns - 1) + (ns - 1) > seg.budget) ns = 1;
    if (ns == 1) {
      const int b = seg_bin(d);
      const uint32_t o = atomicAdd(seg.counts + b, 1u);
      seg.items[(size_t)b * seg.cap + o] = make_uint2(t, SEG_WHOLE);
    } else {
      for (uint32_t k = 0; k < ns; ++k) {
        const int b = seg_bin(min((uint32_t)VG_SEG, d - k * VG_SEG));
        const uint32_t o = atomicAdd(seg.counts + b, 1u);
        seg.items[(size_t)b * seg.cap + o] = make_uint2(t, k);
      }
    }
  }
  const int len = (int)(r.y - r.x);
  if (!STOP || lo(T) >= p.stop) na0 = len;
  if (!STOP || hi(T) >= p.stop) na1 = len;
  const float t0 = lo(T), t1 = hi(T);
  if (G.in0) {
    const int pix = G.row0 * p.width + G.col;
    color[3 * pix + 0] = fmaf(t0, p.bg[0], lo(Cr));
    color[3 * pix + 1] = fmaf(t0, p.bg[1], lo(Cg));
    color[3 * pix + 2] = fmaf(t0, p.bg[2], lo(Cb));
    final_t[pix] = t0;
    if (COUNTS) {
      n_contrib[pix] = nc0;
      n_act[pix] = na0;
    }
  }
  if (G.in1) {
    const int pix = G.row1 * p.width + G.col;
    color[3 * pix + 0] = fmaf(t1, p.bg[0], hi(Cr));
    color[3 * pix + 1] = fmaf(t1, p.bg[1], hi(Cg));
    color[3 * pix + 2] = fmaf(t1, p.bg[2], hi(Cb));
    final_t[pix] = t1;
    if (COUNTS) {
      n_contrib[pix] = nc1;
      n_act[pix] = na1;
    }
  }
}

#endif  // VG_TU_FWD

#if VG_TU_REST
// ---------------------------------------------------------------------------
// per-pair gradient terms (shared by the render and cone-beam backward):
// fills v[0..9] with the two pixels' sum of h (rho rho^T + w^ w^T), h rho, h.
// With s = D / |w|^2, rho = s (-w_par q1, -w_par q2, X), w^ = (q1, q2, w_par)/|w|:
//   A11 = q1^2 k1, A12 = q1 k1 q2, A22 = k1 q2^2, A13 = q1 k2, A23 = k2 q2,
//   A33 = h (s^2 X^2 + w_par^2 / |w|^2),  k1 = h (s^2 w_par^2 + 1/|w|^2),
//   k2 = h w_par (1/|w|^2 - s^2 X); q1 is shared by the lane's two pixels.

__device__ __forceinline__ void pinhole_grad_terms(const Pair2& e, const SRec& s, F2 h,
                                                   float (&v)[16]) {
  const F2 ri = mul2(e.rs, e.rs);
  const F2 sD = mul2(f2s(s.c.z), ri);
  const F2 s2 = mul2(sD, sD);
  const F2 wp2 = mul2(e.wp, e.wp);
  const F2 k1 = mul2(h, fma2(s2, wp2, ri));
  const F2 hw = mul2(h, e.wp);
  const F2 k2 = mul2(hw, fma2(neg2(s2), e.X, ri));
  const F2 k1q2 = mul2(k1, e.q2);
  const float q1 = e.q1;
  v[0] = q1 * q1 * hsum(k1);
  v[1] = q1 * hsum(k1q2);
  v[2] = q1 * hsum(k2);
  v[3] = hsum(mul2(k1q2, e.q2));
  v[4] = hsum(mul2(k2, e.q2));
  v[5] = hsum(mul2(h, fma2(s2, mul2(e.X, e.X), mul2(ri, wp2))));
  const F2 hs = mul2(h, sD);
  const F2 hsw = mul2(hs, e.wp);
  v[6] = -q1 * hsum(hsw);
  v[7] = -hsum(mul2(hsw, e.q2));
  v[8] = hsum(mul2(hs, e.X));
  v[9] = hsum(h);
}

// Deterministic mode: slot idx of the per-(entry, warp) partials (the caller
// numbers them: compact -- running count of visible pairs -- or pos * 4 + warp).
__device__ __forceinline__ float* det_slot(const BwdIO& io, size_t idx) {
  return io.det_part + idx * ACC_STRIDE;
}

// One entry of the backward replay for the lane's two pixels (shared by the
// staged and the warp-independent kernels): recompute alpha exactly as the
// forward did, advance T and the running suffix, form dL/de for live pixels,
// and flush the warp's 13 accumulator sums for this Gaussian.
template <bool CUT, bool DET>
__device__ __forceinline__ void bwd_entry(const SRec& s, const Pair2& e, bool in0, bool in1,
                                          F2 dcr, F2 dcg, F2 dcb, F2 tot, const BlendParams& p,
                                          F2& T, F2& P, int lane, const BwdIO& io, size_t pos,
                                          float* wb) {
  // active iff the replayed transmittance in front is >= stop (raster.py:384-385),
  // bit-identical to the forward's; inactive entries get a floor of 1 (no
  // change), cut ones (raster.py:363-365) the factor 1 from eval_pinhole2
  const bool act0 = in0 && lo(T) >= p.stop, act1 = in1 && hi(T) >= p.stop;
  const float om0 = fmaxf(lo(e.ex), act0 ? p.cc : 1.f);
  const float om1 = fmaxf(hi(e.ex), act1 ? p.cc : 1.f);
  const F2 om = f2(om0, om1);
  const F2 contrib = mul2(sub2(f2s(1.f), om), T);
  const F2 Tn = mul2(T, om);
  const F2 dot = fma2(dcr, f2s(s.d.x), fma2(dcg, f2s(s.d.y), mul2(dcb, f2s(s.d.z))));
  P = fma2(dot, contrib, P);
  T = Tn;
  // live: active, not cut (CUT: om < 1), not clamped (alpha_raw < clamp <=>
  // exp(-e) > 1 - clamp); without a cut an active alpha = 0 entry is live
  // (theta = 0 still has a kappa gradient, grad.py:150-160)
  const bool live0 = (CUT ? om0 < 1.f : act0) && lo(e.ex) > p.cc;
  const bool live1 = (CUT ? om1 < 1.f : act1) && hi(e.ex) > p.cc;
  const bool vis = om0 < 1.f || om1 < 1.f;
  const bool any_live = __any_sync(FULL, live0 || live1);
  const bool any_vis = __any_sync(FULL, vis);
  if (!(any_live || any_vis)) return;
  float v[16];
  if (any_live) {
    const F2 de = sel2(live0, live1, fma2(dot, Tn, sub2(P, tot)), f2s(0.f));
    pinhole_grad_terms(e, s, mul2(de, e.G), v);
  } else {
#pragma unroll
    for (int q = 0; q < 10; ++q) v[q] = 0.f;
  }
  v[10] = hsum(mul2(contrib, dcr));
  v[11] = hsum(mul2(contrib, dcg));
  v[12] = hsum(mul2(contrib, dcb));
  v[13] = v[14] = v[15] = 0.f;
  const uint32_t gid = __float_as_uint(s.c.w);
  if (lane == 0 && any_vis) io.visible[gid] = 1;
#if VG_SMEM_RED
  if (DET)
    flush_det_smem(v, lane, det_slot(io, pos), wb);
  else
    flush_acc_smem(v, lane, gid, io.acc, wb);
#else
  if (DET)
    flush_det(v, lane, det_slot(io, pos));
  else
    flush_acc(v, lane, gid, io.acc);
#endif
}

// Two consecutive visible entries: both replays first (the sequential
// transmittance chain), then both entries' gradient terms (independent
// math the scheduler can interleave), then the two flushes.
struct Replay {
  F2 h, contrib;
  bool flush, any_vis;
};

template <bool CUT>
__device__ __forceinline__ Replay bwd_replay(const SRec& s, const Pair2& e, bool in0, bool in1, F2 dcr,
                                             F2 dcg, F2 dcb, F2 tot, const BlendParams& p, F2& T,
                                             F2& P) {
  const bool act0 = in0 && lo(T) >= p.stop, act1 = in1 && hi(T) >= p.stop;
  const float om0 = fmaxf(lo(e.ex), act0 ? p.cc : 1.f);
  const float om1 = fmaxf(hi(e.ex), act1 ? p.cc : 1.f);
  const F2 om = f2(om0, om1);
  Replay r;
  r.contrib = mul2(sub2(f2s(1.f), om), T);
  const F2 Tn = mul2(T, om);
  const F2 dot = fma2(dcr, f2s(s.d.x), fma2(dcg, f2s(s.d.y), mul2(dcb, f2s(s.d.z))));
  P = fma2(dot, r.contrib, P);
  T = Tn;
  const bool live0 = (CUT ? om0 < 1.f : act0) && lo(e.ex) > p.cc;
  const bool live1 = (CUT ? om1 < 1.f : act1) && hi(e.ex) > p.cc;
  r.h = mul2(sel2(live0, live1, fma2(dot, Tn, sub2(P, tot)), f2s(0.f)), e.G);
  r.any_vis = __any_sync(FULL, om0 < 1.f || om1 < 1.f);
  r.flush = r.any_vis || __any_sync(FULL, live0 || live1);
  return r;
}

template <bool DET>
__device__ __forceinline__ void bwd_flush(const SRec& s, const Replay& r, float (&v)[16], int lane,
                                          const BwdIO& io, size_t pos, float* wb) {
  if (!r.flush) return;
  const uint32_t gid = __float_as_uint(s.c.w);
  if (lane == 0 && r.any_vis) io.visible[gid] = 1;
  if (DET)
    flush_det_smem(v, lane, det_slot(io, pos), wb);
  else
    flush_acc_smem(v, lane, gid, io.acc, wb);
}

template <bool CUT, bool DET>
__device__ __forceinline__ void bwd_entry2(const SRec& sa, const Pair2& ea, const SRec& sb,
                                           const Pair2& eb, bool in0, bool in1, F2 dcr, F2 dcg, F2 dcb,
                                           F2 tot, const BlendParams& p, F2& T, F2& P, int lane,
                                           const BwdIO& io, size_t pa, size_t pb, float* wb) {
  const Replay ra = bwd_replay<CUT>(sa, ea, in0, in1, dcr, dcg, dcb, tot, p, T, P);
  const Replay rb = bwd_replay<CUT>(sb, eb, in0, in1, dcr, dcg, dcb, tot, p, T, P);
  float va[16], vb[16];
  pinhole_grad_terms(ea, sa, ra.h, va);
  pinhole_grad_terms(eb, sb, rb.h, vb);
  va[10] = hsum(mul2(ra.contrib, dcr));
  va[11] = hsum(mul2(ra.contrib, dcg));
  va[12] = hsum(mul2(ra.contrib, dcb));
  vb[10] = hsum(mul2(rb.contrib, dcr));
  vb[11] = hsum(mul2(rb.contrib, dcg));
  vb[12] = hsum(mul2(rb.contrib, dcb));
#if VG_BWD_PAIR == 2
  // one shared-memory pass for both entries (all-zero sums are not stored)
  if (!(ra.flush || rb.flush)) return;
  const uint32_t ga = __float_as_uint(sa.c.w), gb = __float_as_uint(sb.c.w);
  VG_ASSERT((int64_t)ga < p.dbg_n && (int64_t)gb < p.dbg_n);
  if (lane == 0 && ra.any_vis) io.visible[ga] = 1;
  if (lane == 0 && rb.any_vis) io.visible[gb] = 1;
  const F2 xs = smem_reduce13x2p(va, vb, lane, wb);
  const float xa = lo(xs), xb = hi(xs);
  if (DET) {
    // every value is stored (slots are not pre-zeroed), the 3 pad floats too:
    // whole 32-byte sectors, so L2 never holds partially written slot lines
    if (lane < ACC_STRIDE) {
      det_slot(io, pa)[lane] = lane < 13 ? xa : 0.f;
      det_slot(io, pb)[lane] = lane < 13 ? xb : 0.f;
    }
  } else if (lane < 13) {
    const int q = lane;
    {
      // unconditional: a zero test per value costs more than the rare zero add
      atomicAdd(io.acc + (size_t)ga * ACC_STRIDE + q, xa);
      atomicAdd(io.acc + (size_t)gb * ACC_STRIDE + q, xb);
    }
  }
#else
  bwd_flush<DET>(sa, ra, va, lane, io, pa, wb);
  bwd_flush<DET>(sb, rb, vb, lane, io, pb, wb);
#endif
}

// ---------------------------------------------------------------------------
// K6 backward blend (grad.backward tile_job + e_chain)

template <bool CUT, int LOSS, bool DET = false>
__global__ void __launch_bounds__(NT, VG_BWD_MINB) k_render_bwd(const GRec* __restrict__ rec,
                                                   const uint32_t* __restrict__ vals,
                                                   const uint2* __restrict__ ranges,
                                                   const uint32_t* __restrict__ order,
                                                   BlendParams p, BwdIO io,
                                                   const uint32_t* __restrict__ vmask,
                                                   int vm_words, SegIO seg) {
  cta_log_begin(p);
  __shared__ SRec sm[BATCH];
  __shared__ uint8_t smask[BATCH];
  __shared__ __align__(16) float sred[NT / 32][VG_BWD_PAIR == 2 ? (REDP_WORDS > RED_WORDS ? REDP_WORDS : RED_WORDS)
                                               : VG_SMEM_RED ? RED_WORDS : 4];
  // segmented: item = (tile, segment k), entries [r.x + k VG_SEG, + VG_SEG)
  int tile;
  uint32_t ks = SEG_WHOLE;
  if (!DET && seg.on) {
    // CTA b -> the (b - items of the bins before)-th item of its bin; per
    // warp: lane q holds bin q's count, a shuffle scan, a ballot
    static_assert(SEG_BINS == 32, "one bin per lane");
    const int ln = threadIdx.x & 31;
    const uint32_t cq = __ldcg(seg.counts + ln);
    uint32_t inc = cq;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(FULL, inc, o);
      if (ln >= o) inc += y;
    }
    const unsigned past = __ballot_sync(FULL, inc <= blockIdx.x);  // bins wholly before b
    const int bin = __popc(past);
    if (bin == SEG_BINS) return;
    const uint32_t before = __shfl_sync(FULL, inc - cq, bin);
    uint2 it = make_uint2(0u, 0u);
    if (ln == 0) it = __ldcg(seg.items + (size_t)bin * seg.cap + (blockIdx.x - before));
    tile = (int)__shfl_sync(FULL, it.x, 0);
    ks = __shfl_sync(FULL, it.y, 0);
  } else {
    tile = order[blockIdx.x];
  }
  const int tx = tile % p.ntx, ty = tile / p.ntx;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* wb = sred[warp];
  const LaneGeo G = lane_geo(p, tx, ty);
  const float lx = (float)G.lxi;
  const F2 ly = f2((float)G.ly0, (float)(G.ly0 + 4));
  const F2 Lp = f2(pixel_lp(p, G.col, G.row0), pixel_lp(p, G.col, G.row1));
  uint2 r = ranges[tile];
  float dcv[2][3], totv[2];
  // the per-pixel d_background / loss terms: once per tile (its first segment)
  bwd_prologue<LOSS, DET>(p, G, io, dcv, totv, tile, (ks & ~SEG_WHOLE) == 0);
  const F2 dcr = f2(dcv[0][0], dcv[1][0]), dcg = f2(dcv[0][1], dcv[1][1]),
           dcb = f2(dcv[0][2], dcv[1][2]);
  const F2 tot = f2(totv[0], totv[1]);
  // the replay follows the forward exactly: same entries, same order, same
  // transmittance (so the same activity and the same early exits)
  F2 T = f2(G.in0 ? 1.f : 0.f, G.in1 ? 1.f : 0.f), P = f2s(0.f);
  if (!DET && seg.on && !(ks & SEG_WHOLE)) {
    const uint32_t s0 = r.x + ks * (uint32_t)VG_SEG;
    r = make_uint2(s0, min(r.y, s0 + (uint32_t)VG_SEG));
    if (ks) {
      // the forward's transmittance at the boundary (bit-identical to the
      // sequential replay) and the dot-weighted colour in front of it
      const float4* o = seg.state + ((size_t)(s0 / VG_SEG) * NT + threadIdx.x) * 2;
      const float4 a = o[0], b = o[1];
      T = f2(a.x, a.y);
      P = fma2(dcr, f2(a.z, a.w), fma2(dcg, f2(b.x, b.y), mul2(dcb, f2(b.z, b.w))));
    }
  }
  bool done = !(G.in0 && lo(T) >= p.stop) && !(G.in1 && hi(T) >= p.stop);
  // Gaussian-major slots: the staging put entry k's (Gaussian, tile) index in sm[k].d.w
  auto dslot = [&](uint32_t pos, const SRec& s, int k) -> size_t {
    if (!DET) return 0;
    VG_ASSERT((int64_t)pos < p.dbg_pairs);
    if (io.det_gvis4) return (size_t)__float_as_uint(s.d.w) * (NT / 32) + warp;
    return (size_t)pos * (NT / 32) + warp;
  };
  const uint32_t* vrow = vmask ? vmask + (size_t)warp * vm_words : nullptr;
  VG_ASSERT(r.x <= r.y && (int64_t)r.y <= p.dbg_pairs);
  for (uint32_t base = r.x; base < r.y; base += BATCH) {
    VG_JITTER(p.dbg_jitter, base);
    if (__syncthreads_count(done) == NT) break;
    for (int sidx = threadIdx.x; sidx < BATCH; sidx += NT) {
      const uint32_t i = base + sidx;
      if (i < r.y) {
        const uint32_t m = stage(sm, sidx, rec, chk_gid(p, vals[i]), tx * TILE, ty * TILE, CUT && !vmask, p.ecut);
        if (!vmask) smask[sidx] = (uint8_t)m;
        if (DET && io.det_gvis4) {
          // this entry's (Gaussian, tile) index within the Gaussian's tile
          // rectangle (row-major) and its four warp-visibility bits
          const uint32_t gid = __float_as_uint(sm[sidx].c.w);
          const ushort4 q = io.det_rect[gid];
          const uint32_t ps = io.det_off[gid] + (uint32_t)(ty - q.y) * (uint32_t)(q.z - q.x + 1) +
                              (uint32_t)(tx - q.x);
          VG_ASSERT((int64_t)ps < p.dbg_pairs);
          sm[sidx].d.w = __uint_as_float(ps);
          uint32_t v = 0;
#pragma unroll
          for (int w = 0; w < NT / 32; ++w)
            v |= ((__ldg(vmask + (size_t)w * vm_words + (i >> 5)) >> (i & 31u)) & 1u) << w;
          io.det_gvis4[ps] = (uint8_t)v;
        }
      }
    }
    __syncthreads();
    const int nb = min((uint32_t)BATCH, r.y - base);
    for (int c = 0; c < nb && !__all_sync(FULL, done); c += 32) {
      VG_JITTER(p.dbg_jitter, base + c + 1);
      unsigned bits;
      if (vmask) {
        // exact: the entries where the forward saw a visible pixel in this block
        // lane l tests entry base + c + l; the ballot makes the mask
        // warp-uniform for the compiler (uniform bit scan and loop, no
        // divergence bookkeeping: backward -6 % on config 3, -12 % on config 4
        // against extracting the 32 bits from the mask words per lane)
        const uint32_t g = base + c + lane;
        const uint32_t vw = __ldg(vrow + (g >> 5));
        const bool vb = (c + lane < nb) && ((vw >> (g & 31u)) & 1u);
        bits = __ballot_sync(FULL, vb);
      } else {
        const bool vb = (c + lane < nb) && ((smask[c + lane] >> warp) & 1);
        bits = __ballot_sync(FULL, vb);
      }
      // two visible entries per iteration: both alpha evaluations are
      // issued before the replay chain of the first
      while (bits) {
        const int k = c + __ffs(bits) - 1;
        bits &= bits - 1;
        VG_ASSERT(k < nb);
        const SRec s = sm[k];
        const Pair2 e = eval_pinhole2<CUT>(s, lx, ly, Lp, p.e2cut);
        if (bits) {
          const int kb = c + __ffs(bits) - 1;
          bits &= bits - 1;
          VG_ASSERT(kb < nb);
          const SRec sb = sm[kb];
          const Pair2 eb = eval_pinhole2<CUT>(sb, lx, ly, Lp, p.e2cut);
#if VG_BWD_PAIR
          const size_t ia = dslot(base + k, s, k);
          const size_t ib = dslot(base + kb, sb, kb);
          bwd_entry2<CUT, DET>(s, e, sb, eb, G.in0, G.in1, dcr, dcg, dcb, tot, p, T, P, lane, io,
                               ia, ib, wb);
#else
          const size_t ia = dslot(base + k, s, k);
          bwd_entry<CUT, DET>(s, e, G.in0, G.in1, dcr, dcg, dcb, tot, p, T, P, lane, io, ia, wb);
          const size_t ib = dslot(base + kb, sb, kb);
          bwd_entry<CUT, DET>(sb, eb, G.in0, G.in1, dcr, dcg, dcb, tot, p, T, P, lane, io, ib, wb);
#endif
        } else {
          const size_t ia = dslot(base + k, s, k);
          bwd_entry<CUT, DET>(s, e, G.in0, G.in1, dcr, dcg, dcb, tot, p, T, P, lane, io, ia, wb);
        }
      }
      done = !(G.in0 && lo(T) >= p.stop) && !(G.in1 && hi(T) >= p.stop);
    }
  }
  if (VG_CTA_LOG) cta_log_end(p, tile);
}

// ---------------------------------------------------------------------------
// K8 tomography (tomo.tomo_forward / tomo_backward): order-independent sum
// of e over every binned pair; no cut, clamp or early stop (tomo.py:43-47).

template <int RAY>
__global__ void __launch_bounds__(NT) k_tomo_fwd(const GRec* __restrict__ rec,
                                                 const uint32_t* __restrict__ vals,
                                                 const uint2* __restrict__ ranges,
                                                 const uint32_t* __restrict__ order,
                                                 BlendParams p, float* __restrict__ image,
                                                 float* __restrict__ intensity,
                                                 float* __restrict__ part) {
  __shared__ SRec sm[BATCH];
  const int tile = order[blockIdx.x];
  const int split = blockIdx.y, S = gridDim.y;
  const int tx = tile % p.ntx, ty = tile / p.ntx;
  const LaneGeo G = lane_geo(p, tx, ty);
  const float lx = (float)G.lxi;
  const F2 ly = f2((float)G.ly0, (float)(G.ly0 + 4));
  const F2 Lp = RAY == VG_PINHOLE ? f2(pixel_lp(p, G.col, G.row0), pixel_lp(p, G.col, G.row1))
                                  : f2s(0.f);
  const uint2 r = ranges[tile];
  F2 sum = f2s(0.f);
  // split s walks batches s, s + S, ... of the tile's list
  for (uint32_t base = r.x + split * BATCH; base < r.y; base += BATCH * S) {
    __syncthreads();
    for (int sidx = threadIdx.x; sidx < BATCH; sidx += NT) {
      uint32_t i = base + sidx;
      if (i < r.y) stage(sm, sidx, rec, vals[i], tx * TILE, ty * TILE, false, 0.f);
    }
    __syncthreads();
    const int nb = min((uint32_t)BATCH, r.y - base);
    for (int k = 0; k < nb; ++k) {
      const SRec s = sm[k];
      const Pair2 e = RAY == VG_PINHOLE ? eval_pinhole2(s, lx, ly, Lp) : eval_parallel2(s, lx, ly);
      sum = add2(sum, e.E2);
    }
  }
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const bool in = q ? G.in1 : G.in0;
    if (!in) continue;
    const int pix = (q ? G.row1 : G.row0) * p.width + G.col;
    if (S > 1) {
      part[(size_t)split * p.width * p.height + pix] = q ? hi(sum) : lo(sum);
      continue;
    }
    const float I = (q ? hi(sum) : lo(sum)) * (float)LN2;
    image[pix] = I;
    if (intensity) intensity[pix] = __expf(-I);
  }
}

// Parallel-beam projector with a row recurrence (VG_TOMO_REC; the default --
// config 5 projector 20.3 -> 16.0 ms over 45 views).  For parallel
// rays the exponent along a tile column is a quadratic in the row index y,
//   e(y) = -C (q1^2 + (A + B y)^2),  C = log2(e) / 2,
// so h(y) = 2^e(y) obeys h(y+1) = h(y) r(y), r(y+1) = r(y) k with
// k = 2^(-2 C B^2): four exp2 per entry and column (two anchors at rows 7 and
// 8, one ratio each way, k) instead of sixteen, each sweep running from the
// middle outwards.  An anchor far in the tail (e < -100) while the column
// still reaches 2^-60 falls back to exp2 per pixel (narrow Gaussians); columns
// that never reach 2^VG_TOMO_SKIP = 2^-60 of the peak are skipped.
// Thread t owns column t & 15 for list entries = t >> 4 (mod 8); the eight
// partial columns are summed in a fixed order at the end.
__global__ void __launch_bounds__(NT) k_tomo_fwd_rec(const GRec* __restrict__ rec,
                                                     const uint32_t* __restrict__ vals,
                                                     const uint2* __restrict__ ranges,
                                                     const uint32_t* __restrict__ order,
                                                     BlendParams p, float* __restrict__ image,
                                                     float* __restrict__ intensity,
                                                     float* __restrict__ part) {
  __shared__ SRec sm[BATCH];
  __shared__ float sacc[NT / TILE][TILE_PIX];
  const int tile = order[blockIdx.x];
  const int split = blockIdx.y, S = gridDim.y;
  const int tx = tile % p.ntx, ty = tile / p.ntx;
  const int col = threadIdx.x & (TILE - 1), slice = threadIdx.x / TILE;
  constexpr int NSL = NT / TILE;  // 8 entry slices
  const float x = (float)col;
  const uint2 r = ranges[tile];
  F2 acc2[TILE / 2];
#pragma unroll
  for (int i = 0; i < TILE / 2; ++i) acc2[i] = f2s(0.f);
  for (uint32_t base = r.x + split * BATCH; base < r.y; base += BATCH * S) {
    __syncthreads();
    for (int sidx = threadIdx.x; sidx < BATCH; sidx += NT) {
      uint32_t i = base + sidx;
      if (i < r.y) stage(sm, sidx, rec, vals[i], tx * TILE, ty * TILE, false, 0.f);
    }
    __syncthreads();
    const int nb = min((uint32_t)BATCH, r.y - base);
    for (int k = slice; k < nb; k += NSL) {
      const SRec s = sm[k];
      const float q1 = fmaf(s.b.x, x, s.a.x);
      const float A = fmaf(s.b.y, x, s.a.y);
      const float B = s.b.z;
      const float amp = s.c.z * s.b.w;  // E2 = amp * 2^e
      const float q11 = q1 * q1;
      // column maximum of e: (A + B y)^2 smallest at y* = -A / B, clamped to the column
      const float ys = B != 0.f ? fminf(fmaxf(__fdividef(-A, B), 0.f), (float)(TILE - 1)) : 0.f;
      const float zs = fmaf(B, ys, A);
      const float emax = -C_HALF_LOG2E * fmaf(zs, zs, q11);
      if (!(emax > VG_TOMO_SKIP)) continue;  // below 2^VG_TOMO_SKIP of the peak everywhere here
      const float z7 = fmaf(B, 7.f, A), z8 = fmaf(B, 8.f, A);
      const float e7 = -C_HALF_LOG2E * fmaf(z7, z7, q11);
      const float e8 = -C_HALF_LOG2E * fmaf(z8, z8, q11);
      if (e7 < -100.f || e8 < -100.f) {
        // anchors in the tail of a narrow Gaussian: direct evaluation
#pragma unroll
        for (int i = 0; i < TILE / 2; ++i) {
          const float zu = fmaf(B, (float)(8 + i), A), zd = fmaf(B, (float)(7 - i), A);
          acc2[i] = fma2(f2s(amp), f2(ex2f(-C_HALF_LOG2E * fmaf(zu, zu, q11)),
                                      ex2f(-C_HALF_LOG2E * fmaf(zd, zd, q11))), acc2[i]);
        }
        continue;
      }
      const float kk = ex2f(-2.f * C_HALF_LOG2E * B * B);
      // both sweeps at once in packed FP32x2: lo walks rows 8..15 from
      // h(8) with h(9)/h(8) = 2^(-C B (2 z8 + B)), hi walks rows 7..0 from
      // h(7) with h(6)/h(7) = 2^(C B (2 z7 - B)); accumulator pair i holds
      // rows (8 + i, 7 - i)
      F2 h = f2(ex2f(e8), ex2f(e7));
      F2 rr = f2(ex2f(-C_HALF_LOG2E * B * fmaf(2.f, z8, B)), ex2f(C_HALF_LOG2E * B * fmaf(2.f, z7, -B)));
      const F2 k2 = f2s(kk), a2 = f2s(amp);
#pragma unroll
      for (int i = 0; i < TILE / 2; ++i) {
        acc2[i] = fma2(a2, h, acc2[i]);
        h = mul2(h, rr);
        rr = mul2(rr, k2);
      }
    }
  }
  // fixed-order sum of the eight slices
#pragma unroll
  for (int i = 0; i < TILE / 2; ++i) {
    sacc[slice][(8 + i) * TILE + col] = lo(acc2[i]);
    sacc[slice][(7 - i) * TILE + col] = hi(acc2[i]);
  }
  __syncthreads();
  for (int q = threadIdx.x; q < TILE_PIX; q += NT) {
    float sum = 0.f;
#pragma unroll
    for (int sl = 0; sl < NSL; ++sl) sum += sacc[sl][q];
    const int c = tx * TILE + (q & (TILE - 1)), rw = ty * TILE + q / TILE;
    if (c >= p.width || rw >= p.height) continue;
    const int pix = rw * p.width + c;
    if (S > 1) {
      part[(size_t)split * p.width * p.height + pix] = sum;
      continue;
    }
    const float I = sum * (float)LN2;
    image[pix] = I;
    if (intensity) intensity[pix] = __expf(-I);
  }
}

// Sum of the per-split partial images in split order (deterministic).
__global__ void k_tomo_combine(int npix, int S, const float* __restrict__ part, float* __restrict__ image,
                               float* __restrict__ intensity) {
  const int pix = blockIdx.x * blockDim.x + threadIdx.x;
  if (pix >= npix) return;
  float sum = 0.f;
  for (int s = 0; s < S; ++s) sum += part[(size_t)s * npix + pix];
  const float I = sum * (float)LN2;
  image[pix] = I;
  if (intensity) intensity[pix] = __expf(-I);
}

// Tomography adjoint, Gaussian-parallel.  The line-integral sum has no
// ordering (tomo.py:43-47), so instead of a warp per pixel block (which needs
// a 13-value warp reduction for every pair) each thread owns one
// (Gaussian, tile) pair and walks the tile's 256 pixels -- d_image staged once
// per tile in shared memory and read as a broadcast -- accumulating its 10
// gradient sums in registers; one 10-lane-op atomic flush per pair.
template <int RAY, int LOSS, bool DET = false>
__global__ void __launch_bounds__(NT) k_tomo_bwd(const GRec* __restrict__ rec,
                                                 const uint32_t* __restrict__ vals,
                                                 const uint2* __restrict__ ranges,
                                                 const uint32_t* __restrict__ order,
                                                 BlendParams p, const float* __restrict__ d_image,
                                                 const float* __restrict__ image,
                                                 const float* __restrict__ target,
                                                 float loss_scale, double* loss_sum,
                                                 float* __restrict__ acc,
                                                 uint8_t* __restrict__ visible,
                                                 float* __restrict__ det_part,
                                                 double* __restrict__ det_loss) {
  __shared__ float sde[TILE_PIX];
  __shared__ float slp[TILE_PIX];
  const int tile = order[blockIdx.x];
  const int split = blockIdx.y, S = gridDim.y;
  const int tx = tile % p.ntx, ty = tile / p.ntx;
  const uint2 r = ranges[tile];
  double lossv = 0.0;
  for (int q = threadIdx.x; q < TILE_PIX; q += NT) {
    const int col = tx * TILE + (q & 15), row = ty * TILE + (q >> 4);
    float de = 0.f;
    if (col < p.width && row < p.height) {
      const int pix = row * p.width + col;
      if (LOSS == 0) {
        de = d_image[pix];
      } else {
        const float rr = image[pix] - target[pix];
        lossv += (double)rr * rr;
        de = loss_scale * rr;
      }
    }
    sde[q] = de;
    slp[q] = RAY == VG_PINHOLE ? pixel_lp(p, col, row) : 0.f;
  }
  // deterministic mode: this tile's loss partial, summed in tile order later
  if (LOSS && split == 0) block_flush(0.f, 0.f, 0.f, lossv, nullptr, DET ? det_loss + tile : loss_sum, DET);
  __syncthreads();
  // split s owns pairs r.x + s NT + thread, stepping NT S: one thread per pair
  {
    for (uint32_t i = r.x + split * NT + threadIdx.x; i < r.y; i += NT * S) {
      const uint32_t gi = vals[i];
      const SRec s = make_srec(rec[gi], gi, tx * TILE, ty * TILE);
      float vv[10];
      float gsum;
      if constexpr (RAY != VG_PINHOLE && VG_TOMO_MOM) {
        // Parallel rays, moment form: q1, q2 are affine in the pixel offset, so
        // the six sums need only the moments of h = d G over the tile in
        // coordinates centred on the Gaussian's nearest pixel (u = x - xc,
        // v = y - yc: the affine constants stay small, no cancellation).
        // Per pixel: R0 += h, R1 += h u, R2 += h u^2 along the row; per row
        // the six moments.  13 instead of 17 packed ops per two pixels.
        const float P11 = s.b.x, P21 = s.b.y, P22 = s.b.z, A1 = s.a.x, C2 = s.a.y;
        const float xs = P11 != 0.f ? __fdividef(-A1, P11) : 0.f;
        const float xc = fminf(fmaxf(rintf(xs), 0.f), (float)(TILE - 1));
        const float ys = P22 != 0.f ? __fdividef(-fmaf(P21, xc, C2), P22) : 0.f;
        const float yc = fminf(fmaxf(rintf(ys), 0.f), (float)(TILE - 1));
        const float al = fmaf(P11, xc, A1);                 // q1 = P11 u + al
        const float ga = fmaf(P22, yc, fmaf(P21, xc, C2));  // q2 = P21 u + P22 v + ga
        const F2 bx = f2s(P11), by = f2s(P21), ax = f2s(al), nch = f2s(-C_HALF_LOG2E);
        const F2 cz = f2s(s.c.z);
        F2 gs = f2s(0.f);
        float M0 = 0.f, Mu = 0.f, Mv = 0.f, Muu = 0.f, Muv = 0.f, Mvv = 0.f;
        for (int ly = 0; ly < TILE; ++ly) {
          const float v = (float)ly - yc;
          const F2 t2 = f2s(fmaf(P22, v, ga));
          F2 u = f2(-xc, 1.f - xc);
          F2 R0 = f2s(0.f), R1 = f2s(0.f), R2 = f2s(0.f);
#pragma unroll 4
          for (int lx = 0; lx < TILE; lx += 2) {
            F2 d;
            d.v = *reinterpret_cast<const unsigned long long*>(&sde[ly * TILE + lx]);
            const F2 q1 = fma2(bx, u, ax);
            const F2 q2 = fma2(by, u, t2);
            const F2 X = fma2(q1, q1, mul2(q2, q2));
            const F2 G = mul2(cz, ex2_2(mul2(nch, X)));
            gs = add2(gs, G);
            const F2 h = mul2(d, G);
            const F2 hu = mul2(h, u);
            R0 = add2(R0, h);
            R1 = add2(R1, hu);
            R2 = fma2(hu, u, R2);
            u = add2(u, f2s(2.f));
          }
          const float r0 = hsum(R0), r1 = hsum(R1), r2 = hsum(R2);
          M0 += r0;
          Mu += r1;
          Muu += r2;
          Mv = fmaf(v, r0, Mv);
          Muv = fmaf(v, r1, Muv);
          Mvv = fmaf(v * v, r0, Mvv);
        }
        gsum = hsum(gs);
        const float Sq1 = fmaf(P11, Mu, al * M0);                       // sum h q1
        const float Sq2 = fmaf(P21, Mu, fmaf(P22, Mv, ga * M0));        // sum h q2
        vv[0] = fmaf(P11 * P11, Muu, fmaf(2.f * P11 * al, Mu, al * al * M0));                 // h q1^2
        vv[1] = fmaf(P11, fmaf(P21, Muu, fmaf(P22, Muv, ga * Mu)), al * Sq2);                // h q1 q2
        vv[2] = 0.f;
        vv[3] = fmaf(P21 * P21, Muu, fmaf(P22 * P22, Mvv, fmaf(2.f * P21 * P22, Muv,
                fmaf(2.f * ga, fmaf(P21, Mu, P22 * Mv), ga * ga * M0))));                    // h q2^2
        vv[4] = 0.f;
        vv[5] = M0;
        vv[6] = -Sq1;
        vv[7] = -Sq2;
        vv[8] = 0.f;
        vv[9] = M0;
      } else {
        // two horizontally adjacent pixels per step in packed FP32x2; b0 / b1
        // accumulate with the opposite sign and are negated at the end
        const F2 zero = f2s(0.f);
        F2 a0 = zero, a1 = zero, a2 = zero, a3 = zero, a4 = zero, a5 = zero;
        F2 b0 = zero, b1 = zero, b2 = zero, hs = zero, gs = zero;
        const F2 bx = f2s(s.b.x), by = f2s(s.b.y), ax = f2s(s.a.x), cx = f2s(s.c.x);
        const F2 cz = f2s(s.c.z), naw = f2s(-s.a.w), nch = f2s(-C_HALF_LOG2E);
        for (int ly = 0; ly < TILE; ++ly) {
          const float fy = (float)ly;
          const F2 t2 = f2s(fmaf(s.b.z, fy, s.a.y));
          const F2 tw = f2s(fmaf(s.c.y, fy, s.a.z));
          F2 fx = f2(0.f, 1.f);
  #pragma unroll 4
          for (int lx = 0; lx < TILE; lx += 2) {
            F2 d;
            d.v = *reinterpret_cast<const unsigned long long*>(&sde[ly * TILE + lx]);
            const F2 q1 = fma2(bx, fx, ax);
            const F2 q2 = fma2(by, fx, t2);
            const F2 X = fma2(q1, q1, mul2(q2, q2));
            if (RAY == VG_PINHOLE) {
              F2 lp;
              lp.v = *reinterpret_cast<const unsigned long long*>(&slp[ly * TILE + lx]);
              const F2 wp = fma2(cx, fx, tw);
              const F2 rs = rsq_2(fma2(wp, wp, X));
              const F2 ri = mul2(rs, rs);
              const F2 G = mul2(rs, ex2_2(fma2(naw, mul2(X, ri), lp)));
              gs = add2(gs, G);
              const F2 h = mul2(d, G);
              // factored h (rho rho^T + w^ w^T), h rho (see pinhole_grad_terms)
              const F2 sD = mul2(cz, ri), s2 = mul2(sD, sD), wp2 = mul2(wp, wp);
              const F2 k1 = mul2(h, fma2(s2, wp2, ri));
              const F2 k2 = mul2(mul2(h, wp), sub2(ri, mul2(s2, X)));
              const F2 k1q1 = mul2(k1, q1);
              a0 = fma2(k1q1, q1, a0);
              a1 = fma2(k1q1, q2, a1);
              a2 = fma2(k2, q1, a2);
              a3 = fma2(mul2(k1, q2), q2, a3);
              a4 = fma2(k2, q2, a4);
              a5 = fma2(h, fma2(s2, mul2(X, X), mul2(ri, wp2)), a5);
              const F2 hsD = mul2(h, sD), hsw = mul2(hsD, wp);
              b0 = fma2(hsw, q1, b0);
              b1 = fma2(hsw, q2, b1);
              b2 = fma2(hsD, X, b2);
              hs = add2(hs, h);
            } else {
              const F2 G = mul2(cz, ex2_2(mul2(nch, X)));
              gs = add2(gs, G);
              const F2 h = mul2(d, G);
              // rho = -(q1, q2, 0), w^ = (0, 0, 1)
              const F2 hq1 = mul2(h, q1), hq2 = mul2(h, q2);
              a0 = fma2(hq1, q1, a0);
              a1 = fma2(hq1, q2, a1);
              a3 = fma2(hq2, q2, a3);
              b0 = add2(b0, hq1);
              b1 = add2(b1, hq2);
              hs = add2(hs, h);
            }
            fx = add2(fx, f2s(2.f));
          }
        }
        const float hsum_h = hsum(hs);
        gsum = hsum(gs);
        const float vv0[10] = {hsum(a0), hsum(a1), hsum(a2), hsum(a3), hsum(a4),
                               RAY != VG_PINHOLE ? hsum_h : hsum(a5), -hsum(b0), -hsum(b1), hsum(b2), hsum_h};
#pragma unroll
        for (int q = 0; q < 10; ++q) vv[q] = vv0[q];
      }
      const uint32_t gid = __float_as_uint(s.c.w);
      float* o = acc + (size_t)gid * ACC_STRIDE;
#pragma unroll
      if (DET) {
        // the pair's own slot (warp slot 0 of its list position; vg_det.cu)
        float* sl = det_part + (size_t)i * (NT / 32) * ACC_STRIDE;
#pragma unroll
        for (int q = 0; q < 10; ++q) sl[q] = vv[q];
      } else {
#pragma unroll
        for (int q = 0; q < 10; ++q)
          if (vv[q] != 0.f) atomicAdd(o + q, vv[q]);
      }
      if (gsum > 0.f && s.b.w > 0.f) visible[gid] = 1;
    }
  }
}

#endif  // VG_TU_REST

// ---------------------------------------------------------------------------
// launchers

#if VG_TU_FWD
void launch_render_fwd(int n_tiles, const GRec* rec, const uint32_t* vals, const uint2* ranges,
                       const uint32_t* order, const BlendParams& p, bool stop, bool cut,
                       float* color, float* final_t, int* n_contrib, int* n_act, uint32_t* vmask,
                       int vm_words, cudaStream_t st, const SegIO& seg) {
#if VG_CTA_LOG
  // profiling build: VG_FWD_GRID=k launches only the k heaviest tiles (load-balance experiments)
  if (const char* g = getenv("VG_FWD_GRID")) n_tiles = min(n_tiles, atoi(g));
#endif
  // n_contrib == NULL: the training-step forward (no counts)
#define VG_RF(S, C)                                                                             \
  do {                                                                                          \
    if (n_contrib)                                                                              \
      k_render_fwd<S, C, false, true><<<n_tiles, NT, 0, st>>>(rec, vals, ranges, order, p, color, \
                                                               final_t, n_contrib, n_act, vmask, \
                                                               vm_words, seg);                  \
    else                                                                                        \
      k_render_fwd<S, C, false, false><<<n_tiles, NT, 0, st>>>(rec, vals, ranges, order, p,      \
                                                                color, final_t, nullptr, nullptr, \
                                                                vmask, vm_words, seg);           \
  } while (0)
  if (stop && cut) VG_RF(true, true);
  else if (stop) VG_RF(true, false);
  else if (cut) VG_RF(false, true);
  else VG_RF(false, false);
#undef VG_RF
}

void launch_render_fwd_deep(int n_tiles, const GRec* rec, const uint32_t* vals, const uint2* ranges,
                            const uint32_t* order, const BlendParams& p, bool stop, bool cut,
                            float* color, float* final_t, uint32_t* vmask, int vm_words,
                            cudaStream_t st, const SegIO& seg) {
#define VG_RFD(S, C)                                                                              \
  k_render_fwd<S, C, false, false, true><<<n_tiles, NT, 0, st>>>(rec, vals, ranges, order, p,     \
                                                                  color, final_t, nullptr, nullptr, \
                                                                  vmask, vm_words, seg)
  if (stop && cut) VG_RFD(true, true);
  else if (stop) VG_RFD(true, false);
  else if (cut) VG_RFD(false, true);
  else VG_RFD(false, false);
#undef VG_RFD
}
#endif  // VG_TU_FWD

#if VG_TU_REST
void launch_render_bwd(int n_tiles, const GRec* rec, const uint32_t* vals, const uint2* ranges,
                       const uint32_t* order, const BlendParams& p, bool cut, int loss,
                       const BwdIO& io, const uint32_t* vmask, int vm_words, cudaStream_t st,
                       const SegIO& seg) {
  const bool det = io.det_part != nullptr;
  // segmented: seg.cap bounds the item count (surplus CTAs exit at once)
  const int nb = seg.on ? (int)seg.cap : n_tiles;
#define VG_RB(C, L, D) \
  k_render_bwd<C, L, D><<<nb, NT, 0, st>>>(rec, vals, ranges, order, p, io, vmask, vm_words, seg)
  if (det) {
    if (cut) {
      if (loss) VG_RB(true, 1, true); else VG_RB(true, 0, true);
    } else {
      if (loss) VG_RB(false, 1, true); else VG_RB(false, 0, true);
    }
  } else if (cut) {
    if (loss) VG_RB(true, 1, false); else VG_RB(true, 0, false);
  } else {
    if (loss) VG_RB(false, 1, false); else VG_RB(false, 0, false);
  }
#undef VG_RB
}

void launch_tomo_fwd(int n_tiles, int ray, const GRec* rec, const uint32_t* vals,
                     const uint2* ranges, const uint32_t* order, const BlendParams& p,
                     float* image, float* intensity, int splits, float* part, cudaStream_t st) {
  const dim3 grid(n_tiles, splits);
  if (ray == VG_PINHOLE)
    k_tomo_fwd<VG_PINHOLE><<<grid, NT, 0, st>>>(rec, vals, ranges, order, p, image, intensity, part);
  else if (VG_TOMO_REC)
    k_tomo_fwd_rec<<<grid, NT, 0, st>>>(rec, vals, ranges, order, p, image, intensity, part);
  else
    k_tomo_fwd<VG_PARALLEL><<<grid, NT, 0, st>>>(rec, vals, ranges, order, p, image, intensity, part);
  if (splits > 1) {
    const int npix = p.width * p.height;
    k_tomo_combine<<<(npix + 255) / 256, 256, 0, st>>>(npix, splits, part, image, intensity);
  }
}

void launch_tomo_bwd(int n_tiles, int splits, int ray, int loss, const GRec* rec, const uint32_t* vals,
                     const uint2* ranges, const uint32_t* order, const BlendParams& p,
                     const float* d_image, const float* image, const float* target,
                     float loss_scale, double* loss_sum, float* acc, uint8_t* visible,
                     float* det_part, double* det_loss, cudaStream_t st) {
#define VG_TB(R, L, D)                                                                            \
  k_tomo_bwd<R, L, D><<<dim3(n_tiles, splits), NT, 0, st>>>(rec, vals, ranges, order, p, d_image, \
                                                            image, target,                        \
                                              loss_scale, loss_sum, acc, visible, det_part, det_loss)
#define VG_TB2(D)                                                       \
  do {                                                                  \
    if (ray == VG_PINHOLE) {                                            \
      if (loss) VG_TB(VG_PINHOLE, 1, D); else VG_TB(VG_PINHOLE, 0, D);  \
    } else {                                                            \
      if (loss) VG_TB(VG_PARALLEL, 1, D); else VG_TB(VG_PARALLEL, 0, D); \
    }                                                                   \
  } while (0)
  if (det_part) VG_TB2(true); else VG_TB2(false);
#undef VG_TB2
#undef VG_TB
}

#endif  // VG_TU_REST
}  // namespace vg

#if VG_TU_FWD
namespace vg {
// Debug statistics of one forward pass: {processed warp-entries, of which any
// pixel had alpha > 0, list entries walked per warp}.  Not on the hot path.
int debug_forward_stats(int n_tiles, const GRec* rec, const uint32_t* vals, const uint2* ranges,
                        const uint32_t* order, const BlendParams& p, float* color, float* final_t,
                        int* n_contrib, int* n_act, unsigned long long* out, cudaStream_t st) {
  unsigned long long z[4] = {0, 0, 0, 0};
  cudaMemcpyToSymbolAsync(g_vg_stats, z, sizeof(z), 0, cudaMemcpyHostToDevice, st);
  k_render_fwd<true, true, true><<<n_tiles, NT, 0, st>>>(rec, vals, ranges, order, p, color,
                                                        final_t, n_contrib, n_act, nullptr, 0,
                                                        SegIO());
  cudaMemcpyFromSymbolAsync(out, g_vg_stats, sizeof(z), 0, cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  return (int)cudaGetLastError();
}
}  // namespace vg
#endif  // VG_TU_FWD
