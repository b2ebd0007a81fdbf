// Training-step caller of the hot path: the reference's
// optim.Trainer.step + GradAccum.update (optim.py:119-206) as one fused
// per-Gaussian kernel, and the device half of densify_and_prune
// (optim.py:218-317): split / clone / prune decisions with the primitive
// budget, and the compaction that keeps the surviving rows and appends the
// children (Adam moments of children start at zero).  Host-side pieces
// (the split offsets' random draws, in the reference's generator order, and
// the event log) stay in paper_2412_03378_b200/optim.py.
//
// Precision: parameters and Adam moments are float32 on the device (the
// reference is float64); bias corrections and learning rates arrive from
// the host in float64 and are rounded once.
#include <climits>

#include "vg_kernels.cuh"

namespace vg {
namespace optim {

constexpr int NM = 14;  // moments per primitive: position 3, scale 3, rotation 4, colour 3, density 1
constexpr int G_POS = 0, G_SCALE = 1, G_ROT = 2, G_COL = 3, G_DEN = 4;

__device__ __forceinline__ float softplus10(float x) {
  // log(1 + e^{10x}) / 10, overflow-free (optim.py:110-111)
  const float y = 10.f * x;
  return (fmaxf(y, 0.f) + log1pf(expf(-fabsf(y)))) * 0.1f;
}
__device__ __forceinline__ float softplus10_inv(float c) {
  // optim.py:114-116 on colours clipped to >= 1e-6
  const float y = fmaxf(c, 1e-6f);
  return y + log1pf(-expf(-10.f * y)) * 0.1f;
}

struct AdamArgs {
  vg_train_state s;
  vg_grads g;
  float lr[5];
  float b1, b2, omb1, omb2, eps, inv_bc1, inv_bc2;  // omb = 1 - beta, rounded once from float64
  int* bad;  // [5] first primitive with a non-finite update per group
};

__device__ __forceinline__ float adam(float& m, float& v, float g, float lr, const AdamArgs& a) {
  m = a.b1 * m + a.omb1 * g;
  v = a.b2 * v + a.omb2 * g * g;
  return lr * (m * a.inv_bc1) / (sqrtf(v * a.inv_bc2) + a.eps);
}

__global__ void __launch_bounds__(256) k_adam_step(AdamArgs a) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= a.s.n) return;
  float* mo = a.s.moments + (int64_t)2 * NM * i;
  float m[NM], v[NM];
#pragma unroll
  for (int k = 0; k < NM; ++k) {
    m[k] = mo[k];
    v[k] = mo[NM + k];
  }
  float g[NM];
  for (int k = 0; k < 3; ++k) g[k] = a.g.d_means[3 * i + k];
  for (int k = 0; k < 3; ++k) g[3 + k] = a.g.d_scales[3 * i + k];
  for (int k = 0; k < 4; ++k) g[6 + k] = a.g.d_rotations[4 * i + k];
  float craw[3];
  for (int k = 0; k < 3; ++k) {
    craw[k] = a.s.color_raw[3 * i + k];
    // d/d(raw) of softplus = sigmoid(10 raw) (optim.py:148)
    g[10 + k] = a.g.d_colors[3 * i + k] / (1.f + expf(-10.f * craw[k]));
  }
  g[13] = a.g.d_thetas[i];
  // GradAccum.update (optim.py:199-203): norms of visible primitives
  if (a.s.accum_norm && a.g.visible && a.g.visible[i]) {
    a.s.accum_norm[i] += sqrtf(g[0] * g[0] + g[1] * g[1] + g[2] * g[2]);
    a.s.accum_count[i] += 1.f;
  }
  float u[NM];
  const int grp[NM] = {G_POS, G_POS, G_POS, G_SCALE, G_SCALE, G_SCALE, G_ROT, G_ROT, G_ROT, G_ROT,
                       G_COL, G_COL, G_COL, G_DEN};
#pragma unroll
  for (int k = 0; k < NM; ++k) {
    u[k] = adam(m[k], v[k], g[k], a.lr[grp[k]], a);
    if (!isfinite(u[k])) atomicMin(a.bad + grp[k], (int)i);
  }
#pragma unroll
  for (int k = 0; k < NM; ++k) {
    mo[k] = m[k];
    mo[NM + k] = v[k];
  }
  // constraint projections (optim.py:166-175)
  for (int k = 0; k < 3; ++k) a.s.means[3 * i + k] -= u[k];
  for (int k = 0; k < 3; ++k)
    a.s.scales[3 * i + k] = fmaxf(a.s.scales[3 * i + k] - u[3 + k], (float)SCALE_FLOOR);
  float q[4], qn = 0.f;
  for (int k = 0; k < 4; ++k) {
    q[k] = a.s.rotations[4 * i + k] - u[6 + k];
    qn += q[k] * q[k];
  }
  qn = rsqrtf(qn);
  for (int k = 0; k < 4; ++k) a.s.rotations[4 * i + k] = q[k] * qn;
  for (int k = 0; k < 3; ++k) {
    const float r = craw[k] - u[10 + k];
    a.s.color_raw[3 * i + k] = r;
    a.s.colors[3 * i + k] = softplus10(r);
  }
  a.s.thetas[i] = fminf(fmaxf(a.s.thetas[i] - u[13], 0.f), 1.f);
}

__global__ void k_init_bad(int* bad) {
  if (threadIdx.x < 5) bad[threadIdx.x] = INT_MAX;
}

// ---------------------------------------------------------------------------
// densify_and_prune, device half

constexpr uint8_t F_SPLIT = 1, F_CLONE = 2, F_PRUNE = 4;

// Decisions before the budget (optim.py:224-233, 292-294).
__global__ void k_densify_flags(vg_densify_args d, uint8_t* __restrict__ flags,
                                uint32_t* __restrict__ grow) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= d.n) return;
  double s[3];
  for (int k = 0; k < 3; ++k) s[k] = fmax((double)d.scales[3 * i + k], SCALE_FLOOR);
  const double theta = d.thetas[i];
  const double kappa = kappa_of(theta, s, nullptr, nullptr);
  const double ceiling = kappa_of(1.0, s, nullptr, nullptr);
  const double max_scale = fmax(fmax((double)d.scales[3 * i], (double)d.scales[3 * i + 1]),
                                (double)d.scales[3 * i + 2]);
  const double avg = (double)d.accum_norm[i] / fmax((double)d.accum_count[i], 1.0);
  const bool big = max_scale > d.prune_scale_fraction * d.extent;
  const bool split = (avg > d.split_grad_threshold && big) || kappa > d.high_kappa_split_fraction * ceiling;
  const bool clone = avg > d.clone_grad_threshold && !big && !split;
  const bool prune = theta < d.prune_theta_min || max_scale > d.prune_scale_fraction * d.extent;
  flags[i] = (split ? F_SPLIT : 0) | (clone ? F_CLONE : 0) | (prune ? F_PRUNE : 0);
  grow[i] = (split || clone) ? 1u : 0u;
}

// Budget (optim.py:235-240): only the first `budget` growing primitives (in
// index order) grow; then the output slot of every primitive: kept rows in
// order, split children (2 per split parent), clone children.  counts =
// {kept, splits, clones} packed as uint4 channel ranks (exclusive scans).
__global__ void k_densify_budget(int64_t n, uint8_t* __restrict__ flags,
                                 const uint32_t* __restrict__ grow_rank, int64_t budget,
                                 uint4* __restrict__ chan) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint8_t f = flags[i];
  if ((f & (F_SPLIT | F_CLONE)) && (int64_t)grow_rank[i] >= budget) f &= (uint8_t)~(F_SPLIT | F_CLONE);
  if (f & (F_SPLIT | F_CLONE)) f &= (uint8_t)~F_PRUNE;  // replaced parents are not pruned
  flags[i] = f;
  const bool keep = !(f & (F_SPLIT | F_CLONE | F_PRUNE));
  chan[i] = make_uint4(keep ? 1u : 0u, (f & F_SPLIT) ? 1u : 0u, (f & F_CLONE) ? 1u : 0u, 0u);
}

// Compaction + children (optim.py:243-317).  xi: 6 standard normals per
// split parent, in split-rank order (the reference's rng draws).
__global__ void k_densify_write(vg_densify_args d, const uint8_t* __restrict__ flags,
                                const uint4* __restrict__ rank, uint4 tot,
                                const double* __restrict__ xi, vg_train_state out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= d.n) return;
  const uint8_t f = flags[i];
  const uint4 r = rank[i];
  const float* mu = d.means + 3 * i;
  const float* sc = d.scales + 3 * i;
  const float* qq = d.rotations + 4 * i;
  auto put = [&](int64_t o, const float* m3, const float* s3, float theta, bool fresh) {
    for (int k = 0; k < 3; ++k) {
      out.means[3 * o + k] = m3[k];
      out.scales[3 * o + k] = s3[k];
      out.colors[3 * o + k] = d.colors[3 * i + k];
      out.color_raw[3 * o + k] =
          fresh ? softplus10_inv(d.colors[3 * i + k]) : d.color_raw[3 * i + k];
    }
    for (int k = 0; k < 4; ++k) out.rotations[4 * o + k] = qq[k];
    out.thetas[o] = theta;
    float* mo = out.moments + (int64_t)2 * NM * o;
    const float* mi = d.moments + (int64_t)2 * NM * i;
    for (int k = 0; k < 2 * NM; ++k) mo[k] = fresh ? 0.f : mi[k];
  };
  if (!(f & (F_SPLIT | F_CLONE | F_PRUNE))) {
    put(r.x, mu, sc, d.thetas[i], false);
    return;
  }
  if (!(f & (F_SPLIT | F_CLONE))) return;  // pruned
  // children: kappa halved, theta from the child scales, clamped at the ceiling
  double s[3];
  for (int k = 0; k < 3; ++k) s[k] = fmax((double)sc[k], SCALE_FLOOR);
  const double kappa = kappa_of((double)d.thetas[i], s, nullptr, nullptr);
  float cs[3];
  for (int k = 0; k < 3; ++k) cs[k] = (f & F_SPLIT) ? (float)((double)sc[k] / 1.6) : sc[k];
  double csd[3];
  for (int k = 0; k < 3; ++k) csd[k] = fmax((double)cs[k], SCALE_FLOOR);
  double im, lf;
  const double ceiling = kappa_of(1.0, csd, &im, &lf);
  const double target = 0.5 * kappa;
  double th = 1.0;
  if (!(target > ceiling * (1.0 + 1e-12)))
    th = fmin(fmax(-expm1(-target / im) / THETA_CEILING, 0.0), 1.0);  // core.theta_for_kappa
  if (f & F_SPLIT) {
    double R[9];
    quat_rotmat(qq, R, nullptr);
    for (int c = 0; c < 2; ++c) {
      const double* x = xi + 6 * (int64_t)r.y + 3 * c;
      float cm[3];
      for (int a = 0; a < 3; ++a) {
        double acc = mu[a];
        for (int k = 0; k < 3; ++k) acc += R[a * 3 + k] * ((double)sc[k] * x[k]);
        cm[a] = (float)acc;
      }
      put((int64_t)tot.x + 2 * (int64_t)r.y + c, cm, cs, (float)th, true);
    }
  } else {
    for (int c = 0; c < 2; ++c)
      put((int64_t)tot.x + 2 * (int64_t)tot.y + 2 * (int64_t)r.z + c, mu, cs, (float)th, true);
  }
}

// ---------------------------------------------------------------------------
// exclusive scan of uint32 / uint4 (4 channels) over n elements: per-block
// sums, one CTA over the block sums, then the add-back.

constexpr int SB = 1024;

template <typename T>
__device__ __forceinline__ T add(T a, T b);
template <>
__device__ __forceinline__ uint32_t add(uint32_t a, uint32_t b) { return a + b; }
template <>
__device__ __forceinline__ uint4 add(uint4 a, uint4 b) {
  return make_uint4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}
template <typename T>
__device__ __forceinline__ T zero();
template <>
__device__ __forceinline__ uint32_t zero() { return 0u; }
template <>
__device__ __forceinline__ uint4 zero() { return make_uint4(0u, 0u, 0u, 0u); }

template <typename T>
__device__ __forceinline__ T shfl_up(T v, int o) {
  return __shfl_up_sync(0xffffffffu, v, o);
}
template <>
__device__ __forceinline__ uint4 shfl_up(uint4 v, int o) {
  return make_uint4(__shfl_up_sync(0xffffffffu, v.x, o), __shfl_up_sync(0xffffffffu, v.y, o),
                    __shfl_up_sync(0xffffffffu, v.z, o), __shfl_up_sync(0xffffffffu, v.w, o));
}

// block-wide inclusive scan (SB threads) into `incl`; returns the block total
template <typename T>
__device__ __forceinline__ T block_scan(T v, T& incl) {
  __shared__ T ws[SB / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T y = shfl_up(x, o);
    if (lane >= o) x = add(x, y);
  }
  if (lane == 31) ws[warp] = x;
  __syncthreads();
  if (warp == 0) {
    T t = ws[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const T y = shfl_up(t, o);
      if (lane >= o) t = add(t, y);
    }
    ws[lane] = t;
  }
  __syncthreads();
  const T before = warp ? ws[warp - 1] : zero<T>();
  const T total = ws[SB / 32 - 1];
  incl = add(before, x);
  __syncthreads();
  return total;
}

template <typename T>
__device__ __forceinline__ T sub(T a, T b);
template <>
__device__ __forceinline__ uint32_t sub(uint32_t a, uint32_t b) { return a - b; }
template <>
__device__ __forceinline__ uint4 sub(uint4 a, uint4 b) {
  return make_uint4(a.x - b.x, a.y - b.y, a.z - b.z, a.w - b.w);
}

template <typename T>
__global__ void __launch_bounds__(SB) k_scan_blocks(const T* __restrict__ in, T* __restrict__ out,
                                                    T* __restrict__ sums, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * SB + threadIdx.x;
  const T v = i < n ? in[i] : zero<T>();
  T incl;
  const T total = block_scan(v, incl);
  if (i < n) out[i] = sub(incl, v);
  if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

template <typename T>
__global__ void __launch_bounds__(SB) k_scan_sums(T* __restrict__ sums, int64_t nb, T* __restrict__ total) {
  T carry = zero<T>();
  for (int64_t b0 = 0; b0 < nb; b0 += SB) {
    const int64_t b = b0 + threadIdx.x;
    const T v = b < nb ? sums[b] : zero<T>();
    T incl;
    const T t = block_scan(v, incl);
    if (b < nb) sums[b] = add(carry, sub(incl, v));
    carry = add(carry, t);
  }
  if (threadIdx.x == 0) *total = carry;
}

template <typename T>
__global__ void k_scan_add(T* __restrict__ out, const T* __restrict__ sums, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = add(out[i], sums[i / SB]);
}

template <typename T>
cudaError_t exclusive_scan(const T* in, T* out, T* scratch, T* total, int64_t n, cudaStream_t st) {
  const int64_t nb = (n + SB - 1) / SB;
  if (nb == 0) return cudaMemsetAsync(total, 0, sizeof(T), st);
  k_scan_blocks<T><<<(unsigned)nb, SB, 0, st>>>(in, out, scratch, n);
  k_scan_sums<T><<<1, SB, 0, st>>>(scratch, nb, total);
  k_scan_add<T><<<(unsigned)((n + 255) / 256), 256, 0, st>>>(out, scratch, n);
  return cudaGetLastError();
}

}  // namespace optim

cudaError_t scan_u32(const uint32_t* in, uint32_t* out, void* scratch, uint32_t* total, int64_t n,
                     cudaStream_t st) {
  return optim::exclusive_scan<uint32_t>(in, out, (uint32_t*)scratch, total, n, st);
}
size_t scan_u32_scratch_bytes(int64_t n) { return sizeof(uint32_t) * (size_t)((n + 1023) / 1024 + 1); }

}  // namespace vg

using namespace vg;
using namespace vg::optim;

extern "C" {

int vg_adam_step(vg_train_state* s, const vg_grads* g, const vg_adam_hparams* h, int32_t* bad,
                 void* stream) {
  if (!s || !g || !h || !bad) return set_error(VG_EINVAL, "vg_adam_step: NULL argument");
  if (s->n < 0 || h->t < 1) return set_error(VG_EINVAL, "vg_adam_step: bad primitive count or step");
  if (s->n > 0 && (!s->means || !s->scales || !s->rotations || !s->thetas || !s->colors ||
                   !s->color_raw || !s->moments || !g->d_means || !g->d_scales ||
                   !g->d_rotations || !g->d_thetas || !g->d_colors))
    return set_error(VG_EINVAL, "vg_adam_step: state and gradient arrays must be non-NULL");
  cudaStream_t st = (cudaStream_t)stream;
  k_init_bad<<<1, 32, 0, st>>>(bad);
  if (s->n == 0) return cudaGetLastError() == cudaSuccess ? VG_OK : set_error(VG_ECUDA, "vg_adam_step: launch failed");
  AdamArgs a;
  a.s = *s;
  a.g = *g;
  for (int k = 0; k < 5; ++k) a.lr[k] = (float)h->lr[k];
  a.b1 = (float)h->beta1;
  a.b2 = (float)h->beta2;
  a.omb1 = (float)(1.0 - h->beta1);
  a.omb2 = (float)(1.0 - h->beta2);
  a.eps = (float)h->eps;
  a.inv_bc1 = (float)(1.0 / (1.0 - pow(h->beta1, (double)h->t)));
  a.inv_bc2 = (float)(1.0 / (1.0 - pow(h->beta2, (double)h->t)));
  a.bad = bad;
  k_adam_step<<<(unsigned)((s->n + 255) / 256), 256, 0, st>>>(a);
  return cudaGetLastError() == cudaSuccess ? VG_OK : set_error(VG_ECUDA, "vg_adam_step: launch failed");
}

size_t vg_densify_scratch_bytes(int64_t n) {
  const int64_t nb = (n + SB - 1) / SB + 1;
  return (size_t)n * (1 + 4 + 4 + 16 + 16) + (size_t)nb * 16 + 64 + 256;
}

static char* align16(char* p) { return (char*)(((uintptr_t)p + 15) & ~(uintptr_t)15); }

int vg_densify_plan(const vg_densify_args* d, void* scratch, uint32_t* counts_dev, void* stream) {
  if (!d || !scratch || !counts_dev) return VG_EINVAL;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t n = d->n;
  char* p = align16((char*)scratch);
  uint8_t* flags = (uint8_t*)p;
  p = align16(p + n);
  uint32_t* grow = (uint32_t*)p;
  p = align16(p + 4 * n);
  uint32_t* grow_rank = (uint32_t*)p;
  p = align16(p + 4 * n);
  uint4* chan = (uint4*)p;
  p = align16(p + 16 * n);
  uint4* rank = (uint4*)p;
  p = align16(p + 16 * n);
  uint4* sums = (uint4*)p;
  // counts_dev: {grown (before budget), kept, splits, clones}
  if (n == 0) return cudaMemsetAsync(counts_dev, 0, 4 * sizeof(uint32_t), st) == cudaSuccess ? VG_OK : VG_ECUDA;
  const unsigned blocks = (unsigned)((n + 255) / 256);
  k_densify_flags<<<blocks, 256, 0, st>>>(*d, flags, grow);
  if (exclusive_scan<uint32_t>(grow, grow_rank, (uint32_t*)sums, counts_dev, n, st) != cudaSuccess)
    return VG_ECUDA;
  const int64_t budget = d->max_primitives > n ? d->max_primitives - n : 0;
  k_densify_budget<<<blocks, 256, 0, st>>>(n, flags, grow_rank, budget, chan);
  // channel totals land in counts_dev[1..3] via a uint4 staged at the end of scratch
  uint4* total4 = (uint4*)align16((char*)scratch + vg_densify_scratch_bytes(n) - 32);
  if (exclusive_scan<uint4>(chan, rank, sums, total4, n, st) != cudaSuccess) return VG_ECUDA;
  if (cudaMemcpyAsync(counts_dev + 1, total4, 3 * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st) !=
      cudaSuccess)
    return VG_ECUDA;
  return cudaGetLastError() == cudaSuccess ? VG_OK : VG_ECUDA;
}

int vg_densify_apply(const vg_densify_args* d, const void* scratch, const uint32_t* counts_host,
                     const double* xi_dev, vg_train_state* out, void* stream) {
  if (!d || !scratch || !counts_host || !out) return VG_EINVAL;
  const int64_t n = d->n;
  if (n == 0) return VG_OK;
  const char* p = align16((char*)scratch);
  const uint8_t* flags = (const uint8_t*)p;
  p = align16((char*)p + n);
  p = align16((char*)p + 4 * n);
  p = align16((char*)p + 4 * n);
  p = align16((char*)p + 16 * n);
  const uint4* rank = (const uint4*)p;
  const uint4 tot = make_uint4(counts_host[1], counts_host[2], counts_host[3], 0u);
  if (tot.y > 0 && !xi_dev) return VG_EINVAL;
  k_densify_write<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(*d, flags, rank, tot,
                                                                               xi_dev, *out);
  return cudaGetLastError() == cudaSuccess ? VG_OK : VG_ECUDA;
}

}  // extern "C"
