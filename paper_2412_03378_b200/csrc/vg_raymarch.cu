// Ground-truth ray marcher on the GPU: the reference's
// validation oracle oracle.raymarch_image (oracle.py:80-161), independent of
// the closed-form transmittance path -- midpoint-rule integration of the
// volume rendering equation through the full mixture density
//   sigma(x) = sum_i kappa_i exp(-q_i(x) / 2)   (q >= 120 contributes 0),
//   alpha_s = 1 - exp(-sigma_s dt),  colour = sum_s T_s alpha_s c(x_s) + T bg,
// with c(x) the kappa-weighted mean colour, over per-ray bounds that cover
// every primitive's [gamma - k beta, gamma + k beta] (clipped to t >= 0).
//
// One 256-thread CTA per pixel ray, float64 throughout.  The per-primitive
// ray coefficients (a, b, c of q(t) = a t^2 + 2 b t + c, kappa, colour) are
// staged in shared memory; each thread owns one step of a 256-step chunk,
// sums the mixture there, and a block-wide prefix product of (1 - alpha)
// carries the transmittance across the chunk.  Brute force over all
// primitives like the reference: a validation tool for small scenes.
#include <cmath>

#include "vg_kernels.cuh"

namespace vg {
namespace march {

constexpr int NTH = 256;
constexpr int CAP = 512;   // primitives staged per round (56 B each)

struct Coef {
  double a, b, c, kappa, r, g, bl;
};

__device__ __forceinline__ void ray_dir(const CamK& cam, int row, int col, double* d) {
  double dv[3] = {((double)col + 0.5 - cam.cx) / cam.fx, ((double)row + 0.5 - cam.cy) / cam.fy, 1.0};
  const double nn = sqrt(dot3(dv, dv));
  for (int k = 0; k < 3; ++k) dv[k] /= nn;
  for (int j = 0; j < 3; ++j) d[j] = cam.R[0 * 3 + j] * dv[0] + cam.R[1 * 3 + j] * dv[1] + cam.R[2 * 3 + j] * dv[2];
}

// q(t) coefficients of primitive i along origin o, unit direction d:
// delta = o - mean, a = d^T M d, b = (M delta) . d, c = delta^T M delta
__device__ __forceinline__ Coef coef_of(const vg_scene& s, int64_t i, const double* o, const double* d) {
  double R[9];
  quat_rotmat(s.rotations + 4 * i, R, nullptr);
  double inv[3];
  for (int k = 0; k < 3; ++k) {
    const double sk = fmax((double)s.scales[3 * i + k], SCALE_FLOOR);
    inv[k] = 1.0 / (sk * sk);
  }
  double M[9];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      double acc = 0.0;
      for (int k = 0; k < 3; ++k) acc += R[a * 3 + k] * inv[k] * R[b * 3 + k];
      M[a * 3 + b] = acc;
    }
  const double dl[3] = {o[0] - s.means[3 * i], o[1] - s.means[3 * i + 1], o[2] - s.means[3 * i + 2]};
  double Md[3], Mdl[3];
  matvec3(M, d, Md);
  matvec3(M, dl, Mdl);
  double sv[3] = {fmax((double)s.scales[3 * i], SCALE_FLOOR), fmax((double)s.scales[3 * i + 1], SCALE_FLOOR),
                  fmax((double)s.scales[3 * i + 2], SCALE_FLOOR)};
  Coef c;
  c.a = dot3(d, Md);
  c.b = dot3(Mdl, d);
  c.c = dot3(Mdl, dl);
  c.kappa = kappa_of((double)s.thetas[i], sv, nullptr, nullptr);
  c.r = s.colors ? s.colors[3 * i] : 0.0;
  c.g = s.colors ? s.colors[3 * i + 1] : 0.0;
  c.bl = s.colors ? s.colors[3 * i + 2] : 0.0;
  return c;
}

template <typename T, typename Op>
__device__ __forceinline__ T block_reduce(T v, Op op, T* sh) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int o = 16; o; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  T r = sh[0];
  for (int w = 1; w < NTH / 32; ++w) r = op(r, sh[w]);
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(NTH) k_raymarch(vg_scene s, CamK cam, int n_steps, double k_sig,
                                                  double t_min, double t_max, float* color,
                                                  float* final_t) {
  __shared__ Coef sc[CAP];
  __shared__ double sred[NTH / 32];
  __shared__ double sprod[NTH];
  const int pix = blockIdx.x;
  const int row = pix / cam.width, col = pix - row * cam.width;
  double d[3];
  ray_dir(cam, row, col, d);
  const double* o = cam.center;
  const int64_t n = s.n;
  if (n == 0) {
    if (threadIdx.x == 0) {
      for (int q = 0; q < 3; ++q) color[3 * pix + q] = (float)s.background[q];
      final_t[pix] = 1.f;
    }
    return;
  }
  // bounds: hull of [gamma - k beta, gamma + k beta] over the primitives (oracle.py:56-77),
  // with gamma = ((M (mean - o)) . d) / a = -b / a in the o - mean convention above
  double t0 = t_min, t1 = t_max;
  if (isnan(t_min) || isnan(t_max)) {
    double lo = INFINITY, hi = -INFINITY;
    for (int64_t i = threadIdx.x; i < n; i += NTH) {
      const Coef c = coef_of(s, i, o, d);
      const double gamma = -c.b / c.a, beta = 1.0 / sqrt(c.a);
      lo = fmin(lo, gamma - k_sig * beta);
      hi = fmax(hi, gamma + k_sig * beta);
    }
    lo = block_reduce(lo, [](double x, double y) { return fmin(x, y); }, sred);
    hi = block_reduce(hi, [](double x, double y) { return fmax(x, y); }, sred);
    const double a0 = fmax(lo, 0.0);
    const double a1 = fmax(hi, a0);
    if (isnan(t_min)) t0 = a0;
    if (isnan(t_max)) t1 = a1;
  }
  const double dt = (t1 - t0) / n_steps;
  double T = 1.0, cr = 0.0, cg = 0.0, cb = 0.0;
  for (int s0 = 0; s0 < n_steps; s0 += NTH) {
    const int st = s0 + threadIdx.x;
    const double t = t0 + ((double)st + 0.5) * dt;
    double sig = 0.0, wr = 0.0, wg = 0.0, wb = 0.0;
    for (int64_t c0 = 0; c0 < n; c0 += CAP) {
      const int nc = (int)min((int64_t)CAP, n - c0);
      __syncthreads();
      for (int i = threadIdx.x; i < nc; i += NTH) sc[i] = coef_of(s, c0 + i, o, d);
      __syncthreads();
      if (st < n_steps) {
        for (int i = 0; i < nc; ++i) {
          const Coef c = sc[i];
          const double q = fmax(c.a * t * t + 2.0 * c.b * t + c.c, 0.0);
          if (q < 120.0) {
            const double w = c.kappa * exp(-0.5 * q);
            sig += w;
            wr += w * c.r;
            wg += w * c.g;
            wb += w * c.bl;
          }
        }
      }
    }
    const double alpha = st < n_steps ? -expm1(-sig * dt) : 0.0;
    // inclusive prefix product of (1 - alpha) over the chunk (Hillis-Steele)
    sprod[threadIdx.x] = 1.0 - alpha;
    __syncthreads();
    for (int off = 1; off < NTH; off <<= 1) {
      const double v = threadIdx.x >= off ? sprod[threadIdx.x - off] : 1.0;
      __syncthreads();
      sprod[threadIdx.x] *= v;
      __syncthreads();
    }
    const double before = T * (threadIdx.x ? sprod[threadIdx.x - 1] : 1.0);
    const double ratio = before * alpha / fmax(sig, 1e-300);
    const double pr = block_reduce(ratio * wr, [](double x, double y) { return x + y; }, sred);
    const double pg = block_reduce(ratio * wg, [](double x, double y) { return x + y; }, sred);
    const double pb = block_reduce(ratio * wb, [](double x, double y) { return x + y; }, sred);
    cr += pr; cg += pg; cb += pb;
    T *= sprod[NTH - 1];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    if (!(dt > 0.0)) {  // degenerate bounds (oracle.py:131-134)
      cr = cg = cb = 0.0;
      T = 1.0;
    }
    color[3 * pix + 0] = (float)(cr + T * s.background[0]);
    color[3 * pix + 1] = (float)(cg + T * s.background[1]);
    color[3 * pix + 2] = (float)(cb + T * s.background[2]);
    final_t[pix] = (float)T;
  }
}

}  // namespace march
}  // namespace vg

extern "C" int vg_raymarch(const vg_scene* s, const vg_camera* cam, int32_t n_steps,
                           double support_sigmas, double t_min, double t_max, float* color,
                           float* final_t, void* stream) {
  using namespace vg;
  if (!s || !cam || !color || !final_t) return set_error(VG_EINVAL, "vg_raymarch: NULL argument");
  if (n_steps < 1) return set_error(VG_EINVAL, "vg_raymarch: n_steps must be positive");
  if (cam->projection != VG_PINHOLE) return set_error(VG_EINVAL, "vg_raymarch: pinhole cameras only");
  if (cam->width <= 0 || cam->height <= 0) return set_error(VG_EINVAL, "vg_raymarch: bad camera size");
  if (s->n > 0 && (!s->means || !s->scales || !s->rotations || !s->thetas))
    return set_error(VG_EINVAL, "vg_raymarch: scene arrays must be non-NULL");
  CamK k;
  k.width = cam->width;
  k.height = cam->height;
  k.ntx = (cam->width + TILE - 1) / TILE;
  k.nty = (cam->height + TILE - 1) / TILE;
  k.projection = cam->projection;
  k.fx = cam->fx; k.fy = cam->fy; k.cx = cam->cx; k.cy = cam->cy;
  k.z_near = cam->z_near;
  k.extent = 0.0;
  for (int i = 0; i < 9; ++i) k.R[i] = cam->rotation[i];
  for (int i = 0; i < 3; ++i) k.t[i] = cam->translation[i];
  for (int j = 0; j < 3; ++j)
    k.center[j] = -(k.R[0 * 3 + j] * k.t[0] + k.R[1 * 3 + j] * k.t[1] + k.R[2 * 3 + j] * k.t[2]);
  march::k_raymarch<<<cam->width * cam->height, march::NTH, 0, (cudaStream_t)stream>>>(
      *s, k, n_steps, support_sigmas, t_min, t_max, color, final_t);
  return cudaGetLastError() == cudaSuccess ? VG_OK : set_error(VG_ECUDA, "vg_raymarch: launch failed");
}
