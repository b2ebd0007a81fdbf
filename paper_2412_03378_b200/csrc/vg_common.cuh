// Shared definitions for the volgauss_b200 kernels (sm_100a).
//
// Numerical design: everything
// per Gaussian is computed in float64 (O(N) work), everything per
// (Gaussian, pixel) pair in float32 in a cancellation-free form:
//
//   whitening  W = S^-1 R_g^T R_c^T  maps view-space vectors to the frame in
//   which the Gaussian is the unit sphere (M = W^T W in view space);
//   m = W d_mu (d_mu = (x/z, y/z, 1)), D = |W v| = z |m|;
//   orthonormal frame e3 = m/|m|, e2 ~ (W e_y)_perp, e1 = e2 x e3.
//   For the pixel offset (du, dv) (pixels, from the projected mean):
//     q1 = P11 du,  q2 = P21 du + P22 dv       (w_perp in the e1,e2 plane)
//     w_par = |m| + n1 du + n2 dv              (w along e3)
//     X = q1^2 + q2^2,  |w|^2 = w_par^2 + X
//     expo = D^2 X / |w|^2,  beta = |d'| / |w|,  peak = exp(-expo/2)
//   which equals the reference's c - b^2/a and 1/sqrt(a)
//   (raster.py:341-349) without its catastrophic cancellation.
#pragma once

#include <cuda_runtime.h>
#include <cstdio>
#include <stdint.h>

#include "volgauss_b200.h"

// Debug builds (-DVG_DEBUG, tools/debug_checks.py; compute-sanitizer is not
// available on the measurement pool): VG_ASSERT traps on a violated index
// bound, VG_JITTER sleeps a hashed number of nanoseconds so that warps
// interleave differently from run to run (a shared-memory race then shows as
// a result that differs between jitter seeds).  Both compile to nothing in
// the release library.
#ifdef VG_DEBUG
#define VG_ASSERT(cond)                                                                  \
  do {                                                                                   \
    if (!(cond)) {                                                                       \
      printf("VG_ASSERT failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #cond, \
             (int)blockIdx.x, (int)threadIdx.x);                                         \
      __trap();                                                                          \
    }                                                                                    \
  } while (0)
#define VG_JITTER(seed, salt)                                                            \
  do {                                                                                   \
    if (seed) {                                                                          \
      unsigned _h = (unsigned)(seed) * 2654435761u ^ (blockIdx.x * 97u + (threadIdx.x >> 5) * 131u + \
                                                     (unsigned)(salt) * 7919u);            \
      _h ^= _h >> 13; _h *= 0x5bd1e995u; _h ^= _h >> 15;                                 \
      __nanosleep(_h & 2047u);                                                           \
    }                                                                                    \
  } while (0)
#else
#define VG_ASSERT(cond) do { } while (0)
#define VG_JITTER(seed, salt) do { } while (0)
#endif

namespace vg {

constexpr int TILE = 16;
constexpr int TILE_PIX = TILE * TILE;
constexpr double SQRT_2PI = 2.5066282746310002;
constexpr double LOG2E = 1.4426950408889634;
constexpr double LN2 = 0.69314718055994531;
constexpr double SCALE_FLOOR = 1e-7;    // core.py:18
constexpr double THETA_CEILING = 0.99;  // core.py:22
constexpr double DILATION = 0.3;        // raster.py:30
constexpr double BASE_SIGMA = 3.0;      // raster.py:35

// Per-Gaussian blend record (80 B), written by preprocess, gathered per tile.
struct __align__(16) GRec {
  double u, v;            // projected mean in pixel coordinates (continuous)
  float P11, P21, P22;    // q = P (du, dv)
  float n1, n2, wm;       // w_par = wm + n1 du + n2 dv       (pinhole)
  float cD2;              // 0.5 log2(e) D^2                  (pinhole)
  float D;                // D (pinhole) | beta (parallel)
  float kap2;             // kappa sqrt(2 pi) log2(e)
  float cr, cg, cb;       // RGB (evaluated from SH when present)
  float amp;              // kappa sqrt(2 pi) s_max >= e at any pixel (culling bound)
  float pad0, pad1, pad2;
};
static_assert(sizeof(GRec) == 80, "GRec must be 80 bytes");

// Camera in the form kernels take by value.
struct CamK {
  int width, height, ntx, nty, projection;
  double fx, fy, cx, cy, z_near, extent;
  double R[9];
  double t[3];
  double center[3];
};

struct Frame {
  double R[9];    // R_g, row-major (columns are the local axes in world)
  double s[3];    // floored scales
  double v[3];    // view-space mean
  double e[9];    // rows: e1, e2, e3 in whitened-local coordinates
  double P11, P21, P22, n1, n2, wm, D, beta;
  double pu, pv;  // projected mean, pixel coordinates
};

__host__ __device__ inline double dot3(const double* a, const double* b) {
  return a[0] * b[0] + a[1] * b[1] + a[2] * b[2];
}

// core.quat_to_rotmat (core.py:81-101)
__host__ __device__ inline void quat_rotmat(const float* qf, double* R, double* qhat) {
  double w = qf[0], x = qf[1], y = qf[2], z = qf[3];
  double n = sqrt(w * w + x * x + y * y + z * z);
  w /= n; x /= n; y /= n; z /= n;
  if (qhat) { qhat[0] = w; qhat[1] = x; qhat[2] = y; qhat[3] = z; }
  R[0] = 1 - 2 * (y * y + z * z); R[1] = 2 * (x * y - w * z);     R[2] = 2 * (x * z + w * y);
  R[3] = 2 * (x * y + w * z);     R[4] = 1 - 2 * (x * x + z * z); R[5] = 2 * (y * z - w * x);
  R[6] = 2 * (x * z - w * y);     R[7] = 2 * (y * z + w * x);     R[8] = 1 - 2 * (x * x + y * y);
}

// Whitening W (view -> whitened local): row i = (R_c g_i)^T / s_i, g_i = column i of R_g.
// (Record-only quantities -- the blend record and the gradient frame, not the
// bit-exact binning -- so the float64 divisions here and below are one
// reciprocal each and multiplies: float64 division is a long Newton sequence.)
__host__ __device__ __forceinline__ void whitening(const CamK& c, const double* R, const double* s, double* W) {
  for (int i = 0; i < 3; ++i) {
    double g0 = R[0 * 3 + i], g1 = R[1 * 3 + i], g2 = R[2 * 3 + i];
    const double is = 1.0 / s[i];
    for (int j = 0; j < 3; ++j)
      W[i * 3 + j] = (c.R[j * 3 + 0] * g0 + c.R[j * 3 + 1] * g1 + c.R[j * 3 + 2] * g2) * is;
  }
}

__host__ __device__ inline void matvec3(const double* W, const double* x, double* y) {
  y[0] = W[0] * x[0] + W[1] * x[1] + W[2] * x[2];
  y[1] = W[3] * x[0] + W[4] * x[1] + W[5] * x[2];
  y[2] = W[6] * x[0] + W[7] * x[1] + W[8] * x[2];
}

// Build e1,e2 from e3 and a vector g1 (not parallel to e3); returns plane coords.
__host__ __device__ __forceinline__ void plane_basis(const double* e3, const double* g1, double* e) {
  double k = dot3(g1, e3);
  double p[3] = {g1[0] - k * e3[0], g1[1] - k * e3[1], g1[2] - k * e3[2]};
  const double ipn = 1.0 / sqrt(dot3(p, p));
  double e2[3] = {p[0] * ipn, p[1] * ipn, p[2] * ipn};
  double e1[3] = {e2[1] * e3[2] - e2[2] * e3[1], e2[2] * e3[0] - e2[0] * e3[2],
                  e2[0] * e3[1] - e2[1] * e3[0]};
  for (int j = 0; j < 3; ++j) { e[j] = e1[j]; e[3 + j] = e2[j]; e[6 + j] = e3[j]; }
}

// Per-Gaussian frame for either ray model.  Returns false when the mean is
// not in front of the near plane (pinhole) -- such Gaussians are never binned.
__host__ __device__ __forceinline__ bool make_frame(const CamK& c, const float* mu, const float* sc,
                                           const float* q, Frame& f) {
  quat_rotmat(q, f.R, nullptr);
  for (int i = 0; i < 3; ++i) f.s[i] = fmax((double)sc[i], SCALE_FLOOR);
  double m3[3] = {mu[0], mu[1], mu[2]};
  for (int j = 0; j < 3; ++j) f.v[j] = c.R[j * 3 + 0] * m3[0] + c.R[j * 3 + 1] * m3[1] + c.R[j * 3 + 2] * m3[2] + c.t[j];
  double W[9];
  whitening(c, f.R, f.s, W);
  if (c.projection == VG_PINHOLE) {
    double z = f.v[2];
    if (!(z > c.z_near)) return false;
    const double iz = 1.0 / z;
    double dmu[3] = {f.v[0] * iz, f.v[1] * iz, 1.0};
    double m[3];
    matvec3(W, dmu, m);
    double mn = sqrt(dot3(m, m));
    const double imn = 1.0 / mn;
    double e3[3] = {m[0] * imn, m[1] * imn, m[2] * imn};
    const double ifx = 1.0 / c.fx, ify = 1.0 / c.fy;
    double G0[3] = {W[0] * ifx, W[3] * ifx, W[6] * ifx};
    double G1[3] = {W[1] * ify, W[4] * ify, W[7] * ify};
    plane_basis(e3, G1, f.e);
    f.P11 = dot3(f.e, G0);
    f.P21 = dot3(f.e + 3, G0);
    f.P22 = dot3(f.e + 3, G1);
    f.n1 = dot3(e3, G0);
    f.n2 = dot3(e3, G1);
    f.wm = mn;
    f.D = z * mn;
    f.beta = 0.0;
    f.pu = c.fx * f.v[0] / z + c.cx;
    f.pv = c.fy * f.v[1] / z + c.cy;
  } else {
    // orthographic rays along the view z axis; detector pixel pitch 2 extent / size
    double w[3] = {W[2], W[5], W[8]};
    double wn = sqrt(dot3(w, w));
    double e3[3] = {w[0] / wn, w[1] / wn, w[2] / wn};
    double sx = 2.0 * c.extent / c.width, sy = 2.0 * c.extent / c.height;
    double G0[3] = {W[0] * sx, W[3] * sx, W[6] * sx};
    double G1[3] = {W[1] * sy, W[4] * sy, W[7] * sy};
    plane_basis(e3, G1, f.e);
    f.P11 = dot3(f.e, G0);
    f.P21 = dot3(f.e + 3, G0);
    f.P22 = dot3(f.e + 3, G1);
    f.n1 = f.n2 = 0.0;
    f.wm = wn;
    f.D = 0.0;
    f.beta = 1.0 / wn;
    f.pu = (f.v[0] / c.extent + 1.0) * 0.5 * c.width;
    f.pv = (f.v[1] / c.extent + 1.0) * 0.5 * c.height;
  }
  return true;
}

// density_kappa (core.py:132-143)
__host__ __device__ inline double kappa_of(double theta, const double* s, double* inv_mean,
                                           double* lfac) {
  double im = (1.0 / s[0] + 1.0 / s[1] + 1.0 / s[2]) / 3.0;
  double lf = -log1p(-THETA_CEILING * theta);
  if (inv_mean) *inv_mean = im;
  if (lfac) *lfac = lf;
  return lf * im;
}

// Real SH basis up to degree 3 (band 0 = 1, so the DC coefficient is the RGB).
__host__ __device__ inline void sh_basis(const double* d, double* b) {
  double x = d[0], y = d[1], z = d[2];
  double xx = x * x, yy = y * y, zz = z * z;
  const double c1 = 0.4886025119029199;
  b[0] = 1.0;
  b[1] = -c1 * y; b[2] = c1 * z; b[3] = -c1 * x;
  b[4] = 1.0925484305920792 * x * y;
  b[5] = -1.0925484305920792 * y * z;
  b[6] = 0.31539156525252005 * (2 * zz - xx - yy);
  b[7] = -1.0925484305920792 * x * z;
  b[8] = 0.5462742152960396 * (xx - yy);
  b[9] = -0.5900435899266435 * y * (3 * xx - yy);
  b[10] = 2.890611442640554 * x * y * z;
  b[11] = -0.4570457994644658 * y * (4 * zz - xx - yy);
  b[12] = 0.3731763325901154 * z * (2 * zz - 3 * xx - 3 * yy);
  b[13] = -0.4570457994644658 * x * (4 * zz - xx - yy);
  b[14] = 1.445305721320277 * z * (xx - yy);
  b[15] = -0.5900435899266435 * x * (xx - 3 * yy);
}

// the same basis in float32 with explicit FMAs (preprocess colour evaluation)
__device__ __forceinline__ void sh_basis_f(float x, float y, float z, float* b) {
  const float xx = x * x, yy = y * y, zz = z * z;
  const float c1 = 0.4886025119029199f;
  b[0] = 1.f;
  b[1] = -c1 * y; b[2] = c1 * z; b[3] = -c1 * x;
  b[4] = 1.0925484305920792f * x * y;
  b[5] = -1.0925484305920792f * y * z;
  b[6] = 0.31539156525252005f * fmaf(2.f, zz, -xx - yy);
  b[7] = -1.0925484305920792f * x * z;
  b[8] = 0.5462742152960396f * (xx - yy);
  b[9] = -0.5900435899266435f * y * fmaf(3.f, xx, -yy);
  b[10] = 2.890611442640554f * x * y * z;
  b[11] = -0.4570457994644658f * y * fmaf(4.f, zz, -xx - yy);
  b[12] = 0.3731763325901154f * z * fmaf(2.f, zz, -3.f * xx - 3.f * yy);
  b[13] = -0.4570457994644658f * x * fmaf(4.f, zz, -xx - yy);
  b[14] = 1.445305721320277f * z * (xx - yy);
  b[15] = -0.5900435899266435f * x * fmaf(-3.f, yy, xx);
}

// ---------------------------------------------------------------------------
// fast SFU math (MUFU.EX2 / MUFU.RSQ / MUFU.LG2)

__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rsqf(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float lg2f(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

}  // namespace vg
