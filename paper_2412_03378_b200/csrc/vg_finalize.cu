// K7: per-Gaussian gradient finalisation (float64), one thread per Gaussian.
//
// Input: the 13 linear accumulators the backward blend produced per
// Gaussian, in the Gaussian's whitened e-frame (vg_common.cuh):
//   A_raw = sum h (rho rho^T + w^ w^T)   (6, symmetric)
//   B_raw = sum h rho                     (3)
//   H     = sum h,  h = dL/de * beta * peak
//   Cd    = sum contrib * dL/dcolor       (3)
// with rho = W r (closest-approach offset, whitened) and w^ = W d / |W d|.
// Because g_expo = -1/2 dL/de e = -1/2 kappa sqrt(2 pi) h, the envelope form
// of grad.e_chain (grad.py:216-239) is
//   dL/dM     = W^-1 [ -1/2 kappa sqrt(2pi) A_raw ]_loc W^-T,
//   dL/dmean  = 2 M sum g r = 2 R S^-1 [ -1/2 kappa sqrt(2pi) B_raw ]_loc,
//   dL/dkappa = sqrt(2 pi) H,
// which equals the reference's ga dd^T + gb delta d^T + gc delta delta^T
// (after symmetrisation, which is all analytic_param_chain reads).  The
// parameter chain then follows grad.analytic_param_chain / _factored_grads /
// _quat_grads (grad.py:72-104, 242-259), with RtGR = S A_loc S.
// The accumulators are zeroed here so the next view starts clean.
#include "vg_kernels.cuh"

namespace vg {

struct FinalIn {
  int64_t n;
  const float* means;
  const float* scales;
  const float* rots;
  const float* thetas;
  const float* sh;
  float* acc;  // n * 16
};

__global__ void __launch_bounds__(128) k_finalize(FinalIn in, CamK c, vg_grads g) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= in.n) return;
  float4* a4 = reinterpret_cast<float4*>(in.acc + 16 * i);
  float4 x0 = a4[0], x1 = a4[1], x2 = a4[2], x3 = a4[3];
  float raw[13] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w, x2.x, x2.y, x2.z, x2.w, x3.x};
  bool any = false;
  for (int k = 0; k < 13; ++k) any |= raw[k] != 0.f;
  if (!any && g.accumulate) return;  // nothing to add for this view
  if (any) { float4 z = make_float4(0.f, 0.f, 0.f, 0.f); a4[0] = z; a4[1] = z; a4[2] = z; a4[3] = z; }

  double dmu[3] = {0, 0, 0}, ds[3] = {0, 0, 0}, dq[4] = {0, 0, 0, 0}, dth = 0, dk = 0;
  const float* sc = in.scales + 3 * i;
  if (any) {
    Frame f;
    make_frame(c, in.means + 3 * i, sc, in.rots + 4 * i, f);
    double im, lf;
    double theta = in.thetas[i];
    double kappa = kappa_of(theta, f.s, &im, &lf);
    double k2 = -0.5 * kappa * SQRT_2PI;
    double Ae[9] = {raw[0], raw[1], raw[2], raw[1], raw[3], raw[4], raw[2], raw[4], raw[5]};
    double Be[3] = {raw[6], raw[7], raw[8]};
    dk = SQRT_2PI * (double)raw[9];
    // to the whitened-local frame: A_loc = E^T A_e E with E rows e1,e2,e3
    double T1[9], Al[9], Bl[3];
    for (int a = 0; a < 3; ++a)
      for (int j = 0; j < 3; ++j)
        T1[a * 3 + j] = Ae[a * 3 + 0] * f.e[0 * 3 + j] + Ae[a * 3 + 1] * f.e[1 * 3 + j] + Ae[a * 3 + 2] * f.e[2 * 3 + j];
    for (int ii = 0; ii < 3; ++ii)
      for (int j = 0; j < 3; ++j)
        Al[ii * 3 + j] = k2 * (f.e[0 * 3 + ii] * T1[0 * 3 + j] + f.e[1 * 3 + ii] * T1[1 * 3 + j] + f.e[2 * 3 + ii] * T1[2 * 3 + j]);
    for (int j = 0; j < 3; ++j) Bl[j] = k2 * (f.e[0 * 3 + j] * Be[0] + f.e[1 * 3 + j] * Be[1] + f.e[2 * 3 + j] * Be[2]);
    // dL/dmean = 2 R S^-1 B_loc
    for (int a = 0; a < 3; ++a) {
      double s = 0;
      for (int k = 0; k < 3; ++k) s += f.R[a * 3 + k] * Bl[k] / f.s[k];
      dmu[a] = 2.0 * s;
    }
    // theta / scale chains (grad.py:248-257)
    dth = dk * im * THETA_CEILING / (1.0 - THETA_CEILING * theta);
    for (int k = 0; k < 3; ++k) {
      double dsk = dk * (-lf / (3.0 * f.s[k] * f.s[k])) + (-2.0 * Al[k * 4] / f.s[k]);
      ds[k] = ((double)sc[k] >= SCALE_FLOOR) ? dsk : 0.0;
    }
    // dL/dR = 2 R S A_loc S^-1  (= (G + G^T) R diag(1/s^2), G = R S A S R^T)
    double dR[9];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) {
        double s = 0;
        for (int k = 0; k < 3; ++k) s += f.R[a * 3 + k] * f.s[k] * Al[k * 3 + b];
        dR[a * 3 + b] = 2.0 * s / f.s[b];
      }
    // _quat_grads / _rotmat_quat_jacobian (grad.py:72-90)
    double qh[4], Rtmp[9];
    quat_rotmat(in.rots + 4 * i, Rtmp, qh);
    double w = qh[0], x = qh[1], y = qh[2], z = qh[3];
    double J[4][9] = {{0, -z, y, z, 0, -x, -y, x, 0},
                      {0, y, z, y, -2 * x, -w, z, w, -2 * x},
                      {-2 * y, x, w, x, 0, z, -w, z, -2 * y},
                      {-2 * z, -w, x, w, -2 * z, y, x, y, 0}};
    double dqh[4];
    for (int k = 0; k < 4; ++k) {
      double s = 0;
      for (int e = 0; e < 9; ++e) s += dR[e] * 2.0 * J[k][e];
      dqh[k] = s;
    }
    const float* qf = in.rots + 4 * i;
    double qn = sqrt((double)qf[0] * qf[0] + (double)qf[1] * qf[1] + (double)qf[2] * qf[2] + (double)qf[3] * qf[3]);
    double rad = qh[0] * dqh[0] + qh[1] * dqh[1] + qh[2] * dqh[2] + qh[3] * dqh[3];
    for (int k = 0; k < 4; ++k) dq[k] = (dqh[k] - qh[k] * rad) / qn;
  }
  const float dcol[3] = {raw[10], raw[11], raw[12]};
  const bool add = g.accumulate != 0;
#define VG_PUT(ptr, idx, val) \
  do { if (ptr) { float _v = (float)(val); if (add) ptr[idx] += _v; else ptr[idx] = _v; } } while (0)
  for (int k = 0; k < 3; ++k) {
    VG_PUT(g.d_means, 3 * i + k, dmu[k]);
    VG_PUT(g.d_scales, 3 * i + k, ds[k]);
    VG_PUT(g.d_colors, 3 * i + k, dcol[k]);
  }
  for (int k = 0; k < 4; ++k) VG_PUT(g.d_rotations, 4 * i + k, dq[k]);
  VG_PUT(g.d_thetas, i, dth);
  VG_PUT(g.d_kappas, i, dk);
  if (g.d_sh && in.sh) {
    double b[16] = {0};
    if (dcol[0] != 0.f || dcol[1] != 0.f || dcol[2] != 0.f) {
      double d[3] = {in.means[3 * i] - c.center[0], in.means[3 * i + 1] - c.center[1],
                     in.means[3 * i + 2] - c.center[2]};
      double dn = sqrt(dot3(d, d));
      d[0] /= dn; d[1] /= dn; d[2] /= dn;
      sh_basis(d, b);
    }
    for (int l = 0; l < 16; ++l)
      for (int ch = 0; ch < 3; ++ch) VG_PUT(g.d_sh, 48 * i + 3 * l + ch, b[l] * dcol[ch]);
  }
#undef VG_PUT
}

void launch_finalize(int64_t n, const vg_scene& s, const CamK& c, float* acc, const vg_grads& g,
                     cudaStream_t st) {
  if (n <= 0) return;
  FinalIn in{n, s.means, s.scales, s.rotations, s.thetas, s.sh, acc};
  k_finalize<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(in, c, g);
}

}  // namespace vg
