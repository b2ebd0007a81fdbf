// K7: per-Gaussian gradient finalisation, split in two passes.
//
// (a) k_view_accumulate, once per view (float32, one thread per Gaussian):
//   The backward blend leaves 13 linear accumulators per Gaussian in that
//   view's whitened e-frame (vg_common.cuh, vg_blend.cu):
//     A_raw = sum h (rho rho^T + w^ w^T)   (6, symmetric)
//     B_raw = sum h rho                     (3)
//     H     = sum h,  h = dL/de * beta * peak
//     Cd    = sum contrib * dL/dcolor       (3)
//   with rho = W r (closest-approach offset, whitened) and w^ = W d / |W d|.
//   The e-frame (stored by preprocess) is view dependent; rotating A and B
//   into the Gaussian's whitened-LOCAL frame makes them view independent, so
//   they are summed over views in a per-context accumulator.  RGB colour
//   gradients are summed the same way.  With SH colour the pull-back onto the
//   16 x 3 coefficients depends on the view direction, so each view only
//   stores its 3-float dL/dRGB (a slab per view) and k_sh_pull folds all the
//   views of the step in one pass (48 register accumulators per Gaussian)
//   instead of a 384-byte read-modify-write per Gaussian and view.
//
// (b) k_finalize_params, once per step (float64): because
//   g_expo = -1/2 dL/de e = -1/2 kappa sqrt(2 pi) h, the envelope form of
//   grad.e_chain (grad.py:216-239) is
//     dL/dM     = W^-1 [ -1/2 kappa sqrt(2pi) A_loc ] W^-T,   W = S^-1 R^T,
//     dL/dmean  = 2 M sum g r = 2 R S^-1 [ -1/2 kappa sqrt(2pi) B_loc ],
//     dL/dkappa = sqrt(2 pi) H,
//   which equals the reference's ga dd^T + gb delta d^T + gc delta delta^T
//   after symmetrisation (all analytic_param_chain reads).  The parameter
//   chain follows grad.analytic_param_chain / _factored_grads / _quat_grads
//   (grad.py:72-104, 242-259) with R^T G R = S A_loc S.
#include "vg_kernels.cuh"

namespace vg {

struct ViewAccIn {
  int64_t n;
  const float* means;
  const float* scales;  // splat mode: the EWA projection is re-derived per view
  const float* rots;
  const float* sh;       // optional SH-3 coefficients (selects the SH pull-back)
  const float* frame;    // n * 12: e1, e2, e3 (whitened-local), pad
  float* acc;            // n * 16 per-view accumulators (zeroed here)
  float* lacc;           // n * 12 view-independent accumulators
  float* cacc;           // [3][n] RGB gradient accumulators (SoA: coalesced)
  float* dcol;           // SH scenes: this view's dL/dRGB slab [3][n]
  double* center;        // SH scenes: this view's camera centre (written by thread 0)
  const uint32_t* seg_counts;          // segmented backward: publish the next view's decision
  unsigned long long* seg_decision;
  uint32_t seg_slots;
  float seg_ratio;
};

struct FinalIn {
  int64_t n;
  const float* scales;
  const float* rots;
  const float* thetas;
  float* lacc;  // n * 12 (zeroed here)
};

__global__ void __launch_bounds__(256) k_view_accumulate(ViewAccIn in, CamK c) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (in.seg_decision && i == 0) seg_publish(in.seg_counts, in.seg_decision, in.seg_slots, in.seg_ratio);
  if (i >= in.n) return;
  // all loads issued up front (one memory round trip instead of three)
  float4* a4 = reinterpret_cast<float4*>(in.acc + 16 * i);
  const float4* f4 = reinterpret_cast<const float4*>(in.frame + 12 * i);
  float4* l4 = reinterpret_cast<float4*>(in.lacc + 12 * i);
  const float4 x0 = a4[0], x1 = a4[1], x2 = a4[2], x3 = a4[3];
  const float4 f0 = __ldg(f4), f1 = __ldg(f4 + 1), f2 = __ldg(f4 + 2);
  float4 l0 = l4[0], l1 = l4[1], l2 = l4[2];
  const float raw[13] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w, x2.x, x2.y, x2.z, x2.w, x3.x};
  bool any = false;
#pragma unroll
  for (int k = 0; k < 13; ++k) any |= raw[k] != 0.f;
  const int64_t n = in.n;
  if (in.dcol) {
    if (i == 0) {
      in.center[0] = c.center[0];
      in.center[1] = c.center[1];
      in.center[2] = c.center[2];
    }
    in.dcol[i] = raw[10];
    in.dcol[n + i] = raw[11];
    in.dcol[2 * n + i] = raw[12];
  }
  if (!any) return;
  const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
  a4[0] = z; a4[1] = z; a4[2] = z; a4[3] = z;
  // rotate into the whitened-local frame: A_loc = sum_ab A_e[a][b] e_a e_b^T
  const float e[3][3] = {{f0.x, f0.y, f0.z}, {f0.w, f1.x, f1.y}, {f1.z, f1.w, f2.x}};
  const float Ae[3][3] = {{raw[0], raw[1], raw[2]}, {raw[1], raw[3], raw[4]}, {raw[2], raw[4], raw[5]}};
  float T1[3][3];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      T1[a][j] = fmaf(Ae[a][0], e[0][j], fmaf(Ae[a][1], e[1][j], Ae[a][2] * e[2][j]));
  float Al[6];
  const int ii[6] = {0, 0, 0, 1, 1, 2}, jj[6] = {0, 1, 2, 1, 2, 2};
#pragma unroll
  for (int q = 0; q < 6; ++q)
    Al[q] = fmaf(e[0][ii[q]], T1[0][jj[q]], fmaf(e[1][ii[q]], T1[1][jj[q]], e[2][ii[q]] * T1[2][jj[q]]));
  float Bl[3];
#pragma unroll
  for (int j = 0; j < 3; ++j) Bl[j] = fmaf(e[0][j], raw[6], fmaf(e[1][j], raw[7], e[2][j] * raw[8]));
  l0.x += Al[0]; l0.y += Al[1]; l0.z += Al[2]; l0.w += Al[3];
  l1.x += Al[4]; l1.y += Al[5]; l1.z += Bl[0]; l1.w += Bl[1];
  l2.x += Bl[2]; l2.y += raw[9];
  l4[0] = l0; l4[1] = l1; l4[2] = l2;
  // colour: dL/dRGB of this view (SH scenes: deferred to k_sh_pull)
  if (in.dcol) return;
  if (raw[10] != 0.f) in.cacc[i] += raw[10];
  if (raw[11] != 0.f) in.cacc[n + i] += raw[11];
  if (raw[12] != 0.f) in.cacc[2 * n + i] += raw[12];
}

// mode="splat" (the EWA comparator): the view's accumulators (slot 0
// dL/dopacity, 1..3 dL/dconic (xx, xy, yy), 4..5 dL/dmean2d; colour 10..12)
// are pulled through this view's EWA projection (grad.py:262-302,
// _splat_projection_backward) into view-independent world-space terms:
// lacc 0..5 dL/dSigma (xx, xy, xz, yy, yz, zz), 6..8 dL/dmean, 9 dL/dopacity.
__global__ void __launch_bounds__(128) k_view_accumulate_splat(ViewAccIn in, CamK c) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= in.n) return;
  float4* a4 = reinterpret_cast<float4*>(in.acc + 16 * i);
  const float4 x0 = a4[0], x1 = a4[1], x2 = a4[2], x3 = a4[3];
  const float raw[13] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w, x2.x, x2.y, x2.z, x2.w, x3.x};
  bool any = false;
#pragma unroll
  for (int k = 0; k < 13; ++k) any |= raw[k] != 0.f;
  const int64_t n = in.n;
  if (in.dcol) {
    if (i == 0) { in.center[0] = c.center[0]; in.center[1] = c.center[1]; in.center[2] = c.center[2]; }
    in.dcol[i] = raw[10];
    in.dcol[n + i] = raw[11];
    in.dcol[2 * n + i] = raw[12];
  }
  if (!any) return;
  const float4 zf = make_float4(0.f, 0.f, 0.f, 0.f);
  a4[0] = zf; a4[1] = zf; a4[2] = zf; a4[3] = zf;
  if (raw[0] != 0.f || raw[1] != 0.f || raw[2] != 0.f || raw[3] != 0.f || raw[4] != 0.f ||
      raw[5] != 0.f) {
    // re-derive this view's projection exactly as preprocess did
    double R[9];
    quat_rotmat(in.rots + 4 * i, R, nullptr);
    double s[3];
    for (int k = 0; k < 3; ++k) s[k] = fmax((double)in.scales[3 * i + k], SCALE_FLOOR);
    double Sig[9];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) {
        double acc = 0.0;
        for (int k = 0; k < 3; ++k) acc += R[a * 3 + k] * (s[k] * s[k]) * R[b * 3 + k];
        Sig[a * 3 + b] = acc;
      }
    const double m3[3] = {in.means[3 * i], in.means[3 * i + 1], in.means[3 * i + 2]};
    double v[3];
    for (int j = 0; j < 3; ++j)
      v[j] = c.R[j * 3 + 0] * m3[0] + c.R[j * 3 + 1] * m3[1] + c.R[j * 3 + 2] * m3[2] + c.t[j];
    const double z = v[2], x = v[0], y = v[1];
    const double limx = 1.3 * (0.5 * c.width / c.fx), limy = 1.3 * (0.5 * c.height / c.fy);
    const double rx = fmin(fmax(x / z, -limx), limx), ry = fmin(fmax(y / z, -limy), limy);
    const bool ox = !(fabs(x / z) > limx), oy = !(fabs(y / z) > limy);
    const double J[6] = {c.fx / z, 0.0, -c.fx * rx / z, 0.0, c.fy / z, -c.fy * ry / z};
    double U[6];
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 3; ++b)
        U[a * 3 + b] = J[a * 3] * c.R[b] + J[a * 3 + 1] * c.R[3 + b] + J[a * 3 + 2] * c.R[6 + b];
    double cov[4];
    for (int a = 0; a < 2; ++a)
      for (int l = 0; l < 2; ++l) {
        double acc = 0.0;
        for (int j = 0; j < 3; ++j)
          for (int k = 0; k < 3; ++k) acc += U[a * 3 + j] * Sig[j * 3 + k] * U[l * 3 + k];
        cov[a * 2 + l] = acc;
      }
    cov[0] += DILATION;
    cov[3] += DILATION;
    const double det = cov[0] * cov[3] - cov[1] * cov[2];
    const double L[4] = {cov[3] / det, -cov[1] / det, -cov[2] / det, cov[0] / det};
    const double gl[4] = {raw[1], raw[2], raw[2], raw[3]};
    // g_cov = -L gl L
    double t[4], gc[4];
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 2; ++b) t[a * 2 + b] = gl[a * 2] * L[b] + gl[a * 2 + 1] * L[2 + b];
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 2; ++b) gc[a * 2 + b] = -(L[a * 2] * t[b] + L[a * 2 + 1] * t[2 + b]);
    // dSigma = U^T g_cov U
    double dS[9];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) {
        double acc = 0.0;
        for (int p = 0; p < 2; ++p)
          for (int q = 0; q < 2; ++q) acc += U[p * 3 + a] * gc[p * 2 + q] * U[q * 3 + b];
        dS[a * 3 + b] = acc;
      }
    // d_u = (g_cov + g_cov^T) U Sigma ; d_j = d_u R_c^T
    double US[6];
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 3; ++b)
        US[a * 3 + b] = U[a * 3] * Sig[b] + U[a * 3 + 1] * Sig[3 + b] + U[a * 3 + 2] * Sig[6 + b];
    double du[6];
    for (int a = 0; a < 2; ++a)
      for (int b = 0; b < 3; ++b)
        du[a * 3 + b] = (gc[a * 2] + gc[a]) * US[b] + (gc[a * 2 + 1] + gc[2 + a]) * US[3 + b];
    double dj[6];
    for (int a = 0; a < 2; ++a)
      for (int k = 0; k < 3; ++k)
        dj[a * 3 + k] = du[a * 3] * c.R[k * 3] + du[a * 3 + 1] * c.R[k * 3 + 1] + du[a * 3 + 2] * c.R[k * 3 + 2];
    const double fx = c.fx, fy = c.fy, z2 = z * z, z3 = z2 * z;
    const double dup = raw[4], dvp = raw[5];
    double dv[3];
    dv[0] = dj[2] * (-fx / z2) * (ox ? 1.0 : 0.0) + dup * fx / z;
    dv[1] = dj[5] * (-fy / z2) * (oy ? 1.0 : 0.0) + dvp * fy / z;
    dv[2] = dj[0] * (-fx / z2) + dj[4] * (-fy / z2) +
            dj[2] * (fx * rx / z2 + (fx * x / z3) * (ox ? 1.0 : 0.0)) +
            dj[5] * (fy * ry / z2 + (fy * y / z3) * (oy ? 1.0 : 0.0)) + dup * (-fx * x / z2) +
            dvp * (-fy * y / z2);
    float4* l4 = reinterpret_cast<float4*>(in.lacc + 12 * i);
    float4 l0 = l4[0], l1 = l4[1], l2 = l4[2];
    l0.x += (float)dS[0]; l0.y += (float)dS[1]; l0.z += (float)dS[2]; l0.w += (float)dS[4];
    l1.x += (float)dS[5]; l1.y += (float)dS[8];
    // dL/dmean (world) = dv R_c
    l1.z += (float)(dv[0] * c.R[0] + dv[1] * c.R[3] + dv[2] * c.R[6]);
    l1.w += (float)(dv[0] * c.R[1] + dv[1] * c.R[4] + dv[2] * c.R[7]);
    l2.x += (float)(dv[0] * c.R[2] + dv[1] * c.R[5] + dv[2] * c.R[8]);
    l2.y += raw[0];
    l4[0] = l0; l4[1] = l1; l4[2] = l2;
  }
  if (in.dcol) return;
  if (raw[10] != 0.f) in.cacc[i] += raw[10];
  if (raw[11] != 0.f) in.cacc[n + i] += raw[11];
  if (raw[12] != 0.f) in.cacc[2 * n + i] += raw[12];
}

// mode="splat" parameter chain (grad.py:93-104 _factored_grads with
// F = Sigma = R diag(s^2) R^T, then _quat_grads): dL/dSigma -> scales,
// rotations; dL/dmean and dL/dopacity pass through; thetas / kappas get 0.
__global__ void __launch_bounds__(128) k_finalize_splat(FinalIn in, vg_grads g) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= in.n) return;
  float4* l4 = reinterpret_cast<float4*>(in.lacc + 12 * i);
  const float4 l0 = l4[0], l1 = l4[1], l2 = l4[2];
  const float raw[10] = {l0.x, l0.y, l0.z, l0.w, l1.x, l1.y, l1.z, l1.w, l2.x, l2.y};
  bool any = false;
#pragma unroll
  for (int k = 0; k < 10; ++k) any |= raw[k] != 0.f;
  const bool add = g.accumulate != 0;
  if (!any && add) return;
  if (any) {
    const float4 zf = make_float4(0.f, 0.f, 0.f, 0.f);
    l4[0] = zf; l4[1] = zf; l4[2] = zf;
  }
  double ds[3] = {0, 0, 0}, dq[4] = {0, 0, 0, 0};
  if (any) {
    double R[9], qh[4];
    quat_rotmat(in.rots + 4 * i, R, qh);
    const float* sc = in.scales + 3 * i;
    double s[3];
    for (int k = 0; k < 3; ++k) s[k] = fmax((double)sc[k], SCALE_FLOOR);
    const double G[9] = {raw[0], raw[1], raw[2], raw[1], raw[3], raw[4], raw[2], raw[4], raw[5]};
    // d_scale = diag(R^T G R) * 2 s (live scales only)
    for (int k = 0; k < 3; ++k) {
      double acc = 0.0;
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) acc += R[a * 3 + k] * G[a * 3 + b] * R[b * 3 + k];
      ds[k] = ((double)sc[k] >= SCALE_FLOOR) ? acc * 2.0 * s[k] : 0.0;
    }
    // dL/dR = (G + G^T) R diag(s^2)
    double dR[9];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) {
        double acc = 0.0;
        for (int k = 0; k < 3; ++k) acc += 2.0 * G[a * 3 + k] * R[k * 3 + b];
        dR[a * 3 + b] = acc * s[b] * s[b];
      }
    const double w = qh[0], x = qh[1], y = qh[2], z = qh[3];
    const double J[4][9] = {{0, -z, y, z, 0, -x, -y, x, 0},
                            {0, y, z, y, -2 * x, -w, z, w, -2 * x},
                            {-2 * y, x, w, x, 0, z, -w, z, -2 * y},
                            {-2 * z, -w, x, w, -2 * z, y, x, y, 0}};
    double dqh[4];
    for (int k = 0; k < 4; ++k) {
      double acc = 0;
      for (int e = 0; e < 9; ++e) acc += dR[e] * 2.0 * J[k][e];
      dqh[k] = acc;
    }
    const float* qf = in.rots + 4 * i;
    const double qn = sqrt((double)qf[0] * qf[0] + (double)qf[1] * qf[1] + (double)qf[2] * qf[2] +
                           (double)qf[3] * qf[3]);
    const double rad = qh[0] * dqh[0] + qh[1] * dqh[1] + qh[2] * dqh[2] + qh[3] * dqh[3];
    for (int k = 0; k < 4; ++k) dq[k] = (dqh[k] - qh[k] * rad) / qn;
  }
#define VG_PUT(ptr, idx, val) \
  do { if (ptr) { float _v = (float)(val); if (add) ptr[idx] += _v; else ptr[idx] = _v; } } while (0)
  for (int k = 0; k < 3; ++k) {
    VG_PUT(g.d_means, 3 * i + k, raw[6 + k]);
    VG_PUT(g.d_scales, 3 * i + k, ds[k]);
  }
  for (int k = 0; k < 4; ++k) VG_PUT(g.d_rotations, 4 * i + k, dq[k]);
  VG_PUT(g.d_thetas, i, 0.0);
  VG_PUT(g.d_kappas, i, 0.0);
  VG_PUT(g.d_splat_opacities, i, raw[9]);
#undef VG_PUT
}

// SH pull-back of the step's views, with d_v = (mean_i - centre_v) / |.| and
// the real SH basis of vg_common.cuh (DC band basis = 1):
//   d_sh[i][l][ch] (+)= sum_v b_l(d_v) dRGB_v[ch]
//   d_means[i]     +=  sum_v (I - d_v d_v^T) / |mean_i - centre_v|
//                          * sum_l grad b_l(d_v) (sum_ch sh[i][l][ch] dRGB_v[ch])
// (the colour's dependence on the view direction; RGB = sum_l b_l sh_l is
// linear, unclamped, as in preprocess).  One thread per Gaussian, 48 register
// accumulators, the per-view slabs read coalesced.
__device__ __forceinline__ void sh_basis_vjp(const float x, const float y, const float z,
                                             const float (&g)[16], float (&o)[3]) {
  const float c1 = 0.4886025119029199f, C4 = 1.0925484305920792f, C6 = 0.31539156525252005f,
              C8 = 0.5462742152960396f, C9 = -0.5900435899266435f, C10 = 2.890611442640554f,
              C11 = -0.4570457994644658f, C12 = 0.3731763325901154f, C13 = -0.4570457994644658f,
              C14 = 1.445305721320277f, C15 = -0.5900435899266435f;
  const float xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
  // d b_l / d(x, y, z) for the polynomial basis, contracted with g_l
  o[0] = -c1 * g[3] + C4 * y * g[4] - 2.f * C6 * x * g[6] - C4 * z * g[7] + 2.f * C8 * x * g[8] +
         6.f * C9 * xy * g[9] + C10 * yz * g[10] - 2.f * C11 * xy * g[11] - 6.f * C12 * xz * g[12] +
         C13 * (4.f * zz - 3.f * xx - yy) * g[13] + 2.f * C14 * xz * g[14] +
         3.f * C15 * (xx - yy) * g[15];
  o[1] = -c1 * g[1] + C4 * x * g[4] - C4 * z * g[5] - 2.f * C6 * y * g[6] - 2.f * C8 * y * g[8] +
         3.f * C9 * (xx - yy) * g[9] + C10 * xz * g[10] + C11 * (4.f * zz - xx - 3.f * yy) * g[11] -
         6.f * C12 * yz * g[12] - 2.f * C13 * xy * g[13] - 2.f * C14 * yz * g[14] -
         6.f * C15 * xy * g[15];
  o[2] = c1 * g[2] - C4 * y * g[5] + 4.f * C6 * z * g[6] - C4 * x * g[7] + C10 * xy * g[10] +
         8.f * C11 * yz * g[11] + C12 * (6.f * zz - 3.f * xx - 3.f * yy) * g[12] +
         8.f * C13 * xz * g[13] + C14 * (xx - yy) * g[14];
}

__global__ void __launch_bounds__(128) k_sh_pull(int64_t n, const float* __restrict__ means,
                                                 const float* __restrict__ sh,
                                                 const float* __restrict__ dcol,
                                                 const double* __restrict__ centers, int nviews,
                                                 float* __restrict__ d_sh, float* __restrict__ d_means,
                                                 int add) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float acc[48];
#pragma unroll
  for (int k = 0; k < 48; ++k) acc[k] = 0.f;
  float dm[3] = {0.f, 0.f, 0.f};
  const double m[3] = {means[3 * i], means[3 * i + 1], means[3 * i + 2]};
  const float4* sh4 = reinterpret_cast<const float4*>(sh + 48 * i);
  bool any = false;
  for (int v = 0; v < nviews; ++v) {
    const float* sl = dcol + (size_t)v * 3 * n;
    const float dc[3] = {sl[i], sl[n + i], sl[2 * n + i]};
    if (dc[0] == 0.f && dc[1] == 0.f && dc[2] == 0.f) continue;
    any = true;
    double d[3] = {m[0] - centers[3 * v], m[1] - centers[3 * v + 1], m[2] - centers[3 * v + 2]};
    const double dn = sqrt(dot3(d, d));
    const double idn = 1.0 / dn;
    d[0] *= idn; d[1] *= idn; d[2] *= idn;
    // the basis in float32, like the preprocess colour evaluation
    float b[16];
    sh_basis_f((float)d[0], (float)d[1], (float)d[2], b);
#pragma unroll
    for (int l = 0; l < 16; ++l) {
      const float bl = b[l];
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) acc[3 * l + ch] = fmaf(bl, dc[ch], acc[3 * l + ch]);
    }
    if (d_means) {
      // g_l = sum_ch sh[l][ch] dRGB[ch] (the coefficients re-read from L1/L2)
      float g[16];
#pragma unroll
      for (int k = 0; k < 12; ++k) {
        const float4 c = __ldg(sh4 + k);
        const float cv[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int idx = 4 * k + e, l = idx / 3, ch = idx % 3;
          g[l] = (ch == 0 ? 0.f : g[l]) + cv[e] * dc[ch];
        }
      }
      const float x = (float)d[0], y = (float)d[1], z = (float)d[2];
      float gd[3];
      sh_basis_vjp(x, y, z, g, gd);
      // through d = u / |u|: (I - d d^T) gd / |u|
      const float r = gd[0] * x + gd[1] * y + gd[2] * z;
      const float inv = (float)idn;
      dm[0] += (gd[0] - r * x) * inv;
      dm[1] += (gd[1] - r * y) * inv;
      dm[2] += (gd[2] - r * z) * inv;
    }
  }
  if (any && d_means) {
    // k_finalize_params has already written (or added) this step's geometric term
    for (int k = 0; k < 3; ++k) d_means[3 * i + k] += dm[k];
  }
  if (!d_sh || (!any && add)) return;
  float4* o = reinterpret_cast<float4*>(d_sh + 48 * i);
#pragma unroll
  for (int k = 0; k < 12; ++k) {
    float4 v = make_float4(acc[4 * k], acc[4 * k + 1], acc[4 * k + 2], acc[4 * k + 3]);
    if (add) {
      const float4 u = o[k];
      v.x += u.x; v.y += u.y; v.z += u.z; v.w += u.w;
    }
    o[k] = v;
  }
}

// Colour / SH gradients from the SoA accumulators into the caller's AoS
// layout (N*3 or N*16*3), 32 Gaussians per block transposed through shared
// memory so both sides are coalesced; zeroes the accumulators.
template <int W>
__global__ void __launch_bounds__(256) k_color_out(int64_t n, float* cacc, float* out, int add) {
  __shared__ float t[32][W + 1];
  const int64_t g0 = (int64_t)blockIdx.x * 32;
  for (int k = threadIdx.x; k < 32 * W; k += blockDim.x) {
    const int comp = k / 32, gi = k % 32;
    const int64_t g = g0 + gi;
    float v = 0.f;
    if (g < n) {
      float* p = cacc + (int64_t)comp * n + g;
      v = *p;
      if (v != 0.f) *p = 0.f;
    }
    t[gi][comp] = v;
  }
  __syncthreads();
  if (!out) return;
  for (int k = threadIdx.x; k < 32 * W; k += blockDim.x) {
    const int gi = k / W, comp = k % W;
    const int64_t g = g0 + gi;
    if (g < n) {
      float* o = out + g * W + comp;
      *o = add ? *o + t[gi][comp] : t[gi][comp];
    }
  }
}



__global__ void __launch_bounds__(128) k_finalize_params(FinalIn in, vg_grads g) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= in.n) return;
  float4* l4 = reinterpret_cast<float4*>(in.lacc + 12 * i);
  const float4 l0 = l4[0], l1 = l4[1], l2 = l4[2];
  const float raw[10] = {l0.x, l0.y, l0.z, l0.w, l1.x, l1.y, l1.z, l1.w, l2.x, l2.y};
  bool any = false;
#pragma unroll
  for (int k = 0; k < 10; ++k) any |= raw[k] != 0.f;
  const bool add = g.accumulate != 0;
  if (!any && add) return;
  if (any) {
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
    l4[0] = z; l4[1] = z; l4[2] = z;
  }
  double dmu[3] = {0, 0, 0}, ds[3] = {0, 0, 0}, dq[4] = {0, 0, 0, 0}, dth = 0, dk = 0;
  const float* sc = in.scales + 3 * i;
  if (any) {
    double R[9], qh[4];
    quat_rotmat(in.rots + 4 * i, R, qh);
    double s[3];
    for (int k = 0; k < 3; ++k) s[k] = fmax((double)sc[k], SCALE_FLOOR);
    double im, lf;
    const double theta = in.thetas[i];
    const double kappa = kappa_of(theta, s, &im, &lf);
    const double k2 = -0.5 * kappa * SQRT_2PI;
    const double Al[9] = {k2 * raw[0], k2 * raw[1], k2 * raw[2], k2 * raw[1], k2 * raw[3],
                          k2 * raw[4], k2 * raw[2], k2 * raw[4], k2 * raw[5]};
    const double Bl[3] = {k2 * raw[6], k2 * raw[7], k2 * raw[8]};
    dk = SQRT_2PI * (double)raw[9];
    // dL/dmean = 2 R S^-1 B_loc
    for (int a = 0; a < 3; ++a) {
      double acc = 0;
      for (int k = 0; k < 3; ++k) acc += R[a * 3 + k] * Bl[k] / s[k];
      dmu[a] = 2.0 * acc;
    }
    // theta / scale chains (grad.py:248-257)
    dth = dk * im * THETA_CEILING / (1.0 - THETA_CEILING * theta);
    for (int k = 0; k < 3; ++k) {
      const double dsk = dk * (-lf / (3.0 * s[k] * s[k])) + (-2.0 * Al[k * 4] / s[k]);
      ds[k] = ((double)sc[k] >= SCALE_FLOOR) ? dsk : 0.0;
    }
    // dL/dR = 2 R S A_loc S^-1  (= (G + G^T) R diag(1/s^2), G = R S A S R^T)
    double dR[9];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) {
        double acc = 0;
        for (int k = 0; k < 3; ++k) acc += R[a * 3 + k] * s[k] * Al[k * 3 + b];
        dR[a * 3 + b] = 2.0 * acc / s[b];
      }
    // _quat_grads / _rotmat_quat_jacobian (grad.py:72-90)
    const double w = qh[0], x = qh[1], y = qh[2], z = qh[3];
    const double J[4][9] = {{0, -z, y, z, 0, -x, -y, x, 0},
                            {0, y, z, y, -2 * x, -w, z, w, -2 * x},
                            {-2 * y, x, w, x, 0, z, -w, z, -2 * y},
                            {-2 * z, -w, x, w, -2 * z, y, x, y, 0}};
    double dqh[4];
    for (int k = 0; k < 4; ++k) {
      double acc = 0;
      for (int e = 0; e < 9; ++e) acc += dR[e] * 2.0 * J[k][e];
      dqh[k] = acc;
    }
    const float* qf = in.rots + 4 * i;
    const double qn = sqrt((double)qf[0] * qf[0] + (double)qf[1] * qf[1] + (double)qf[2] * qf[2] +
                           (double)qf[3] * qf[3]);
    const double rad = qh[0] * dqh[0] + qh[1] * dqh[1] + qh[2] * dqh[2] + qh[3] * dqh[3];
    for (int k = 0; k < 4; ++k) dq[k] = (dqh[k] - qh[k] * rad) / qn;
  }
#define VG_PUT(ptr, idx, val) \
  do { if (ptr) { float _v = (float)(val); if (add) ptr[idx] += _v; else ptr[idx] = _v; } } while (0)
  for (int k = 0; k < 3; ++k) {
    VG_PUT(g.d_means, 3 * i + k, dmu[k]);
    VG_PUT(g.d_scales, 3 * i + k, ds[k]);
  }
  for (int k = 0; k < 4; ++k) VG_PUT(g.d_rotations, 4 * i + k, dq[k]);
  VG_PUT(g.d_thetas, i, dth);
  VG_PUT(g.d_kappas, i, dk);
#undef VG_PUT
}

void launch_view_accumulate(int64_t n, const vg_scene& s, const CamK& c, const float* frame,
                            float* acc, float* lacc, float* cacc, float* dcol, double* center,
                            bool splat, cudaStream_t st, const SegIO* seg) {
  if (n <= 0) return;
  ViewAccIn in{n, s.means, s.scales, s.rotations, s.sh, frame, acc, lacc, cacc, dcol, center,
               seg ? seg->counts : nullptr, seg ? seg->decision : nullptr, seg ? seg->slots : 1u,
               seg ? seg->ratio : 1.f};
  if (splat) {
    k_view_accumulate_splat<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(in, c);
    return;
  }
  k_view_accumulate<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(in, c);
}

// dst += src, src = 0 (merging the deferred accumulators of two contexts)
__global__ void __launch_bounds__(256) k_merge_acc(int64_t n4, float4* __restrict__ dst,
                                                   float4* __restrict__ src) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n4) return;
  const float4 a = src[i];
  float4 b = dst[i];
  b.x += a.x; b.y += a.y; b.z += a.z; b.w += a.w;
  dst[i] = b;
  src[i] = make_float4(0.f, 0.f, 0.f, 0.f);
}

__global__ void k_merge_acc_tail(int64_t n, float* __restrict__ dst, float* __restrict__ src) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  dst[i] += src[i];
  src[i] = 0.f;
}

void launch_merge_acc(int64_t n, float* dst, float* src, cudaStream_t st) {
  if (n <= 0) return;
  const bool aligned = ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) == 0;
  const int64_t n4 = aligned ? n / 4 : 0;
  if (n4)
    k_merge_acc<<<(unsigned)((n4 + 255) / 256), 256, 0, st>>>(n4, reinterpret_cast<float4*>(dst),
                                                             reinterpret_cast<float4*>(src));
  const int64_t rest = n - 4 * n4;
  if (rest)
    k_merge_acc_tail<<<(unsigned)((rest + 255) / 256), 256, 0, st>>>(rest, dst + 4 * n4, src + 4 * n4);
}

int launch_finalize_params(int64_t n, const vg_scene& s, float* lacc, float* cacc,
                           const float* dcol, const double* centers, int sh_views,
                           const vg_grads& g, bool splat, cudaStream_t st) {
  if (n <= 0) return 0;
  FinalIn in{n, s.scales, s.rotations, s.thetas, lacc};
  if (splat)
    k_finalize_splat<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(in, g);
  else
    k_finalize_params<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(in, g);
  if (!splat && g.d_splat_opacities && g.accumulate == 0)
    cudaMemsetAsync(g.d_splat_opacities, 0, sizeof(float) * (size_t)n, st);
  const unsigned blocks = (unsigned)((n + 31) / 32);
  const int add = g.accumulate != 0;
  if (s.sh) {
    if (g.d_sh || g.d_means)
      k_sh_pull<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(n, s.means, s.sh, dcol, centers, sh_views,
                                                            g.d_sh, g.d_means, add);
    // d_colors (dL/d evaluated RGB) is not tracked separately for SH scenes
    if (g.d_colors && !add) cudaMemsetAsync(g.d_colors, 0, sizeof(float) * 3 * (size_t)n, st);
  } else {
    k_color_out<3><<<blocks, 256, 0, st>>>(n, cacc, g.d_colors, add);
  }
  return 2;
}

}  // namespace vg
