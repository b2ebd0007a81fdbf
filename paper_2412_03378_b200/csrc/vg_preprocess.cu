// K1: per-Gaussian preprocessing (float64), one thread per Gaussian.
//
// Replaces raster.prepare's per-primitive half (raster.py:154-209, 263-288;
// core.py:81-153): view transform, validity z > z_near, EWA screen
// covariance with 0.3 px^2 dilation, lambda_max, the amplitude-aware bin
// radius, the tile rectangle and its tile count, kappa, and the 64-byte blend
// record the tile kernels gather.  Compiled with -fmad=false so the binning
// arithmetic rounds like the reference's numpy float64 (tile lists must match
// bit for bit).
#include "vg_kernels.cuh"

namespace vg {

struct PrepOut {
  GRec* rec;
  float* depth;        // sort key (float32 view depth)
  ushort4* rect;       // tile rectangle x0, y0, x1, y1 (inclusive); x1 < x0: not binned
  double* gm;          // sort_by="gamma" only: M (xx, xy, xz, yy, yz, zz) and M (mean - centre)
  float* frame;        // e1, e2, e3 in whitened-local coordinates (12 floats)
};

#ifndef VG_PRE_NT
#define VG_PRE_NT 64  // threads per CTA (A/B, 16 views of config 3: 256x3 CTAs 1.96 ms, 128x5 1.86, 64x10 1.84)
#endif
#ifndef VG_PRE_MINB
#define VG_PRE_MINB 10  // <= 96 registers (80 spilled ~350 bytes per thread)
#endif

__global__ void __launch_bounds__(VG_PRE_NT, VG_PRE_MINB) k_preprocess(int64_t n, const float* __restrict__ means,
                                                    const float* __restrict__ scales,
                                                    const float* __restrict__ rots,
                                                    const float* __restrict__ thetas,
                                                    const float* __restrict__ colors,
                                                    const float* __restrict__ sh,
                                                    const float* __restrict__ opac, CamK c,
                                                    double bin_cut, PrepOut o) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  Frame f;
  bool ok = make_frame(c, means + 3 * i, scales + 3 * i, rots + 4 * i, f);
  uint32_t cnt = 0;
  ushort4 rect = make_ushort4(1, 0, 0, 0);
  double conic[3] = {0.0, 0.0, 0.0}, lam_max = 1.0;
  double kappa = kappa_of((double)thetas[i], f.s, nullptr, nullptr);
  if (ok) {
    // --- EWA screen covariance (raster.py:175-209) or orthographic projection
    double Sig[9];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) {
        double acc = 0.0;
        for (int k = 0; k < 3; ++k) acc += f.R[a * 3 + k] * (f.s[k] * f.s[k]) * f.R[b * 3 + k];
        Sig[a * 3 + b] = acc;
      }
    double U[6];
    if (c.projection == VG_PINHOLE) {
      double z = f.v[2];
      double limx = 1.3 * (0.5 * c.width / c.fx), limy = 1.3 * (0.5 * c.height / c.fy);
      double rx = fmin(fmax(f.v[0] / z, -limx), limx);
      double ry = fmin(fmax(f.v[1] / z, -limy), limy);
      double J[6] = {c.fx / z, 0.0, -c.fx * rx / z, 0.0, c.fy / z, -c.fy * ry / z};
      for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 3; ++b)
          U[a * 3 + b] = J[a * 3 + 0] * c.R[0 * 3 + b] + J[a * 3 + 1] * c.R[1 * 3 + b] +
                         J[a * 3 + 2] * c.R[2 * 3 + b];
    } else {
      double sx = c.width / (2.0 * c.extent), sy = c.height / (2.0 * c.extent);
      for (int b = 0; b < 3; ++b) { U[b] = sx * c.R[b]; U[3 + b] = sy * c.R[3 + b]; }
    }
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
    // --- bounding radius (raster.py:154-172)
    double half_tr = 0.5 * (cov[0] + cov[3]);
    double det = cov[0] * cov[3] - cov[1] * cov[2];
    double lam = half_tr + sqrt(fmax(half_tr * half_tr - det, 0.0));
    lam_max = lam;
    if (opac) {  // the splat record's conic (raster._inv2x2, raster.py:212-219)
      conic[0] = cov[3] / det;
      conic[1] = -cov[1] / det;
      conic[2] = cov[0] / det;
    }
    double smax = fmax(fmax(f.s[0], f.s[1]), f.s[2]);
    double amp = SQRT_2PI * kappa * smax;
    double cut = fmax(bin_cut, 1e-12);
    double need = sqrt(2.0 * log(fmax(1.05 * amp / cut, 1.0)));
    // splat alphas are bounded by the opacity <= 1: 3 sigma (raster.py:154-172)
    double mult = opac ? BASE_SIGMA : fmax(BASE_SIGMA, need + 0.5);
    double r = mult * sqrt(lam);
    // --- tile rectangle (raster.py:233-244)
    double u = f.pu, v = f.pv;
    bool outside = (u + r < 0.0) || (u - r >= c.width) || (v + r < 0.0) || (v - r >= c.height);
    if (!outside) {
      double fx0 = fmin(fmax(floor((u - r) / TILE), 0.0), (double)(c.ntx - 1));
      double fx1 = fmin(fmax(floor((u + r) / TILE), 0.0), (double)(c.ntx - 1));
      double fy0 = fmin(fmax(floor((v - r) / TILE), 0.0), (double)(c.nty - 1));
      double fy1 = fmin(fmax(floor((v + r) / TILE), 0.0), (double)(c.nty - 1));
      rect = make_ushort4((unsigned short)fx0, (unsigned short)fy0, (unsigned short)fx1,
                          (unsigned short)fy1);
      cnt = (uint32_t)(rect.z - rect.x + 1) * (uint32_t)(rect.w - rect.y + 1);
    }
  }
  o.rect[i] = rect;
  o.depth[i] = (float)f.v[2];
  if (!cnt) return;
  if (opac) {
    // splat record (vg_splat.cu): the conic (raster._inv2x2, raster.py:212-219),
    // opacity, lambda_min(conic) for culling, colour
    GRec g{};
    g.u = f.pu;
    g.v = f.pv;
    g.P11 = (float)(conic[0]);
    g.P21 = (float)(conic[1]);
    g.P22 = (float)(conic[2]);
    g.kap2 = opac[i];
    g.amp = opac[i];
    g.n1 = (float)(1.0 / lam_max);
    if (colors) { g.cr = colors[3 * i]; g.cg = colors[3 * i + 1]; g.cb = colors[3 * i + 2]; }
    if (sh) {
      double d[3] = {means[3 * i] - c.center[0], means[3 * i + 1] - c.center[1],
                     means[3 * i + 2] - c.center[2]};
      const double dn = sqrt(dot3(d, d));
      d[0] /= dn; d[1] /= dn; d[2] /= dn;
      double b[16], rgb[3] = {0.0, 0.0, 0.0};
      sh_basis(d, b);
      for (int l = 0; l < 16; ++l)
        for (int ch = 0; ch < 3; ++ch) rgb[ch] += b[l] * sh[48 * i + 3 * l + ch];
      g.cr = (float)rgb[0]; g.cg = (float)rgb[1]; g.cb = (float)rgb[2];
    }
    o.rec[i] = g;
    return;
  }
  if (o.gm) {
    // core.precision_matrices (core.py:111-119) and raster.prepare's
    // minv_delta (raster.py:276-280), for the gamma re-sort
    double M[9];
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) {
        double acc = 0.0;
        for (int k = 0; k < 3; ++k) acc += f.R[a * 3 + k] * (1.0 / (f.s[k] * f.s[k])) * f.R[b * 3 + k];
        M[a * 3 + b] = acc;
      }
    const double dl[3] = {(double)means[3 * i] - c.center[0], (double)means[3 * i + 1] - c.center[1],
                          (double)means[3 * i + 2] - c.center[2]};
    double* q = o.gm + 9 * i;
    q[0] = M[0]; q[1] = M[1]; q[2] = M[2]; q[3] = M[4]; q[4] = M[5]; q[5] = M[8];
    for (int a = 0; a < 3; ++a) q[6 + a] = M[a * 3] * dl[0] + M[a * 3 + 1] * dl[1] + M[a * 3 + 2] * dl[2];
  }
  // --- blend record
  GRec g;
  g.u = f.pu;
  g.v = f.pv;
  g.P11 = (float)f.P11;
  g.P21 = (float)f.P21;
  g.P22 = (float)f.P22;
  g.n1 = (float)f.n1;
  g.n2 = (float)f.n2;
  g.wm = (float)f.wm;
  g.cD2 = (float)(0.5 * LOG2E * f.D * f.D);
  g.D = (float)(c.projection == VG_PINHOLE ? f.D : f.beta);
  g.kap2 = (float)(kappa * SQRT_2PI * LOG2E);
  g.amp = (float)(SQRT_2PI * kappa * fmax(fmax(f.s[0], f.s[1]), f.s[2]));
  g.pad0 = g.pad1 = g.pad2 = 0.f;
  double rgb[3] = {0.0, 0.0, 0.0};
  if (sh) {
    // SH-3 colour (no reference counterpart): the direction in float64, the
    // basis and the 48-term contraction in float32 with explicit FMAs (this
    // file is built without FMA contraction for the binning's sake; float64
    // without FMAs made the contraction ~300 float64 operations per Gaussian)
    double d[3] = {means[3 * i] - c.center[0], means[3 * i + 1] - c.center[1],
                   means[3 * i + 2] - c.center[2]};
    const double idn = 1.0 / sqrt(dot3(d, d));
    float b[16];
    sh_basis_f((float)(d[0] * idn), (float)(d[1] * idn), (float)(d[2] * idn), b);
    // 192 contiguous bytes per Gaussian: 12 x 16-byte loads (not 48 scalar ones)
    // (each loaded value is folded in at once: no 48-float array to hold)
    const float4* q4 = reinterpret_cast<const float4*>(sh + 48 * i);
    float rf[3] = {0.f, 0.f, 0.f};
#pragma unroll
    for (int k = 0; k < 12; ++k) {
      const float4 v = __ldg(q4 + k);
      const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int idx = 4 * k + e;
        rf[idx % 3] = fmaf(b[idx / 3], vv[e], rf[idx % 3]);
      }
    }
    rgb[0] = rf[0]; rgb[1] = rf[1]; rgb[2] = rf[2];
  } else if (colors) {
    rgb[0] = colors[3 * i]; rgb[1] = colors[3 * i + 1]; rgb[2] = colors[3 * i + 2];
  }
  float4* fr = reinterpret_cast<float4*>(o.frame + 12 * i);
  fr[0] = make_float4((float)f.e[0], (float)f.e[1], (float)f.e[2], (float)f.e[3]);
  fr[1] = make_float4((float)f.e[4], (float)f.e[5], (float)f.e[6], (float)f.e[7]);
  fr[2] = make_float4((float)f.e[8], 0.f, 0.f, 0.f);
  g.cr = (float)rgb[0];
  g.cg = (float)rgb[1];
  g.cb = (float)rgb[2];
  o.rec[i] = g;
}

void launch_preprocess(int64_t n, const vg_scene& s, const CamK& c, double bin_cut, GRec* rec,
                       float* depth, ushort4* rect, float* frame, double* gm, bool splat,
                       cudaStream_t st) {
  if (n <= 0) return;
  PrepOut o{rec, depth, rect, gm, frame};
  int blocks = (int)((n + VG_PRE_NT - 1) / VG_PRE_NT);
  k_preprocess<<<blocks, VG_PRE_NT, 0, st>>>(n, s.means, s.scales, s.rotations, s.thetas, s.colors,
                                       s.sh, splat ? s.splat_opacities : nullptr, c, bin_cut, o);
}

}  // namespace vg
