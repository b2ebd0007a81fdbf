// K1: per-Gaussian preprocessing (float64), one thread per Gaussian.
//
// Replaces raster.prepare's per-primitive half (raster.py:154-209, 263-288;
// core.py:81-153): view transform, validity z > z_near, EWA screen
// covariance with 0.3 px^2 dilation, lambda_max, the amplitude-aware bin
// radius, the tile rectangle and its tile count, kappa, and the 64-byte blend
// record the tile kernels gather.  This translation unit holds only the
// binning half and is compiled with -fmad=false so its arithmetic rounds like
// the reference's numpy float64 (tile lists must match bit for bit); the blend
// records are built by vg_records.cu (FMA allowed) for binned Gaussians only.
#include "vg_kernels.cuh"

namespace vg {

struct PrepOut {
  GRec* rec;
  float* depth;        // sort key (float32 view depth)
  int4* rect;          // tile rectangle x0, y0, x1, y1 (inclusive)
  uint32_t* count;     // tiles overlapped (0 = not binned)
  float* frame;        // e1, e2, e3 in whitened-local coordinates (12 floats)
};

__global__ void __launch_bounds__(256) k_preprocess(int64_t n, const float* __restrict__ means,
                                                    const float* __restrict__ scales,
                                                    const float* __restrict__ rots,
                                                    const float* __restrict__ thetas,
                                                    const float* __restrict__ colors,
                                                    const float* __restrict__ sh, CamK c,
                                                    double bin_cut, PrepOut o) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  Frame f;
  // binning needs only R, s and the view-space mean (raster.py:175-209)
  quat_rotmat(rots + 4 * i, f.R, nullptr);
  for (int k = 0; k < 3; ++k) f.s[k] = fmax((double)scales[3 * i + k], SCALE_FLOOR);
  {
    const double m3[3] = {means[3 * i], means[3 * i + 1], means[3 * i + 2]};
    for (int j = 0; j < 3; ++j)
      f.v[j] = c.R[j * 3 + 0] * m3[0] + c.R[j * 3 + 1] * m3[1] + c.R[j * 3 + 2] * m3[2] + c.t[j];
  }
  bool ok = c.projection != VG_PINHOLE || f.v[2] > c.z_near;
  if (c.projection == VG_PINHOLE) {
    f.pu = c.fx * f.v[0] / f.v[2] + c.cx;
    f.pv = c.fy * f.v[1] / f.v[2] + c.cy;
  } else {
    f.pu = (f.v[0] / c.extent + 1.0) * 0.5 * c.width;
    f.pv = (f.v[1] / c.extent + 1.0) * 0.5 * c.height;
  }
  uint32_t cnt = 0;
  int4 rect = make_int4(0, 0, -1, -1);
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
    double smax = fmax(fmax(f.s[0], f.s[1]), f.s[2]);
    double amp = SQRT_2PI * kappa * smax;
    double cut = fmax(bin_cut, 1e-12);
    double need = sqrt(2.0 * log(fmax(1.05 * amp / cut, 1.0)));
    double mult = fmax(BASE_SIGMA, need + 0.5);
    double r = mult * sqrt(lam);
    // --- tile rectangle (raster.py:233-244)
    double u = f.pu, v = f.pv;
    bool outside = (u + r < 0.0) || (u - r >= c.width) || (v + r < 0.0) || (v - r >= c.height);
    if (!outside) {
      double fx0 = fmin(fmax(floor((u - r) / TILE), 0.0), (double)(c.ntx - 1));
      double fx1 = fmin(fmax(floor((u + r) / TILE), 0.0), (double)(c.ntx - 1));
      double fy0 = fmin(fmax(floor((v - r) / TILE), 0.0), (double)(c.nty - 1));
      double fy1 = fmin(fmax(floor((v + r) / TILE), 0.0), (double)(c.nty - 1));
      rect = make_int4((int)fx0, (int)fy0, (int)fx1, (int)fy1);
      cnt = (uint32_t)((rect.z - rect.x + 1) * (rect.w - rect.y + 1));
    }
  }
  o.count[i] = cnt;
  o.rect[i] = rect;
  o.depth[i] = (float)f.v[2];
}

void launch_preprocess(int64_t n, const vg_scene& s, const CamK& c, double bin_cut, GRec* rec,
                       float* depth, int4* rect, uint32_t* count, float* frame, cudaStream_t st) {
  if (n <= 0) return;
  PrepOut o{rec, depth, rect, count, frame};
  int blocks = (int)((n + 255) / 256);
  k_preprocess<<<blocks, 256, 0, st>>>(n, s.means, s.scales, s.rotations, s.thetas, s.colors,
                                       s.sh, c, bin_cut, o);
  launch_records(n, s, c, count, rec, frame, st);
}

}  // namespace vg
