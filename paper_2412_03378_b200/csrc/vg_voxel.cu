// Mixture density on a voxel grid (tomo.voxelize, tomo.py:345-389): every
// primitive adds kappa exp(-q/2) to the voxel centres inside a world box of
// CULL_SIGMAS = 5 largest standard deviations around its mean where
// q = (x - mu)^T M (x - mu) <= 25; the box's index range is the reference's
// searchsorted over the cell-centred axes, evaluated exactly on the same
// float64 centres.  One CTA per primitive, float64 throughout, float64
// atomics into the grid (the summation order of overlapping primitives is
// not fixed: results agree with the reference to float64 rounding).
#include <cmath>

#include "vg_kernels.cuh"

namespace vg {
namespace voxel {

constexpr double CULL_SIGMAS = 5.0;

struct Axes {
  double bmin[3], sp[3];
  int n[3];
};

__device__ __forceinline__ double centre(const Axes& a, int ax, int k) {
  return a.bmin[ax] + ((double)k + 0.5) * a.sp[ax];
}

// numpy.searchsorted(axis_centres, v, side="left" | "right") for one key --
// the plain binary search numpy runs, so it agrees with the reference on any
// box: ascending (the usual case: the count of centres < v, resp. <= v), and
// also degenerate (zero spacing: every centre at bbox_min) or reversed
// (descending centres), which tomo.voxelize accepts unchecked
__device__ __forceinline__ int count_below(const Axes& a, int ax, double v, bool inclusive) {
  int lo = 0, hi = a.n[ax];
  while (lo < hi) {
    const int mid = lo + ((hi - lo) >> 1);
    const double c = centre(a, ax, mid);
    if (inclusive ? c <= v : c < v) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__global__ void __launch_bounds__(256) k_voxelize(vg_scene s, Axes a, double* __restrict__ out) {
  const int64_t i = blockIdx.x;
  double R[9];
  quat_rotmat(s.rotations + 4 * i, R, nullptr);
  double sv[3], inv[3];
  for (int k = 0; k < 3; ++k) {
    sv[k] = fmax((double)s.scales[3 * i + k], SCALE_FLOOR);
    inv[k] = 1.0 / (sv[k] * sv[k]);
  }
  double M[9];
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      double acc = 0.0;
      for (int k = 0; k < 3; ++k) acc += R[r * 3 + k] * inv[k] * R[c * 3 + k];
      M[r * 3 + c] = acc;
    }
  const double kappa = kappa_of((double)s.thetas[i], sv, nullptr, nullptr);
  const double reach = CULL_SIGMAS * fmax(sv[0], fmax(sv[1], sv[2]));
  const double mu[3] = {(double)s.means[3 * i], (double)s.means[3 * i + 1], (double)s.means[3 * i + 2]};
  int lo[3], cnt[3];
  for (int ax = 0; ax < 3; ++ax) {
    lo[ax] = count_below(a, ax, mu[ax] - reach, false);
    const int hi = count_below(a, ax, mu[ax] + reach, true);
    cnt[ax] = hi - lo[ax];
    if (cnt[ax] <= 0) return;
  }
  const int64_t total = (int64_t)cnt[0] * cnt[1] * cnt[2];
  for (int64_t t = threadIdx.x; t < total; t += blockDim.x) {
    const int iz = (int)(t % cnt[2]) + lo[2];
    const int64_t r = t / cnt[2];
    const int iy = (int)(r % cnt[1]) + lo[1];
    const int ix = (int)(r / cnt[1]) + lo[0];
    const double d[3] = {centre(a, 0, ix) - mu[0], centre(a, 1, iy) - mu[1], centre(a, 2, iz) - mu[2]};
    double Md[3];
    matvec3(M, d, Md);
    const double q = dot3(d, Md);
    if (q <= CULL_SIGMAS * CULL_SIGMAS)
      atomicAdd(out + ((int64_t)ix * a.n[1] + iy) * a.n[2] + iz, kappa * exp(-0.5 * q));
  }
}

}  // namespace voxel
}  // namespace vg

extern "C" int vg_voxelize(const vg_scene* s, const double* bbox_min, const double* bbox_max,
                           const int32_t* shape, double* out, void* stream) {
  using namespace vg;
  if (!s || !bbox_min || !bbox_max || !shape || !out) return set_error(VG_EINVAL, "vg_voxelize: NULL argument");
  voxel::Axes a;
  for (int k = 0; k < 3; ++k) {
    if (shape[k] <= 0) return set_error(VG_EINVAL, "vg_voxelize: resolution must be positive");
    a.n[k] = shape[k];
    a.bmin[k] = bbox_min[k];
    a.sp[k] = (bbox_max[k] - bbox_min[k]) / (double)shape[k];
  }
  if (s->n > 0 && (!s->means || !s->scales || !s->rotations || !s->thetas))
    return set_error(VG_EINVAL, "vg_voxelize: scene arrays must be non-NULL");
  cudaStream_t st = (cudaStream_t)stream;
  const size_t cells = (size_t)shape[0] * shape[1] * shape[2];
  if (cudaMemsetAsync(out, 0, sizeof(double) * cells, st) != cudaSuccess)
    return set_error(VG_ECUDA, "vg_voxelize: memset failed");
  if (s->n > 0) voxel::k_voxelize<<<(unsigned)s->n, 256, 0, st>>>(*s, a, out);
  return cudaGetLastError() == cudaSuccess ? VG_OK : set_error(VG_ECUDA, "vg_voxelize: launch failed");
}
