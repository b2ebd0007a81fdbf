// K1b: blend records for the binned Gaussians (float64 with FMA contraction,
// one thread per Gaussian; unbinned ones exit at once).  Builds the
// whitening frame of vg_common.cuh (make_frame), the 80-byte record the tile
// kernels stage, the e-frame K7 rotates gradients with, and the per-view RGB
// (SH-3 evaluated when present).  Its arithmetic does not affect tile lists,
// so unlike vg_preprocess.cu it is compiled with the default -fmad=true.
#include "vg_kernels.cuh"

namespace vg {

__global__ void __launch_bounds__(256) k_records(int64_t n, const float* __restrict__ means,
                                                 const float* __restrict__ scales,
                                                 const float* __restrict__ rots,
                                                 const float* __restrict__ thetas,
                                                 const float* __restrict__ colors,
                                                 const float* __restrict__ sh, CamK c,
                                                 const uint32_t* __restrict__ count,
                                                 GRec* __restrict__ rec, float* __restrict__ frame) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || !count[i]) return;
  Frame f;
  make_frame(c, means + 3 * i, scales + 3 * i, rots + 4 * i, f);
  const double kappa = kappa_of((double)thetas[i], f.s, nullptr, nullptr);
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
    double d[3] = {means[3 * i] - c.center[0], means[3 * i + 1] - c.center[1],
                   means[3 * i + 2] - c.center[2]};
    const double dn = sqrt(dot3(d, d));
    d[0] /= dn; d[1] /= dn; d[2] /= dn;
    double b[16];
    sh_basis(d, b);
    // 192 contiguous bytes per Gaussian: 12 x 16-byte loads (not 48 scalar ones)
    const float4* q4 = reinterpret_cast<const float4*>(sh + 48 * i);
    float q[48];
#pragma unroll
    for (int k = 0; k < 12; ++k) {
      const float4 v = __ldg(q4 + k);
      q[4 * k] = v.x; q[4 * k + 1] = v.y; q[4 * k + 2] = v.z; q[4 * k + 3] = v.w;
    }
#pragma unroll
    for (int l = 0; l < 16; ++l)
      for (int ch = 0; ch < 3; ++ch) rgb[ch] += b[l] * q[l * 3 + ch];
  } else if (colors) {
    rgb[0] = colors[3 * i]; rgb[1] = colors[3 * i + 1]; rgb[2] = colors[3 * i + 2];
  }
  float4* fr = reinterpret_cast<float4*>(frame + 12 * i);
  fr[0] = make_float4((float)f.e[0], (float)f.e[1], (float)f.e[2], (float)f.e[3]);
  fr[1] = make_float4((float)f.e[4], (float)f.e[5], (float)f.e[6], (float)f.e[7]);
  fr[2] = make_float4((float)f.e[8], 0.f, 0.f, 0.f);
  g.cr = (float)rgb[0];
  g.cg = (float)rgb[1];
  g.cb = (float)rgb[2];
  rec[i] = g;
}

void launch_records(int64_t n, const vg_scene& s, const CamK& c, const uint32_t* count, GRec* rec,
                    float* frame, cudaStream_t st) {
  if (n <= 0) return;
  k_records<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, s.means, s.scales, s.rotations,
                                                          s.thetas, s.colors, s.sh, c, count, rec,
                                                          frame);
}

}  // namespace vg
