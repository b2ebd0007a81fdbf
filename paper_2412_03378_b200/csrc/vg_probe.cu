// Roofline denominators for the blend kernels, measured on the device at its
// live clock: FP32 FFMA issue throughput and MUFU (ex2) throughput.
// MEASURED_PEAKS.json carries only HBM and bf16 GEMM peaks, while the blend
// kernels are FP32 / SFU bound.
#include <cuda_runtime.h>

#include "vg_kernels.cuh"

namespace vg {

template <int KIND>
__global__ void __launch_bounds__(256) k_probe(float seed, int iters, float* sink) {
  float a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = seed + threadIdx.x * 1e-3f + j;
  if (KIND == 0) {
    const float m = 0.99999f, c = 1e-6f;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int j = 0; j < 8; ++j) a[j] = fmaf(a[j], m, c);
    }
  } else {
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int j = 0; j < 8; ++j) a[j] = ex2f(-a[j]);
    }
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += a[j];
  if (s == 12345.f) sink[threadIdx.x] = s;
}

}  // namespace vg

extern "C" int vg_probe_peaks(int32_t device, double* fp32_per_s, double* mufu_per_s) {
  using namespace vg;
  if (cudaSetDevice(device) != cudaSuccess) return VG_ECUDA;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  float* sink = nullptr;
  if (cudaMalloc(&sink, 1024 * sizeof(float)) != cudaSuccess) return VG_ECUDA;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = sms * 8, threads = 256;
  double res[2] = {0, 0};
  for (int kind = 0; kind < 2; ++kind) {
    const int iters = kind == 0 ? 8192 : 2048;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      if (kind == 0) k_probe<0><<<blocks, threads>>>(0.5f, iters, sink);
      else k_probe<1><<<blocks, threads>>>(0.5f, iters, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      double ops = (double)blocks * threads * iters * 8;
      double r = ops / (ms * 1e-3);
      if (r > res[kind]) res[kind] = r;
    }
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(sink);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return VG_ECUDA;
  *fp32_per_s = res[0];
  *mufu_per_s = res[1];
  return VG_OK;
}
