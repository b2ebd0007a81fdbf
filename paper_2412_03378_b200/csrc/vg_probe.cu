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

// ---------------------------------------------------------------------------
// Streaming copy between device memory and pinned (mapped) host memory by a
// small kernel: the device-side reads / writes carry evict-first cache hints
// (__ldcs / __stcs), so a host download does not flush the L2 working set of
// the kernels running beside it (a copy-engine transfer passes through L2).
namespace vg {
__global__ void __launch_bounds__(256) k_copy_stream(const float4* __restrict__ src,
                                                     float4* __restrict__ dst, int64_t n4) {
  // four independent 16-byte loads in flight per thread (host memory is ~1 us away)
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n4; i += 4 * stride) {
    const float4 a = __ldcs(src + i), b = __ldcs(src + i + stride), c = __ldcs(src + i + 2 * stride),
                 d = __ldcs(src + i + 3 * stride);
    __stcs(dst + i, a);
    __stcs(dst + i + stride, b);
    __stcs(dst + i + 2 * stride, c);
    __stcs(dst + i + 3 * stride, d);
  }
  for (; i < n4; i += stride) __stcs(dst + i, __ldcs(src + i));
}
__global__ void k_copy_stream_tail(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[i];
}
}  // namespace vg

extern "C" int vg_copy_streaming(void* dst, const void* src, size_t bytes, int32_t ctas, void* stream) {
  using namespace vg;
  if ((!dst || !src) && bytes) return set_error(VG_EINVAL, "vg_copy_streaming: NULL pointer");
  if (bytes == 0) return VG_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const bool aligned = ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) == 0;
  const int64_t n4 = aligned ? (int64_t)(bytes / 16) : 0;
  if (n4)
    k_copy_stream<<<ctas > 0 ? ctas : 16, 256, 0, st>>>(reinterpret_cast<const float4*>(src),
                                                         reinterpret_cast<float4*>(dst), n4);
  const int64_t rest = (int64_t)bytes - 16 * n4;
  if (rest)
    k_copy_stream_tail<<<(unsigned)((rest + 255) / 256), 256, 0, st>>>(
        reinterpret_cast<const uint8_t*>(src) + 16 * n4, reinterpret_cast<uint8_t*>(dst) + 16 * n4, rest);
  return cudaGetLastError() == cudaSuccess ? VG_OK : set_error(VG_ECUDA, "vg_copy_streaming: launch failed");
}
