// Standalone A/B timing of the Gaussian depth sort: CUB onesweep (library,
// reference point only; not linked into the product) against the
// hand-written onesweep of vg_radix.cu (the product path) on N positive float
// depths; both must give the stable order.
//   tools/build_sortbench.sh
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>

#include "vg_kernels.cuh"

#define CK(x)                                                              \
  do {                                                                     \
    cudaError_t e = (x);                                                   \
    if (e != cudaSuccess) {                                                \
      printf("%s: %s\n", #x, cudaGetErrorString(e));                       \
      exit(1);                                                             \
    }                                                                      \
  } while (0)

template <typename F>
static float timeit(F f, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  CK(cudaDeviceSynchronize());
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) f();
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms * 1000.f / reps;
}

int main(int argc, char** argv) {
  const int64_t N = argc > 1 ? atoll(argv[1]) : 1000000;
  const float zlo = argc > 2 ? atof(argv[2]) : 1.f, zhi = argc > 3 ? atof(argv[3]) : 12.f;
  std::mt19937 rng(1);
  std::vector<uint32_t> hd(N), hid(N);
  std::uniform_real_distribution<float> U(zlo, zhi);
  for (int64_t i = 0; i < N; ++i) {
    float z = U(rng);
    if (i % 1000 == 7) z = U(rng);  // plus exact duplicates below
    if (i % 997 == 3 && i > 0) memcpy(&z, &hd[i - 1], 4);
    memcpy(&hd[i], &z, 4);
    hid[i] = (uint32_t)i;
  }
  std::vector<uint32_t> ord(N);
  for (int64_t i = 0; i < N; ++i) ord[i] = (uint32_t)i;
  std::stable_sort(ord.begin(), ord.end(), [&](uint32_t a, uint32_t b) { return hd[a] < hd[b]; });

  uint32_t *dsrc, *dk0, *dk1, *dv0, *dv1;
  CK(cudaMalloc(&dsrc, 4 * N));
  CK(cudaMalloc(&dk0, 4 * N));
  CK(cudaMalloc(&dk1, 4 * N));
  CK(cudaMalloc(&dv0, 4 * N));
  CK(cudaMalloc(&dv1, 4 * N));
  CK(cudaMemcpy(dsrc, hd.data(), 4 * N, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dv0, hid.data(), 4 * N, cudaMemcpyHostToDevice));

  // CUB
  size_t tb = 0;
  CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, dsrc, dk1, dv0, dv1, (int)N));
  tb = std::max(tb, vg::radix_temp_bytes(N, 32));
  void* tmp;
  CK(cudaMalloc(&tmp, tb));
  float t_cub = timeit([&] { cub::DeviceRadixSort::SortPairs(tmp, tb, dsrc, dk1, dv0, dv1, (int)N); }, 20);
  std::vector<uint32_t> out(N);
  CK(cudaMemcpy(out.data(), dv1, 4 * N, cudaMemcpyDeviceToHost));
  const bool ok_cub = out == ord;

  // hand-written onesweep (keys copied in each rep; copy time subtracted)
  int which = 0, nl = 0;
  float t_copy = timeit([&] { CK(cudaMemcpyAsync(dk0, dsrc, 4 * N, cudaMemcpyDeviceToDevice, 0)); }, 20);
  CK(cudaMemcpy(dv0, hid.data(), 4 * N, cudaMemcpyHostToDevice));
  float t_one = timeit([&] {
    CK(cudaMemcpyAsync(dk0, dsrc, 4 * N, cudaMemcpyDeviceToDevice, 0));
    vg::radix_sort_u32(tmp, tb, dk0, dk1, dv0, dv1, N, 32, &which, &nl, 0);
  }, 20) - t_copy;
  CK(cudaMemcpy(dv0, hid.data(), 4 * N, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dk0, dsrc, 4 * N, cudaMemcpyDeviceToDevice));
  vg::radix_sort_u32(tmp, tb, dk0, dk1, dv0, dv1, N, 32, &which, &nl, 0);
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(out.data(), which ? dv1 : dv0, 4 * N, cudaMemcpyDeviceToHost));
  const bool ok_one = out == ord;

  printf("depth sort N=%lld z in [%g, %g]: cub %.1f us (ok %d)  onesweep %.1f us (ok %d)\n",
         (long long)N, zlo, zhi, t_cub, ok_cub, t_one, ok_one);
  return ok_cub && ok_one ? 0 : 1;
}
