// Standalone A/B timing of the binning sorts: CUB onesweep (vg_sort.cu) vs the
// hand-written onesweep (vg_radix.cu) on synthetic inputs shaped like config 3
// (1M float depths; 8.2M pairs with 13-bit tile keys emitted in depth order).
//   nvcc ... tools/sortbench.cu build/csrc/vg_radix.o build/csrc/vg_sort.o -o build/sortbench
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>

#include "vg_kernels.cuh"

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

template <typename F>
static float timeit(F f, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  f();
  CK(cudaDeviceSynchronize());
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) f();
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms * 1000.f / reps;
}

int main(int argc, char** argv) {
  const int64_t N = argc > 1 ? atoll(argv[1]) : 1000000;
  const int64_t P = argc > 2 ? atoll(argv[2]) : 8200000;
  const int tile_bits = 13;
  std::mt19937 rng(1);
  // depths: positive floats in [1, 12]
  std::vector<uint32_t> hd(N), hid(N);
  std::uniform_real_distribution<float> U(1.f, 12.f);
  for (int64_t i = 0; i < N; ++i) { float z = U(rng); memcpy(&hd[i], &z, 4); hid[i] = (uint32_t)i; }
  // tile keys: clustered (each "Gaussian" emits a run of nearby tiles)
  std::vector<uint16_t> hk(P);
  std::vector<uint32_t> hv(P);
  std::uniform_int_distribution<int> T(0, 8159), L(1, 16);
  for (int64_t i = 0; i < P;) {
    int t = T(rng), l = L(rng);
    for (int j = 0; j < l && i < P; ++j, ++i) { hk[i] = (uint16_t)std::min(8159, t + j); hv[i] = (uint32_t)(i / 8); }
  }
  uint32_t *dk0, *dk1, *dv0, *dv1; uint16_t *tk0, *tk1; uint32_t *tv0, *tv1;
  CK(cudaMalloc(&dk0, 4 * N)); CK(cudaMalloc(&dk1, 4 * N)); CK(cudaMalloc(&dv0, 4 * N)); CK(cudaMalloc(&dv1, 4 * N));
  CK(cudaMalloc(&tk0, 2 * P)); CK(cudaMalloc(&tk1, 2 * P)); CK(cudaMalloc(&tv0, 4 * P)); CK(cudaMalloc(&tv1, 4 * P));
  uint32_t* dsrc; uint16_t* tsrc; uint32_t* tvsrc;
  CK(cudaMalloc(&dsrc, 4 * N)); CK(cudaMalloc(&tsrc, 2 * P)); CK(cudaMalloc(&tvsrc, 4 * P));
  CK(cudaMemcpy(dsrc, hd.data(), 4 * N, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dv0, hid.data(), 4 * N, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(tsrc, hk.data(), 2 * P, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(tvsrc, hv.data(), 4 * P, cudaMemcpyHostToDevice));
  size_t tb1 = 0, tb2 = 0;
  CK(vg::depth_sort_temp_bytes(N, &tb1));
  CK(vg::tile_sort_temp_bytes(P, tile_bits, false, &tb2));
  size_t tb = std::max({tb1, tb2, vg::radix_temp_bytes(N, 32), vg::radix_temp_bytes(P, tile_bits)});
  void* tmp; CK(cudaMalloc(&tmp, tb));
  // --- depth sort
  float t_cub_d = timeit([&] {
    vg::depth_sort(tmp, tb, dsrc, dk1, dv0, dv1, N, 0);
  }, 20);
  std::vector<uint32_t> ref_ids(N), my_ids(N);
  CK(cudaMemcpy(ref_ids.data(), dv1, 4 * N, cudaMemcpyDeviceToHost));
  int which = 0, nl = 0;
  float t_my_d = timeit([&] {
    CK(cudaMemcpyAsync(dk0, dsrc, 4 * N, cudaMemcpyDeviceToDevice, 0));
    vg::radix_sort_u32(tmp, tb, dk0, dk1, dv0, dv1, N, 32, &which, &nl, 0);
  }, 20);
  float t_copy_d = timeit([&] { CK(cudaMemcpyAsync(dk0, dsrc, 4 * N, cudaMemcpyDeviceToDevice, 0)); }, 20);
  CK(cudaMemcpy(my_ids.data(), which ? dv1 : dv0, 4 * N, cudaMemcpyDeviceToHost));
  // dv0 may have been overwritten by the ping-pong: reset for next runs is not needed (values = ids permuted)
  bool ok_d = true;
  {
    // both must be the stable order of the keys: compare key sequences and stability
    std::vector<uint32_t> ord(N);
    for (int64_t i = 0; i < N; ++i) ord[i] = (uint32_t)i;
    std::stable_sort(ord.begin(), ord.end(), [&](uint32_t a, uint32_t b) { return hd[a] < hd[b]; });
    for (int64_t i = 0; i < N; ++i) if (ref_ids[i] != ord[i]) { ok_d = false; break; }
  }
  // my sort after 20 reps permuted dv0/dv1 contents repeatedly: check a fresh run
  CK(cudaMemcpy(dv0, hid.data(), 4 * N, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dk0, dsrc, 4 * N, cudaMemcpyDeviceToDevice));
  vg::radix_sort_u32(tmp, tb, dk0, dk1, dv0, dv1, N, 32, &which, &nl, 0);
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(my_ids.data(), which ? dv1 : dv0, 4 * N, cudaMemcpyDeviceToHost));
  bool ok_dm = my_ids == ref_ids;
  // --- tile sort
  auto reset_t = [&] {
    CK(cudaMemcpyAsync(tk0, tsrc, 2 * P, cudaMemcpyDeviceToDevice, 0));
    CK(cudaMemcpyAsync(tv0, tvsrc, 4 * P, cudaMemcpyDeviceToDevice, 0));
  };
  float t_copy_t = timeit(reset_t, 20);
  float t_cub_t = timeit([&] { reset_t(); vg::tile_sort(tmp, tb, tk0, tk1, tv0, tv1, P, tile_bits, false, &which, 0); }, 20);
  std::vector<uint32_t> ref_v(P), my_v(P);
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(ref_v.data(), which ? tv1 : tv0, 4 * P, cudaMemcpyDeviceToHost));
  float t_my_t = timeit([&] { reset_t(); vg::radix_sort_u16(tmp, tb, tk0, tk1, tv0, tv1, P, tile_bits, &which, &nl, 0); }, 20);
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(my_v.data(), which ? tv1 : tv0, 4 * P, cudaMemcpyDeviceToHost));
  bool ok_t = my_v == ref_v;
  printf("depth sort N=%lld: cub %.1f us  mine %.1f us (incl. key copy %.1f)  ok_ref=%d ok_mine=%d\n",
         (long long)N, t_cub_d, t_my_d - t_copy_d, t_copy_d, ok_d, ok_dm);
  printf("tile sort P=%lld: cub %.1f us  mine %.1f us  (reset copies %.1f subtracted)  ok=%d\n",
         (long long)P, t_cub_t - t_copy_t, t_my_t - t_copy_t, t_copy_t, ok_t);
  printf("hbm floor (2 passes x 12 B/pair): %.1f us\n", 2.0 * 12.0 * P / 6.5e6);
  return 0;
}
