// K3: hand-written stable LSD radix sort of (key, value) pairs, onesweep style
// (one kernel per 8-bit digit pass with decoupled look-back), for the two
// sorts of the binning pipeline (raster._build_grid's lexsort,
// raster.py:256): the 32-bit float-depth keys of the Gaussians and the
// 16/32-bit tile keys of the depth-ordered pairs.
//
//   1. k_hist: one read of the keys builds the 256-bin histogram of every
//      digit position (shared-memory counters, one global add per bin/block).
//   2. k_scan: exclusive scan of each histogram -> global bucket bases.
//   3. k_pass (per digit): a block takes the next tile of 256 x 16 items
//      (dynamic tile id, so look-back only waits on tiles that already
//      started), ranks its items stably with warp match_any + per-warp digit
//      counters, publishes its per-digit counts and looks back over the
//      preceding tiles for their prefix, reorders the tile through shared
//      memory by digit and writes each digit run contiguously.
// Stability follows from ranking in input order (warp-major, then round, then
// lane) and from combining tiles in tile order.
#include <cuda_runtime.h>

#include "vg_kernels.cuh"

namespace vg {
namespace radix {

constexpr int BITS = 8;
constexpr int BINS = 256;
constexpr int THREADS = 256;
constexpr int WARPS = THREADS / 32;
#ifndef VG_RADIX_ITEMS
#define VG_RADIX_ITEMS 16
#endif
constexpr int ITEMS = VG_RADIX_ITEMS;          // per thread
constexpr int TILE_ITEMS = THREADS * ITEMS;   // 4096
constexpr uint32_t FLAG_AGG = 1u << 30;
constexpr uint32_t FLAG_INC = 2u << 30;
constexpr uint32_t VALUE_MASK = (1u << 30) - 1;

inline size_t temp_bytes(int64_t n, int key_bits) {
  const int passes = (key_bits + BITS - 1) / BITS;
  const int64_t tiles = (n + TILE_ITEMS - 1) / TILE_ITEMS;
  return sizeof(uint32_t) * (2 * (size_t)passes * BINS + 8 +
                             (size_t)passes * (size_t)(tiles > 0 ? tiles : 1) * BINS);
}

template <typename K>
__global__ void __launch_bounds__(THREADS) k_hist(const K* __restrict__ keys, int64_t n, int passes,
                                                  uint32_t* __restrict__ hist) {
  // per-warp sub-histograms: shared atomics only collide within a warp, and a
  // digit shared by the whole warp (the near-constant top byte of float
  // depths) is added once by lane 0
  __shared__ uint32_t h[WARPS][4][BINS];
  for (int i = threadIdx.x; i < WARPS * 4 * BINS; i += THREADS) (&h[0][0][0])[i] = 0;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * THREADS;
  const int64_t n_round = (n + stride - 1) / stride * stride;  // whole warps iterate together
  for (int64_t i = (int64_t)blockIdx.x * THREADS + threadIdx.x; i < n_round; i += stride) {
    const bool valid = i < n;
    const uint32_t k = valid ? (uint32_t)keys[i] : 0u;
    const unsigned vm = __ballot_sync(0xffffffffu, valid);
    for (int p = 0; p < passes; ++p) {
      const uint32_t d = (k >> (BITS * p)) & (BINS - 1);
      const uint32_t d0 = __shfl_sync(0xffffffffu, d, 0);
      if (vm == 0xffffffffu && __all_sync(0xffffffffu, d == d0)) {
        if (lane == 0) h[warp][p][d0] += 32u;
      } else if (valid) {
        atomicAdd(&h[warp][p][d], 1u);
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < passes * BINS; i += THREADS) {
    uint32_t v = 0;
#pragma unroll
    for (int w = 0; w < WARPS; ++w) v += (&h[w][0][0])[i];
    if (v) atomicAdd(hist + i, v);
  }
}

// One block of 256 threads per pass: exclusive scan of the pass's histogram.
__global__ void k_scan(const uint32_t* __restrict__ hist, uint32_t* __restrict__ base) {
  __shared__ uint32_t s[BINS];
  const int p = blockIdx.x, d = threadIdx.x;
  const uint32_t v = hist[p * BINS + d];
  s[d] = v;
  __syncthreads();
  for (int off = 1; off < BINS; off <<= 1) {
    const uint32_t t = d >= off ? s[d - off] : 0u;
    __syncthreads();
    s[d] += t;
    __syncthreads();
  }
  base[p * BINS + d] = s[d] - v;
}

__device__ __forceinline__ uint32_t ld_volatile(const uint32_t* p) {
  return *reinterpret_cast<const volatile uint32_t*>(p);
}
__device__ __forceinline__ void st_volatile(uint32_t* p, uint32_t v) {
  *reinterpret_cast<volatile uint32_t*>(p) = v;
}

template <typename K>
__global__ void __launch_bounds__(THREADS, 3) k_pass(const K* __restrict__ kin, K* __restrict__ kout,
                                                     const uint32_t* __restrict__ vin,
                                                     uint32_t* __restrict__ vout, int64_t n, int shift,
                                                     const uint32_t* __restrict__ bucket_base,
                                                     uint32_t* __restrict__ status,
                                                     uint32_t* __restrict__ tile_counter, int nbits) {
  __shared__ uint32_t s_tile;
  __shared__ uint32_t wcnt[WARPS][BINS];  // per-warp digit counts -> exclusive offsets
  __shared__ uint32_t s_scan[BINS];       // tile-local exclusive offset per digit
  __shared__ uint32_t s_global[BINS];     // global output base of this tile per digit
  __shared__ uint32_t s_wsum[WARPS];
  __shared__ K s_keys[TILE_ITEMS];
  __shared__ uint32_t s_vals[TILE_ITEMS];
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1u);
  for (int i = threadIdx.x; i < WARPS * BINS; i += THREADS) (&wcnt[0][0])[i] = 0;
  __syncthreads();
  const uint32_t tile = s_tile;
  const int64_t tbase = (int64_t)tile * TILE_ITEMS;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  const int64_t wbase = tbase + warp * (32 * ITEMS) + lane;
  uint32_t dig[ITEMS];
  uint32_t rank[ITEMS];
  // warp-striped load: warp w owns items [w*32*ITEMS, (w+1)*32*ITEMS) of the tile
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int64_t idx = wbase + i * 32;
    dig[i] = idx < n ? (((uint32_t)kin[idx] >> shift) & (BINS - 1)) : 0xffffffffu;
  }
  // Stable ranks within the warp in (round, lane) order.  The lanes sharing
  // a digit are found with one ballot per digit bit (multisplit); the leader
  // of each group adds the group size to the warp's counter with a shared
  // atomic (atomics of one warp to one address apply in issue order, so
  // rounds need no barrier) and broadcasts the old value to its peers.
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const bool valid = dig[i] != 0xffffffffu;
    unsigned peers = __ballot_sync(0xffffffffu, valid);
    if (!valid) peers = ~peers;
#pragma unroll
    for (int b = 0; b < BITS; ++b) {
      if (b < nbits) {
        const bool bit = (dig[i] >> b) & 1u;
        const unsigned bal = __ballot_sync(0xffffffffu, bit);
        peers &= bit ? bal : ~bal;
      }
    }
    const int leader = __ffs(peers) - 1;
    uint32_t old = 0;
    if (valid && lane == leader) old = atomicAdd(&wcnt[warp][dig[i]], (uint32_t)__popc(peers));
    rank[i] = __popc(peers & lt) + __shfl_sync(0xffffffffu, old, leader);
  }
  __syncthreads();
  // per digit (thread d < 256): exclusive prefix over warps, publish, look back
  uint32_t run = 0;
  if (threadIdx.x < BINS) {
    const int d = threadIdx.x;
#pragma unroll
    for (int w = 0; w < WARPS; ++w) {
      const uint32_t c = wcnt[w][d];
      wcnt[w][d] = run;
      run += c;
    }
    uint32_t* st = status + (size_t)tile * BINS + d;
    uint32_t excl = 0;
    if (tile == 0) {
      st_volatile(st, FLAG_INC | run);
    } else {
      st_volatile(st, FLAG_AGG | run);
      // walk back over the predecessors, four status words per round trip
      int64_t t = (int64_t)tile - 1;
      bool found = false;
      while (!found) {
        uint32_t v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j)
          v[j] = t - j >= 0 ? ld_volatile(status + (size_t)(t - j) * BINS + d) : FLAG_INC;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (found) break;
          if ((v[j] & ~VALUE_MASK) == 0u) break;  // not published yet: re-poll from here
          excl += v[j] & VALUE_MASK;
          --t;
          if (v[j] & FLAG_INC) found = true;
        }
      }
      st_volatile(st, FLAG_INC | (excl + run));
    }
    s_global[d] = bucket_base[d] + excl;
  }
  // tile-local exclusive offsets per digit: warp scans + one pass over warp sums
  {
    uint32_t x = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) s_wsum[warp] = x;
    __syncthreads();
    uint32_t add = 0;
#pragma unroll
    for (int w = 0; w < BINS / 32; ++w) add += (w < warp) ? s_wsum[w] : 0u;
    if (threadIdx.x < BINS) s_scan[threadIdx.x] = add + x - run;
  }
  __syncthreads();
  // reorder the tile through shared memory by digit (stable): keys from the
  // digits' source registers, values straight from global
  const int tile_n = (int)min((int64_t)TILE_ITEMS, n - tbase);
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    if (dig[i] != 0xffffffffu) rank[i] += s_scan[dig[i]] + wcnt[warp][dig[i]];
  }
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int64_t idx = wbase + i * 32;
    if (idx < n) {
      s_keys[rank[i]] = kin[idx];
      s_vals[rank[i]] = vin ? vin[idx] : (uint32_t)idx;  // NULL: identity values
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < tile_n; i += THREADS) {
    const K k = s_keys[i];
    const uint32_t d = ((uint32_t)k >> shift) & (BINS - 1);
    const uint32_t out = s_global[d] + (uint32_t)i - s_scan[d];
    kout[out] = k;
    vout[out] = s_vals[i];
  }
}

template <typename K>
cudaError_t sort_pairs(void* tmp, size_t tmp_bytes, K* k0, K* k1, uint32_t* v0, uint32_t* v1,
                       int64_t n, int key_bits, int* which, int* launches, cudaStream_t st,
                       bool identity = false) {
  *which = 0;
  if (n <= 1) {  // nothing to sort; the identity of one item is 0
    return (identity && n == 1) ? cudaMemsetAsync(v0, 0, sizeof(uint32_t), st) : cudaSuccess;
  }
  const int passes = (key_bits + BITS - 1) / BITS;
  const int64_t tiles = (n + TILE_ITEMS - 1) / TILE_ITEMS;
  if (tmp_bytes < temp_bytes(n, key_bits)) return cudaErrorInvalidValue;
  uint32_t* hist = (uint32_t*)tmp;
  uint32_t* base = hist + passes * BINS;
  uint32_t* counters = base + passes * BINS;
  uint32_t* status = counters + 8;
  // histograms, tile counters and every pass's look-back status in one memset
  cudaError_t e = cudaMemsetAsync(
      tmp, 0, sizeof(uint32_t) * (2 * (size_t)passes * BINS + 8 + (size_t)passes * tiles * BINS), st);
  if (e != cudaSuccess) return e;
  int hist_blocks = (int)((n + THREADS * 8 - 1) / (THREADS * 8));
  if (hist_blocks > 1184) hist_blocks = 1184;
  k_hist<K><<<hist_blocks, THREADS, 0, st>>>(k0, n, passes, hist);
  k_scan<<<passes, BINS, 0, st>>>(hist, base);
  *launches += 2;
  K* kin = k0;
  K* kout = k1;
  uint32_t* vin = v0;
  uint32_t* vout = v1;
  for (int p = 0; p < passes; ++p) {
    k_pass<K><<<(unsigned)tiles, THREADS, 0, st>>>(kin, kout, (p == 0 && identity) ? nullptr : vin,
                                                   vout, n, BITS * p,
                                                   base + p * BINS,
                                                   status + (size_t)p * tiles * BINS, counters + p,
                                                   min(BITS, key_bits - BITS * p));
    *launches += 1;
    K* tk = kin; kin = kout; kout = tk;
    uint32_t* tv = vin; vin = vout; vout = tv;
  }
  *which = passes & 1;
  return cudaGetLastError();
}

}  // namespace radix

size_t radix_temp_bytes(int64_t n, int key_bits) { return radix::temp_bytes(n, key_bits); }

cudaError_t radix_sort_u32(void* tmp, size_t tmp_bytes, uint32_t* k0, uint32_t* k1, uint32_t* v0,
                           uint32_t* v1, int64_t n, int key_bits, int* which, int* launches,
                           cudaStream_t st, bool identity_values) {
  return radix::sort_pairs<uint32_t>(tmp, tmp_bytes, k0, k1, v0, v1, n, key_bits, which, launches,
                                     st, identity_values);
}

cudaError_t radix_sort_u16(void* tmp, size_t tmp_bytes, uint16_t* k0, uint16_t* k1, uint32_t* v0,
                           uint32_t* v1, int64_t n, int key_bits, int* which, int* launches,
                           cudaStream_t st) {
  return radix::sort_pairs<uint16_t>(tmp, tmp_bytes, k0, k1, v0, v1, n, key_bits, which, launches,
                                     st);
}

}  // namespace vg
