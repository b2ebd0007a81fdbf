// K2 + K3 + K4: span binning (raster._build_grid, raster.py:222-260).
//
// The reference duplicates every (Gaussian, tile) pair and lexsorts them by
// (tile, depth, index).  Here the Gaussians are already in (float32 depth,
// index) order (the depth sort of vg_capi.cu), and every Gaussian covers a
// rectangle of tiles, so the per-tile lists are built by two *stable
// expansions* instead of a sort of the pairs:
//
//   step 1  Gaussians (depth order) -> row spans: each Gaussian emits one
//           span (g, x0..x1) into every tile row y0..y1 it covers; the spans
//           of a row keep depth order.
//   step 2  spans of a row (depth order) -> tile entries: each span emits g
//           into the lists of tiles (y, x0..x1); each list keeps depth order.
//
// Both steps are the same primitive.  The items are cut into chunks of 1024
// (one CTA each); item i of a chunk covers the bucket interval [lo_i, hi_i]
// (rows in step 1, tile columns in step 2).  A chunk's stable rank of item i
// in bucket b is the number of earlier items of the chunk covering b, read
// from per-bucket coverage bitmaps (one ballot per bucket and warp) and their
// per-word prefix popcounts; the chunk's base in bucket b is the exclusive
// prefix of the per-chunk bucket counts over the preceding chunks (a count
// kernel and a scan kernel).  No sort, no atomics on the output positions:
// the lists are bit-identical to a stable sort by tile of the depth-ordered
// pairs, i.e. to lexsort((prim, float32(depth), tile)).
//
// Step 2's chunks never straddle rows: every row's span list is padded to a
// multiple of 1024 (the padding is never read: item validity comes from the
// row's span count).  The host reads back the pair total and the number of
// step-2 chunks once, to size the outputs (the pipeline's one host sync).
#include <climits>

#include "vg_kernels.cuh"

namespace vg {
namespace span {

constexpr unsigned FULLM = 0xffffffffu;
constexpr int CH = 1024;         // items per chunk
constexpr int CT = 256;          // threads per chunk CTA
constexpr int WPC = CH / 32;     // bitmap words per bucket
constexpr int BMS = WPC + 1;     // padded bitmap row stride (conflict-free prefix pass)
constexpr int SCAN_T = 1024;     // threads of the single-CTA kernels

// dynamic shared memory of a chunk CTA with B buckets
inline size_t chunk_smem(int B) {
  return sizeof(int) * 2 * CH + sizeof(uint32_t) * CH * 2 + sizeof(uint32_t) * (size_t)B * BMS +
         sizeof(uint16_t) * (size_t)B * BMS + sizeof(uint32_t) * (size_t)B + 64;
}

struct ChunkSm {
  int* lo;
  int* hi;
  uint32_t* g;      // item payload: Gaussian id
  uint32_t* x;      // item payload: x0 | x1 << 16 (step 1)
  uint32_t* bm;     // [B][BMS] coverage bits
  uint16_t* pre;    // [B][BMS] exclusive popcount prefix per word
  uint32_t* base;   // [B] output base of this chunk per bucket
};

__device__ __forceinline__ ChunkSm carve(int B) {
  extern __shared__ __align__(16) unsigned char smraw[];
  ChunkSm s;
  s.lo = reinterpret_cast<int*>(smraw);
  s.hi = s.lo + CH;
  s.g = reinterpret_cast<uint32_t*>(s.hi + CH);
  s.x = s.g + CH;
  s.bm = s.x + CH;
  s.base = s.bm + (size_t)B * BMS;
  s.pre = reinterpret_cast<uint16_t*>(s.base + B);
  return s;
}

// Coverage bitmaps and per-word exclusive prefix popcounts of one chunk.
__device__ __forceinline__ void rank_tables(int B, const ChunkSm& s) {
  for (int i = threadIdx.x; i < B * BMS; i += CT) s.bm[i] = 0u;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int w = warp; w < WPC; w += CT / 32) {
    const int i = w * 32 + lane;
    const int l = s.lo[i], h = s.hi[i];
    const int wl = __reduce_min_sync(FULLM, l), wh = __reduce_max_sync(FULLM, h);
    for (int b = wl; b <= wh; ++b) {
      const unsigned m = __ballot_sync(FULLM, l <= b && b <= h);
      if (lane == 0) s.bm[b * BMS + w] = m;
    }
  }
  __syncthreads();
  for (int b = threadIdx.x; b < B; b += CT) {
    uint32_t run = 0;
    for (int w = 0; w < WPC; ++w) {
      s.pre[b * BMS + w] = (uint16_t)run;
      run += __popc(s.bm[b * BMS + w]);
    }
  }
  __syncthreads();
}

__device__ __forceinline__ uint32_t rank_of(const ChunkSm& s, int i, int b) {
  const int w = i >> 5;
  return s.pre[b * BMS + w] + __popc(s.bm[b * BMS + w] & ((1u << (i & 31)) - 1u));
}

// Per-chunk bucket counts (shared atomics), written as C[b][chunk].
__device__ __forceinline__ void count_out(int B, const ChunkSm& s, uint32_t* C, int nchunks,
                                          int chunk) {
  uint32_t* cnt = s.base;
  for (int b = threadIdx.x; b < B; b += CT) cnt[b] = 0u;
  __syncthreads();
  for (int i = threadIdx.x; i < CH; i += CT)
    for (int b = s.lo[i]; b <= s.hi[i]; ++b) atomicAdd(&cnt[b], 1u);
  __syncthreads();
  for (int b = threadIdx.x; b < B; b += CT) C[(size_t)b * nchunks + chunk] = cnt[b];
}

// ---------------------------------------------------------------------------
// step 1: Gaussians in depth order -> row spans

__device__ __forceinline__ void load_gaussians(int64_t n, const uint32_t* __restrict__ perm,
                                               const uint32_t* __restrict__ count,
                                               const int4* __restrict__ rect, const ChunkSm& s,
                                               uint32_t* pairs) {
  const int64_t base = (int64_t)blockIdx.x * CH;
  uint32_t mine = 0;
  for (int i = threadIdx.x; i < CH; i += CT) {
    const int64_t k = base + i;
    int l = INT_MAX, h = -1;
    uint32_t g = 0, xr = 0;
    if (k < n) {
      g = perm[k];
      const uint32_t c = count[g];
      if (c) {
        const int4 r = rect[g];
        l = r.y;
        h = r.w;
        xr = (uint32_t)r.x | ((uint32_t)r.z << 16);
        mine += c;
      }
    }
    s.lo[i] = l;
    s.hi[i] = h;
    s.g[i] = g;
    s.x[i] = xr;
  }
  if (pairs) *pairs = mine;
}

__global__ void __launch_bounds__(CT) k_rows_count(int64_t n, const uint32_t* __restrict__ perm,
                                                   const uint32_t* __restrict__ count,
                                                   const int4* __restrict__ rect, int nty,
                                                   int nchunks, uint32_t* __restrict__ C1,
                                                   unsigned long long* __restrict__ pairs_total) {
  const ChunkSm s = carve(nty);
  uint32_t mine;
  load_gaussians(n, perm, count, rect, s, &mine);
  for (int o = 16; o; o >>= 1) mine += __shfl_xor_sync(FULLM, mine, o);
  if ((threadIdx.x & 31) == 0 && mine) atomicAdd(pairs_total, (unsigned long long)mine);
  __syncthreads();
  count_out(nty, s, C1, nchunks, blockIdx.x);
}

__global__ void __launch_bounds__(CT) k_rows_place(int64_t n, const uint32_t* __restrict__ perm,
                                                   const uint32_t* __restrict__ count,
                                                   const int4* __restrict__ rect, int nty,
                                                   int nchunks, const uint32_t* __restrict__ R1,
                                                   const uint32_t* __restrict__ row_chunk0,
                                                   uint2* __restrict__ spans) {
  const ChunkSm s = carve(nty);
  load_gaussians(n, perm, count, rect, s, nullptr);
  for (int y = threadIdx.x; y < nty; y += CT)
    s.base[y] = row_chunk0[y] * (uint32_t)CH + R1[(size_t)y * nchunks + blockIdx.x];
  __syncthreads();
  rank_tables(nty, s);
  for (int i = threadIdx.x; i < CH; i += CT) {
    const int l = s.lo[i], h = s.hi[i];
    const uint2 v = make_uint2(s.g[i], s.x[i]);
    for (int y = l; y <= h; ++y) spans[s.base[y] + rank_of(s, i, y)] = v;
  }
}

// ---------------------------------------------------------------------------
// single-CTA / per-bucket scans

// Block-wide exclusive scan of 1024 values (one per thread); returns the total.
__device__ __forceinline__ uint32_t block_scan1024(uint32_t v, uint32_t& excl) {
  __shared__ uint32_t ws[SCAN_T / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(FULLM, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) ws[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint32_t t = ws[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(FULLM, t, o);
      if (lane >= o) t += y;
    }
    ws[lane] = t;
  }
  __syncthreads();
  const uint32_t before = warp ? ws[warp - 1] : 0u;
  const uint32_t total = ws[SCAN_T / 32 - 1];
  excl = before + x - v;
  __syncthreads();
  return total;
}

// Per bucket (one CTA each): exclusive prefix of its counts over the chunks,
// in place (C[b][*] becomes the chunk's base within the bucket); total -> tot[b].
__global__ void __launch_bounds__(SCAN_T) k_bucket_scan(uint32_t* __restrict__ C, int nchunks,
                                                        uint32_t* __restrict__ tot) {
  uint32_t* row = C + (size_t)blockIdx.x * nchunks;
  uint32_t carry = 0;
  for (int c0 = 0; c0 < nchunks; c0 += SCAN_T) {
    const int c = c0 + threadIdx.x;
    const uint32_t v = c < nchunks ? row[c] : 0u;
    uint32_t ex;
    const uint32_t t = block_scan1024(v, ex);
    if (c < nchunks) row[c] = carry + ex;
    carry += t;
  }
  if (threadIdx.x == 0) tot[blockIdx.x] = carry;
}

// Rows -> step-2 chunk layout: row y's spans start at chunk row_chunk0[y]
// (each row padded to whole chunks); info = {pairs (u64, untouched), chunks}.
__global__ void __launch_bounds__(SCAN_T) k_rows_layout(const uint32_t* __restrict__ S, int nty,
                                                        uint32_t* __restrict__ row_chunk0,
                                                        unsigned long long* __restrict__ info) {
  uint32_t carry = 0;
  for (int y0 = 0; y0 < nty; y0 += SCAN_T) {
    const int y = y0 + threadIdx.x;
    const uint32_t k = y < nty ? (S[y] + CH - 1) / CH : 0u;
    uint32_t ex;
    const uint32_t t = block_scan1024(k, ex);
    if (y < nty) row_chunk0[y] = carry + ex;
    carry += t;
  }
  if (threadIdx.x == 0) {
    row_chunk0[nty] = carry;
    info[1] = carry;
  }
}

// ---------------------------------------------------------------------------
// step 2: row spans -> tile entries

__device__ __forceinline__ int chunk_row(const uint32_t* __restrict__ row_chunk0, int nty,
                                         uint32_t c) {
  // last y with row_chunk0[y] <= c (rows without spans have equal starts)
  int lo = 0, hi = nty - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (row_chunk0[mid] <= c) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ int load_spans(const uint2* __restrict__ spans,
                                          const uint32_t* __restrict__ S,
                                          const uint32_t* __restrict__ row_chunk0, int nty,
                                          const ChunkSm& s) {
  __shared__ int s_y;
  const uint32_t c = blockIdx.x;
  if (threadIdx.x == 0) s_y = chunk_row(row_chunk0, nty, c);
  __syncthreads();
  const int y = s_y;
  const uint32_t first = (c - row_chunk0[y]) * (uint32_t)CH;
  const int nvalid = (int)min((uint32_t)CH, S[y] - first);
  for (int i = threadIdx.x; i < CH; i += CT) {
    int l = INT_MAX, h = -1;
    uint32_t g = 0;
    if (i < nvalid) {
      const uint2 v = spans[(size_t)c * CH + i];
      g = v.x;
      l = (int)(v.y & 0xffffu);
      h = (int)(v.y >> 16);
    }
    s.lo[i] = l;
    s.hi[i] = h;
    s.g[i] = g;
  }
  return y;
}

__global__ void __launch_bounds__(CT) k_cols_count(const uint2* __restrict__ spans,
                                                   const uint32_t* __restrict__ S,
                                                   const uint32_t* __restrict__ row_chunk0,
                                                   int nty, int ntx, int nchunks,
                                                   uint32_t* __restrict__ C2) {
  const ChunkSm s = carve(ntx);
  load_spans(spans, S, row_chunk0, nty, s);
  __syncthreads();
  count_out(ntx, s, C2, nchunks, blockIdx.x);
}

// Per tile (one thread): exclusive prefix of its column's counts over the
// chunks of its row (in place), tile total -> T.
__global__ void k_tile_scan(uint32_t* __restrict__ C2, int nchunks,
                            const uint32_t* __restrict__ row_chunk0, int ntx, int n_tiles,
                            uint32_t* __restrict__ T) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_tiles) return;
  const int y = t / ntx, x = t - y * ntx;
  uint32_t* col = C2 + (size_t)x * nchunks;
  uint32_t run = 0;
  for (uint32_t c = row_chunk0[y]; c < row_chunk0[y + 1]; ++c) {
    const uint32_t v = col[c];
    col[c] = run;
    run += v;
  }
  T[t] = run;
}

// Single CTA: tile ranges from the tile totals, and the heavy-tiles-first
// launch order (counting sort by descending, bucketed list length).
constexpr int ORD_BINS = 1024;
__device__ __forceinline__ int len_bin(uint32_t len) {
  // exact below 512, then 32-wide buckets; bin 0 = longest
  const uint32_t q = len < 512u ? len : min(1023u, 512u + ((len - 512u) >> 5));
  return 1023 - (int)q;
}

__global__ void __launch_bounds__(SCAN_T) k_tile_ranges_order(const uint32_t* __restrict__ T,
                                                              int n_tiles, uint2* __restrict__ ranges,
                                                              uint32_t* __restrict__ order) {
  __shared__ uint32_t hist[ORD_BINS];
  for (int b = threadIdx.x; b < ORD_BINS; b += SCAN_T) hist[b] = 0u;
  uint32_t carry = 0;
  for (int t0 = 0; t0 < n_tiles; t0 += SCAN_T) {
    const int t = t0 + threadIdx.x;
    const uint32_t v = t < n_tiles ? T[t] : 0u;
    uint32_t ex;
    const uint32_t tot = block_scan1024(v, ex);
    if (t < n_tiles) {
      ranges[t] = make_uint2(carry + ex, carry + ex + v);
      atomicAdd(&hist[len_bin(v)], 1u);
    }
    carry += tot;
  }
  __syncthreads();
  {
    const uint32_t v = hist[threadIdx.x];
    uint32_t ex;
    block_scan1024(v, ex);
    hist[threadIdx.x] = ex;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < n_tiles; t += SCAN_T)
    order[atomicAdd(&hist[len_bin(T[t])], 1u)] = (uint32_t)t;
}

__global__ void __launch_bounds__(CT) k_cols_place(const uint2* __restrict__ spans,
                                                   const uint32_t* __restrict__ S,
                                                   const uint32_t* __restrict__ row_chunk0,
                                                   int nty, int ntx, int nchunks,
                                                   const uint32_t* __restrict__ R2,
                                                   const uint2* __restrict__ ranges,
                                                   uint32_t* __restrict__ vals) {
  const ChunkSm s = carve(ntx);
  const int y = load_spans(spans, S, row_chunk0, nty, s);
  for (int x = threadIdx.x; x < ntx; x += CT)
    s.base[x] = ranges[y * ntx + x].x + R2[(size_t)x * nchunks + blockIdx.x];
  __syncthreads();
  rank_tables(ntx, s);
  for (int i = threadIdx.x; i < CH; i += CT) {
    const int l = s.lo[i], h = s.hi[i];
    const uint32_t g = s.g[i];
    for (int x = l; x <= h; ++x) vals[s.base[x] + rank_of(s, i, x)] = g;
  }
}

}  // namespace span

// ---------------------------------------------------------------------------
// launchers (see vg_kernels.cuh)

int span_max_buckets() { return 1024; }

int64_t span_chunks1(int64_t n) { return (n + span::CH - 1) / span::CH; }

size_t span_scratch1_bytes(int64_t n, int nty) {
  // C1 [nty][chunks1] + S [nty] + row_chunk0 [nty + 1]
  return sizeof(uint32_t) * ((size_t)nty * (size_t)span_chunks1(n) + 2 * (size_t)nty + 1);
}

cudaError_t span_rows_begin(int64_t n, const uint32_t* perm, const uint32_t* count,
                            const int4* rect, int nty, void* scratch1,
                            unsigned long long* info, cudaStream_t st) {
  using namespace span;
  const int nch = (int)span_chunks1(n);
  uint32_t* C1 = (uint32_t*)scratch1;
  uint32_t* S = C1 + (size_t)nty * nch;
  uint32_t* rc0 = S + nty;
  cudaError_t e = cudaMemsetAsync(info, 0, 2 * sizeof(unsigned long long), st);
  if (e != cudaSuccess) return e;
  if (nch > 0) {
    const size_t sm = chunk_smem(nty);
    k_rows_count<<<nch, CT, sm, st>>>(n, perm, count, rect, nty, nch, C1, info);
    k_bucket_scan<<<nty, SCAN_T, 0, st>>>(C1, nch, S);
  } else {
    e = cudaMemsetAsync(S, 0, sizeof(uint32_t) * nty, st);
    if (e != cudaSuccess) return e;
  }
  k_rows_layout<<<1, SCAN_T, 0, st>>>(S, nty, rc0, info);
  return cudaGetLastError();
}

size_t span_scratch2_bytes(int64_t chunks2, int ntx, int n_tiles) {
  // spans [chunks2 * CH] (uint2) + C2 [ntx][chunks2] + T [n_tiles]
  return sizeof(uint2) * (size_t)chunks2 * span::CH +
         sizeof(uint32_t) * ((size_t)ntx * (size_t)chunks2 + (size_t)n_tiles);
}

cudaError_t span_finish(int64_t n, const uint32_t* perm, const uint32_t* count, const int4* rect,
                        int ntx, int nty, const void* scratch1, int64_t chunks2, void* scratch2,
                        uint2* ranges, uint32_t* order, uint32_t* vals, int* launches,
                        cudaStream_t st) {
  using namespace span;
  const int nch1 = (int)span_chunks1(n);
  const int n_tiles = ntx * nty;
  const uint32_t* R1 = (const uint32_t*)scratch1;
  const uint32_t* S = R1 + (size_t)nty * nch1;
  const uint32_t* rc0 = S + nty;
  uint2* spans = (uint2*)scratch2;
  uint32_t* C2 = (uint32_t*)(spans + (size_t)chunks2 * CH);
  uint32_t* T = C2 + (size_t)ntx * chunks2;
  if (chunks2 > 0) {
    k_rows_place<<<nch1, CT, chunk_smem(nty), st>>>(n, perm, count, rect, nty, nch1, R1, rc0,
                                                     spans);
    const size_t sm2 = chunk_smem(ntx);
    k_cols_count<<<(unsigned)chunks2, CT, sm2, st>>>(spans, S, rc0, nty, ntx, (int)chunks2, C2);
    k_tile_scan<<<(n_tiles + 255) / 256, 256, 0, st>>>(C2, (int)chunks2, rc0, ntx, n_tiles, T);
    *launches += 3;
  } else {
    cudaError_t e = cudaMemsetAsync(T, 0, sizeof(uint32_t) * n_tiles, st);
    if (e != cudaSuccess) return e;
  }
  k_tile_ranges_order<<<1, SCAN_T, 0, st>>>(T, n_tiles, ranges, order);
  *launches += 1;
  if (chunks2 > 0) {
    k_cols_place<<<(unsigned)chunks2, CT, chunk_smem(ntx), st>>>(spans, S, rc0, nty, ntx,
                                                                  (int)chunks2, C2, ranges, vals);
    *launches += 1;
  }
  return cudaGetLastError();
}

cudaError_t span_configure() {
  using namespace span;
  const size_t mx = chunk_smem(1024);
  cudaError_t e = cudaFuncSetAttribute(k_rows_count, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mx);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_rows_place, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mx);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_cols_count, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mx);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(k_cols_place, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mx);
  return e;
}

}  // namespace vg
