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
// Both steps are the same primitive.  The items are cut into chunks of CH (512)
// (one CTA each); item i of a chunk covers the bucket interval [lo_i, hi_i]
// (rows in step 1, tile columns in step 2).  A chunk's stable rank of item i
// in bucket b is the number of earlier items of the chunk covering b, read
// from per-bucket coverage bitmaps (one shared atomicOr per pair) and their
// per-word prefix popcounts; the chunk's base in bucket b is the exclusive
// prefix of the per-chunk bucket counts over the preceding chunks (a count
// kernel and a scan kernel).  No sort, no atomics on the output positions:
// the lists are bit-identical to a stable sort by tile of the depth-ordered
// pairs, i.e. to lexsort((prim, float32(depth), tile)).
//
// Step 2's chunks never straddle rows: every row's span list is padded to a
// multiple of CH (the padding is never read: item validity comes from the
// row's span count).  The host reads back the pair total and the number of
// step-2 chunks once, to size the outputs (the pipeline's one host sync).
#include <climits>

#include "vg_kernels.cuh"

namespace vg {
namespace span {

constexpr unsigned FULLM = 0xffffffffu;
#ifndef VG_SPAN_CH
#define VG_SPAN_CH 512  // A/B (16 views of config 3, serial, scan + place): 256: 2.42, 512: 2.21, 768: 2.22, 1024: 2.32 ms
#endif
constexpr int CH = VG_SPAN_CH;   // items per chunk
#ifndef VG_SPAN_CT
#define VG_SPAN_CT 256
#endif
constexpr int CT = VG_SPAN_CT;   // threads per chunk CTA
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

// Coverage bitmaps and per-word exclusive prefix popcounts of one chunk:
// every (item, bucket) pair sets its bit with one shared atomicOr.
__device__ __forceinline__ void rank_tables(int B, const ChunkSm& s) {
  for (int i = threadIdx.x; i < B * BMS; i += CT) s.bm[i] = 0u;
  __syncthreads();
#pragma unroll
  for (int k = 0; k < CH / CT; ++k) {
    const int i = k * CT + threadIdx.x;
    const int l = s.lo[i], h = s.hi[i];
    const uint32_t bit = 1u << (i & 31);
    uint32_t* col = s.bm + (i >> 5);
    for (int b = l; b <= h; ++b) atomicOr(col + b * BMS, bit);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < B; b += CT) {
    uint32_t run = 0;
#pragma unroll 8
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
                                               const ushort4* __restrict__ rect, const ChunkSm& s,
                                               uint32_t* pairs) {
  const int64_t base = (int64_t)blockIdx.x * CH;
  uint32_t mine = 0;
#pragma unroll
  for (int j = 0; j < CH / CT; ++j) {
    const int i = j * CT + threadIdx.x;
    const int64_t k = base + i;
    int l = INT_MAX, h = -1;
    uint32_t g = 0, xr = 0;
    if (k < n) {
      g = perm[k];
      const ushort4 r = rect[g];  // x0, y0, x1, y1; empty when x1 < x0
      if (r.z >= r.x) {
        l = r.y;
        h = r.w;
        xr = (uint32_t)r.x | ((uint32_t)r.z << 16);
        mine += (uint32_t)(r.z - r.x + 1) * (uint32_t)(r.w - r.y + 1);
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
                                                   const ushort4* __restrict__ rect, int nty,
                                                   int nchunks, uint32_t* __restrict__ C1,
                                                   uint32_t* __restrict__ pairs_part) {
  __shared__ uint32_t wsum[CT / 32];
  const ChunkSm s = carve(nty);
  uint32_t mine;
  load_gaussians(n, perm, rect, s, &mine);
  for (int o = 16; o; o >>= 1) mine += __shfl_xor_sync(FULLM, mine, o);
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = mine;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int w = 0; w < CT / 32; ++w) t += wsum[w];
    pairs_part[blockIdx.x] = t;  // summed by the layout step (no same-address atomics)
  }
  count_out(nty, s, C1, nchunks, blockIdx.x);
}

__global__ void __launch_bounds__(CT) k_rows_place(int64_t n, const uint32_t* __restrict__ perm,
                                                   const ushort4* __restrict__ rect, int nty,
                                                   int nchunks, const uint32_t* __restrict__ R1,
                                                   const uint32_t* __restrict__ row_chunk0,
                                                   uint2* __restrict__ spans) {
  const ChunkSm s = carve(nty);
  load_gaussians(n, perm, rect, s, nullptr);
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

// Rows -> step-2 chunk layout: row y's spans start at chunk row_chunk0[y]
// (each row padded to whole chunks); info = {pairs, step-2 chunks}.
__device__ __forceinline__ void rows_layout(const uint32_t* __restrict__ S, int nty,
                                            const uint32_t* __restrict__ pairs_part, int nparts,
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
  unsigned long long p = 0;
  for (int i = threadIdx.x; i < nparts; i += SCAN_T) p += pairs_part[i];
  for (int o = 16; o; o >>= 1) p += __shfl_xor_sync(FULLM, p, o);
  __shared__ unsigned long long ps[SCAN_T / 32];
  if ((threadIdx.x & 31) == 0) ps[threadIdx.x >> 5] = p;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long tot = 0;
    for (int w = 0; w < SCAN_T / 32; ++w) tot += ps[w];
    row_chunk0[nty] = carry;
    info[0] = tot;
    info[1] = carry;
  }
}

// Per bucket (one CTA each): exclusive prefix of its counts over the chunks,
// in place (C[b][*] becomes the chunk's base within the bucket); total ->
// tot[b].  The last CTA to finish lays out the step-2 chunks.
__global__ void __launch_bounds__(SCAN_T) k_bucket_scan(uint32_t* __restrict__ C, int nchunks,
                                                        uint32_t* __restrict__ tot, int nty,
                                                        const uint32_t* __restrict__ pairs_part,
                                                        uint32_t* __restrict__ row_chunk0,
                                                        unsigned long long* __restrict__ info,
                                                        uint32_t* __restrict__ done) {
  __shared__ bool last;
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
  if (threadIdx.x == 0) {
    tot[blockIdx.x] = carry;
    __threadfence();
    last = atomicAdd(done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  rows_layout(tot, nty, pairs_part, nchunks, row_chunk0, info);
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
#pragma unroll
  for (int j = 0; j < CH / CT; ++j) {
    const int i = j * CT + threadIdx.x;
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

// Tile ranges from the tile totals, and the heavy-tiles-first launch order
// (counting sort by descending, bucketed list length).  One 1024-thread CTA.
constexpr int ORD_BINS = 1024;
constexpr int RPT = 8;  // tiles per thread per round
__device__ __forceinline__ int len_bin(uint32_t len) {
  // exact below 512, then 32-wide buckets; bin 0 = longest
  const uint32_t q = len < 512u ? len : min(1023u, 512u + ((len - 512u) >> 5));
  return 1023 - (int)q;
}

__device__ __forceinline__ void tile_ranges_order(const uint32_t* __restrict__ T, int n_tiles,
                                                  uint2* __restrict__ ranges,
                                                  uint32_t* __restrict__ order) {
  __shared__ uint32_t hist[ORD_BINS];
  for (int b = threadIdx.x; b < ORD_BINS; b += SCAN_T) hist[b] = 0u;
  uint32_t carry = 0;
  for (int t0 = 0; t0 < n_tiles; t0 += SCAN_T * RPT) {
    uint32_t v[RPT];
    uint32_t sum = 0;
    const int tb = t0 + threadIdx.x * RPT;
#pragma unroll
    for (int j = 0; j < RPT; ++j) {
      v[j] = tb + j < n_tiles ? __ldcg(T + tb + j) : 0u;
      sum += v[j];
    }
    uint32_t ex;
    const uint32_t tot = block_scan1024(sum, ex);
    uint32_t run = carry + ex;
#pragma unroll
    for (int j = 0; j < RPT; ++j) {
      const bool in = tb + j < n_tiles;
      if (in) ranges[tb + j] = make_uint2(run, run + v[j]);
      run += v[j];
      // warp-aggregated histogram (many tiles share a length bin)
      const int bin = in ? len_bin(v[j]) : -1;
      const unsigned peers = __match_any_sync(FULLM, bin);
      if (in && (threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&hist[bin], (uint32_t)__popc(peers));
    }
    carry += tot;
  }
  __syncthreads();
  {
    const uint32_t h = hist[threadIdx.x];
    uint32_t ex;
    block_scan1024(h, ex);
    hist[threadIdx.x] = ex;
  }
  __syncthreads();
  const unsigned lt = (1u << (threadIdx.x & 31)) - 1u;
  for (int t0 = 0; t0 < n_tiles; t0 += SCAN_T) {
    const int t = t0 + threadIdx.x;
    const bool in = t < n_tiles;
    const int bin = in ? len_bin(__ldcg(T + t)) : -1;
    const unsigned peers = __match_any_sync(FULLM, bin);
    const int leader = __ffs(peers) - 1;
    uint32_t old = 0;
    if (in && (threadIdx.x & 31) == leader) old = atomicAdd(&hist[bin], (uint32_t)__popc(peers));
    old = __shfl_sync(FULLM, old, leader);
    if (in) order[old + __popc(peers & lt)] = (uint32_t)t;
  }
}

// Per tile (one warp): exclusive prefix of its column's counts over the
// chunks of its row (in place, 32 chunks per round), tile total -> T.  The
// last CTA to finish forms the tile ranges and the launch order.
__global__ void __launch_bounds__(SCAN_T) k_tile_scan(uint32_t* __restrict__ C2, int nchunks,
                                                      const uint32_t* __restrict__ row_chunk0,
                                                      int ntx, int n_tiles, uint32_t* __restrict__ T,
                                                      uint2* __restrict__ ranges,
                                                      uint32_t* __restrict__ order,
                                                      uint32_t* __restrict__ done) {
  __shared__ bool last;
  const int t = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (t < n_tiles) {
    const int y = t / ntx, x = t - y * ntx;
    uint32_t* col = C2 + (size_t)x * nchunks;
    uint32_t run = 0;
    const uint32_t c1 = row_chunk0[y + 1];
    for (uint32_t c0 = row_chunk0[y]; c0 < c1; c0 += 32) {
      const uint32_t c = c0 + lane;
      const uint32_t v = c < c1 ? col[c] : 0u;
      uint32_t incl = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(FULLM, incl, o);
        if (lane >= o) incl += u;
      }
      if (c < c1) col[c] = run + incl - v;
      run += __shfl_sync(FULLM, incl, 31);
    }
    if (lane == 0) T[t] = run;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  tile_ranges_order(T, n_tiles, ranges, order);
}

// Without pairs: every tile empty, launch order = tile index.
__global__ void k_tiles_empty(int n_tiles, uint2* __restrict__ ranges, uint32_t* __restrict__ order) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n_tiles) {
    ranges[t] = make_uint2(0u, 0u);
    order[t] = (uint32_t)t;
  }
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

// scratch1: info {pairs, chunks2} (2 x u64) + done counters (2 x u32, padded)
//           + pairs_part [chunks1] + C1 [nty][chunks1] + S [nty] + row_chunk0 [nty + 1]
static constexpr size_t HDR = 32;
size_t span_scratch1_bytes(int64_t n, int nty) {
  const size_t c1 = (size_t)span_chunks1(n);
  return HDR + sizeof(uint32_t) * (c1 + (size_t)nty * c1 + 2 * (size_t)nty + 1);
}

cudaError_t span_rows_begin(int64_t n, const uint32_t* perm, const ushort4* rect, int nty,
                            void* scratch1, int* launches, cudaStream_t st) {
  using namespace span;
  const int nch = (int)span_chunks1(n);
  unsigned long long* info = (unsigned long long*)scratch1;
  uint32_t* done = (uint32_t*)(info + 2);
  uint32_t* part = (uint32_t*)((char*)scratch1 + HDR);
  uint32_t* C1 = part + nch;
  uint32_t* S = C1 + (size_t)nty * nch;
  uint32_t* rc0 = S + nty;
  cudaError_t e = cudaMemsetAsync(scratch1, 0, HDR, st);
  if (e != cudaSuccess || nch == 0) return e;
  k_rows_count<<<nch, CT, chunk_smem(nty), st>>>(n, perm, rect, nty, nch, C1, part);
  k_bucket_scan<<<nty, SCAN_T, 0, st>>>(C1, nch, S, nty, part, rc0, info, done);
  *launches += 2;
  return cudaGetLastError();
}

const unsigned long long* span_info(const void* scratch1) {
  return (const unsigned long long*)scratch1;
}

size_t span_scratch2_bytes(int64_t chunks2, int ntx, int n_tiles) {
  // spans [chunks2 * CH] (uint2) + C2 [ntx][chunks2] + T [n_tiles]
  return sizeof(uint2) * (size_t)chunks2 * span::CH +
         sizeof(uint32_t) * ((size_t)ntx * (size_t)chunks2 + (size_t)n_tiles);
}

cudaError_t span_finish(int64_t n, const uint32_t* perm, const ushort4* rect, int ntx, int nty,
                        void* scratch1, int64_t chunks2, void* scratch2, uint2* ranges,
                        uint32_t* order, uint32_t* vals, int* launches, cudaStream_t st) {
  using namespace span;
  const int nch1 = (int)span_chunks1(n);
  const int n_tiles = ntx * nty;
  if (chunks2 <= 0) {
    k_tiles_empty<<<(n_tiles + 255) / 256, 256, 0, st>>>(n_tiles, ranges, order);
    *launches += 1;
    return cudaGetLastError();
  }
  uint32_t* done = (uint32_t*)((unsigned long long*)scratch1 + 2) + 1;
  const uint32_t* R1 = (const uint32_t*)((char*)scratch1 + HDR) + nch1;
  const uint32_t* S = R1 + (size_t)nty * nch1;
  const uint32_t* rc0 = S + nty;
  uint2* spans = (uint2*)scratch2;
  uint32_t* C2 = (uint32_t*)(spans + (size_t)chunks2 * CH);
  uint32_t* T = C2 + (size_t)ntx * chunks2;
  k_rows_place<<<nch1, CT, chunk_smem(nty), st>>>(n, perm, rect, nty, nch1, R1, rc0, spans);
  const size_t sm2 = chunk_smem(ntx);
  k_cols_count<<<(unsigned)chunks2, CT, sm2, st>>>(spans, S, rc0, nty, ntx, (int)chunks2, C2);
  k_tile_scan<<<(n_tiles + SCAN_T / 32 - 1) / (SCAN_T / 32), SCAN_T, 0, st>>>(
      C2, (int)chunks2, rc0, ntx, n_tiles, T, ranges, order, done);
  k_cols_place<<<(unsigned)chunks2, CT, sm2, st>>>(spans, S, rc0, nty, ntx, (int)chunks2, C2,
                                                    ranges, vals);
  *launches += 4;
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
