// Launcher declarations shared by the kernel translation units and the C ABI.
#pragma once

#include "vg_common.cuh"

namespace vg {

// record the thread-local message of vg_last_error (vg_capi.cu); returns code
int set_error(int code, const char* msg);

struct BlendParams {
  int width, height, ntx;
  float cx, cy, fx, fy;
  float stop;      // early_stop * (1 - 2^-20)  (see blend_params)
  float cut;       // alpha_cut
  float clamp;     // alpha_clamp
  float cc;        // 1 - alpha_clamp (rounded once from float64): clamped transmittance factor
  float omcut;     // largest float below 1: a factor above it is a cut (or inactive) entry
  float e2cut;     // -log1p(-alpha_cut) log2(e): entries with e log2(e) below it are cut
  float ecut;      // culling threshold on e: -log1p(-alpha_cut) * (1 - 1e-3)
  float bg[3];
  // debug builds only (VG_ASSERT bounds, VG_JITTER seed)
  int64_t dbg_n = 0, dbg_pairs = 0;
  unsigned dbg_jitter = 0;
  // diagnostic CTA log (profiling build; vg_debug_cta_log): CTA b < dbg_cta_n
  // of a blend launch writes {start ns, end ns, (SM << 32) | tile, forward:
  // per-warp walk cycles [4], per-warp staging cycles [4]} to dbg_cta[16 b]
  unsigned long long* dbg_cta = nullptr;
  int dbg_cta_n = 0;
};

// compiled in only with -DVG_CTA_LOG=1 (build(profile=True)): even unexecuted,
// the log code changes the backward's register allocation (+3 % on config 3)
#ifndef VG_CTA_LOG
#define VG_CTA_LOG 0
#endif
constexpr int VG_CTA_LOG_STRIDE = 16;  // uint64 per CTA in the log
// (the start time waits in the log itself: no register is held across the kernel)
__device__ __forceinline__ void cta_log_begin(const BlendParams& p) {
  if (VG_CTA_LOG && p.dbg_cta && threadIdx.x == 0 && (int)blockIdx.x < p.dbg_cta_n) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    p.dbg_cta[VG_CTA_LOG_STRIDE * (size_t)blockIdx.x] = t;
  }
}
__device__ __forceinline__ void cta_log_end(const BlendParams& p, int tile) {
  if (!VG_CTA_LOG || !p.dbg_cta) return;
  __syncthreads();
  if (threadIdx.x == 0 && (int)blockIdx.x < p.dbg_cta_n) {
    unsigned long long t;
    unsigned sm;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    unsigned long long* o = p.dbg_cta + VG_CTA_LOG_STRIDE * (size_t)blockIdx.x;
    o[1] = t;
    o[2] = ((unsigned long long)sm << 32) | (unsigned)tile;
  }
}

#ifndef VG_BWD_MINB
// backward blend CTAs per SM requested from ptxas.  5: <= 96 registers.  With
// the cut decided on e (eval_pinhole2) the 80-register budget of 6 CTAs
// spilled: config 3, 16 views, serial: 6 -> 19.26 ms, 5 -> 18.01 ms, 4 -> 19.26 ms
#define VG_BWD_MINB 5
#endif

// Segmented backward (atomic mode).  Every forward that records the
// visibility mask adds its tiles' walked depths (list entries) to a total and
// a maximum; after the backward, the per-view accumulation pass turns them
// into the next view's decision and stores it to mapped host memory
// (seg_publish: one 8-byte store, no copy, no synchronisation, and no code in
// the register-bound blend kernels).
// When the previous view on the context had a tile deeper than the per-slot
// share of its total work (max depth x backward CTA slots > total depth: its
// backward ended on a few long tiles), the host turns segmentation on for the
// next view (SegIO::on), and that forward also (a) stores, at every VG_SEG-entry
// boundary of a tile's list that it reaches, each pixel's transmittance and
// colour sums (state: two float4 per thread, at index boundary / VG_SEG --
// unique, since boundaries of different tiles lie more than VG_SEG apart), and
// (b) appends its tile's backward work items to SEG_BINS bins by work (half
// an octave per bin, heaviest first): VG_SEG-entry segments for a tile deeper
// than `thr` (half the per-slot share, within a budget of extra items), one
// whole-tile item otherwise.  The backward then maps its CTA index over the
// bins in order and runs every item as an independent CTA, a segment starting
// its replay from the recorded state; otherwise it runs one CTA per tile in
// list-length order.  No planning launch: the counters sit after the
// visibility mask and are cleared with it.  Deterministic mode never
// segments: a segment's replay seeds its running sum from the forward's
// colour sums, which rounds differently from the unsegmented replay, and the
// decision depends on the previous view.  The same decision sends a
// tail-bound view's longest-list tiles through the deep-tile forward (both
// modes: its results are bit-identical).  (Config 4: backward -29 %, step
// 33.6 -> 31.3 ms with both; config 3 never segments.)
#ifndef VG_SEG
#define VG_SEG 1024
#endif
static_assert((VG_SEG & (VG_SEG - 1)) == 0 && VG_SEG >= 256, "VG_SEG: a power of two >= BATCH");
constexpr int SEG_BINS = 32;
constexpr uint32_t SEG_WHOLE = 0x80000000u;  // item flag: the whole tile list
struct SegIO {
  float4* state = nullptr;       // forward writes, backward reads
  uint32_t* counts = nullptr;    // [SEG_BINS] items per bin, extra-item budget used, pad,
                                 // then 2 x uint64 {total depth, max depth} of this forward
  uint2* items = nullptr;        // [SEG_BINS][cap] (tile, segment | SEG_WHOLE)
  uint32_t cap = 0;              // items per bin: n_tiles + budget
  uint32_t budget = 0;           // extra (split) items allowed
  uint32_t thr = 0;              // split tiles deeper than this
  uint32_t n_tiles = 0;
  uint32_t slots = 1;            // backward CTA slots (SMs x resident CTAs)
  float ratio = 1.f;             // segment when max depth x slots > ratio x total depth
  int on = 0;                    // this view is segmented
  unsigned long long* decision = nullptr;  // mapped host: (thr << 32) | on, for the next view
};
constexpr int SEG_THREADS = 128;    // threads of a blend CTA (NT in vg_blend.cuh)
inline size_t seg_state_bytes(int64_t pairs) {
  return sizeof(float4) * 2 * SEG_THREADS * (size_t)(pairs / VG_SEG + 1);
}
constexpr int SEG_STATS = SEG_BINS + 4;  // uint32 index of the uint64 stats
constexpr size_t SEG_COUNT_BYTES = sizeof(uint32_t) * SEG_STATS + 2 * sizeof(unsigned long long);
// the next view's decision from this view's (finished) forward statistics
__device__ __forceinline__ void seg_publish(const uint32_t* counts, unsigned long long* decision,
                                            uint32_t slots, float ratio) {
  const unsigned long long* st = reinterpret_cast<const unsigned long long*>(counts + SEG_STATS);
  const unsigned long long total = __ldcg(st), mx = __ldcg(st + 1);
  const unsigned long long on = total > 0 && (double)mx * slots > (double)ratio * (double)total;
  const unsigned long long thr = min(0xffffffffull, max(2ull * VG_SEG, total / (2ull * slots)));
  *(volatile unsigned long long*)decision = (thr << 32) | on;
}
// half-octave bins: 0 = 2^14 entries or more, ..., SEG_BINS - 1 = none
__device__ __forceinline__ int seg_bin(uint32_t w) {
  if (w == 0) return SEG_BINS - 1;
  const int e = 31 - __clz(w);                                  // floor(log2 w)
  if (e >= 15) return 0;
  const int upper = e ? (int)((w >> (e - 1)) & 1u) : 0;         // w >= 1.5 * 2^e
  const int b = 2 * (14 - e) + 1 - upper;
  return b < 0 ? 0 : (b > SEG_BINS - 2 ? SEG_BINS - 2 : b);
}

struct BwdIO {
  const float* color;
  const float* final_t;
  const float* d_color;     // explicit upstream gradient (LOSS == 0)
  const float* d_t;         // optional dL/dT_final (LOSS == 0)
  const float* target;      // fused L2 (LOSS == 1)
  float loss_scale;         // 2 / (H W 3)
  double* loss_sum;         // fused L2: sum of squared residuals
  float* acc;               // per-Gaussian accumulators, 16 floats each
  uint8_t* visible;
  float* d_background;
  // deterministic mode (vg_det.cu): per (entry, warp) slots and per-tile partials
  float* det_part = nullptr;
  float* det_bg = nullptr;
  double* det_loss = nullptr;
  // Gaussian-major slots (render backward with a forward visibility mask): the
  // (entry, warp w) partial of Gaussian g in tile (tx, ty) goes to slot
  // 4 (det_off[g] + (ty - y0) W + (tx - x0)) + w, with (x0, y0, W) from g's
  // tile rectangle det_rect[g], and det_gvis4 at the same (Gaussian, tile)
  // index gets the entry's four warp-visibility bits; slots of invisible
  // pairs are never written nor read
  const uint32_t* det_off = nullptr;
  const ushort4* det_rect = nullptr;
  uint8_t* det_gvis4 = nullptr;
};

// gm (nullable): per binned Gaussian M and M (mean - centre) in float64, for sort_by="gamma"
// splat: mode="splat" records (conic, opacity) and 3-sigma radii
void launch_preprocess(int64_t n, const vg_scene& s, const CamK& c, double bin_cut, GRec* rec,
                       float* depth, ushort4* rect, float* frame, double* gm, bool splat,
                       cudaStream_t st);
// mode="splat" tile kernels (vg_splat.cu)
void launch_splat_fwd(int n_tiles, const GRec* rec, const uint32_t* vals, const uint2* ranges,
                      const uint32_t* order, const BlendParams& p, float* color, float* final_t,
                      int* n_contrib, int* n_act, cudaStream_t st);
void launch_splat_bwd(int n_tiles, const GRec* rec, const uint32_t* vals, const uint2* ranges,
                      const uint32_t* order, const BlendParams& p, int loss, const BwdIO& io,
                      cudaStream_t st);
// deterministic-gradient mode (vg_det.cu)
cudaError_t scan_u32(const uint32_t* in, uint32_t* out, void* scratch, uint32_t* total, int64_t n,
                     cudaStream_t st);
size_t scan_u32_scratch_bytes(int64_t n);
size_t det_part_bytes(int64_t pairs);
// cnt[g] = tiles of g's rectangle, off = their exclusive scan; slot (nullable):
// the pair-major map (g's k-th tile -> its list position)
cudaError_t det_prepare(int64_t n, const ushort4* rect, const uint2* ranges, const uint32_t* vals,
                        int n_tiles, int ntx, uint32_t* cnt, uint32_t* off, uint32_t* slot,
                        void* scan_scratch, uint32_t* total, cudaStream_t st);
cudaError_t det_reduce(int64_t n, const uint32_t* cnt, const uint32_t* off, const uint32_t* slot,
                       const float* part, float* acc, int n_tiles, const float* bg_part,
                       const double* loss_part, float* d_background, double* loss_sum,
                       cudaStream_t st, const uint8_t* gvis4 = nullptr,
                       uint32_t* big_scratch = nullptr);  // gvis4: n + 1 uint32
// deterministic VG_DEFER: out += (bg[3], loss); the sums are cleared
void launch_det_flush(float* bg, double* loss, float* bg_out, double* loss_out, cudaStream_t st);
// sort_by="gamma" re-sort of every tile list (vg_gamma.cu)
size_t gamma_scratch_bytes(int64_t pairs);
void launch_gamma_sort(int n_tiles, const uint2* ranges, uint32_t* vals, const double* gm,
                       int64_t pairs, void* scratch, const CamK& cam, cudaStream_t st);
// vmask (optional): per-warp bit rows of vm_words words marking the list
// entries where the forward saw a visible pixel (the backward's work list).
void launch_render_fwd(int n_tiles, const GRec* rec, const uint32_t* vals, const uint2* ranges,
                       const uint32_t* order, const BlendParams& p, bool stop, bool cut,
                       float* color, float* final_t, int* n_contrib, int* n_act, uint32_t* vmask,
                       int vm_words, cudaStream_t st, const SegIO& seg = SegIO());
// the latency-bound variant for the deepest tiles of a tail-bound view (the
// training forward; run beside launch_render_fwd on the remaining tiles)
void launch_render_fwd_deep(int n_tiles, const GRec* rec, const uint32_t* vals, const uint2* ranges,
                            const uint32_t* order, const BlendParams& p, bool stop, bool cut,
                            float* color, float* final_t, uint32_t* vmask, int vm_words,
                            cudaStream_t st, const SegIO& seg);
int debug_forward_stats(int n_tiles, const GRec* rec, const uint32_t* vals, const uint2* ranges,
                        const uint32_t* order, const BlendParams& p, float* color, float* final_t,
                        int* n_contrib, int* n_act, unsigned long long* out, cudaStream_t st);
void launch_render_bwd(int n_tiles, const GRec* rec, const uint32_t* vals, const uint2* ranges,
                       const uint32_t* order, const BlendParams& p, bool cut, int loss,
                       const BwdIO& io, const uint32_t* vmask, int vm_words, cudaStream_t st,
                       const SegIO& seg = SegIO());
// Tomography splits each tile's pair list over `splits` CTAs (small detectors
// with long lists would otherwise leave most SMs idle): the forward writes
// per-split partial images into `part` (splits * H * W floats, unused when
// splits == 1) and sums them in split order; the adjoint's pairs are
// independent.
void launch_tomo_fwd(int n_tiles, int ray, const GRec* rec, const uint32_t* vals,
                     const uint2* ranges, const uint32_t* order, const BlendParams& p,
                     float* image, float* intensity, int splits, float* part, cudaStream_t st);
void launch_tomo_bwd(int n_tiles, int splits, int ray, int loss, const GRec* rec, const uint32_t* vals,
                     const uint2* ranges, const uint32_t* order, const BlendParams& p,
                     const float* d_image,
                     const float* image, const float* target, float loss_scale, double* loss_sum,
                     float* acc, uint8_t* visible, float* det_part, double* det_loss,
                     cudaStream_t st);
// SH scenes: dcol / center receive this view's dL/dRGB slab [3][n] and camera centre
// seg (nullable): publish the segmentation decision (seg_publish) from block 0
void launch_view_accumulate(int64_t n, const vg_scene& s, const CamK& c, const float* frame,
                            float* acc, float* lacc, float* cacc, float* dcol, double* center,
                            bool splat, cudaStream_t st, const SegIO* seg = nullptr);
// returns the number of kernels launched; SH scenes fold the sh_views slabs of dcol
void launch_merge_acc(int64_t n, float* dst, float* src, cudaStream_t st);
int launch_finalize_params(int64_t n, const vg_scene& s, float* lacc, float* cacc,
                           const float* dcol, const double* centers, int sh_views,
                           const vg_grads& g, bool splat, cudaStream_t st);

// hand-written onesweep radix sort (vg_radix.cu); result buffer in *which
size_t radix_temp_bytes(int64_t n, int key_bits);
// identity_values: v0 is not read, the values start as 0..n-1 (stable index order)
cudaError_t radix_sort_u32(void* tmp, size_t tmp_bytes, uint32_t* k0, uint32_t* k1, uint32_t* v0,
                           uint32_t* v1, int64_t n, int key_bits, int* which, int* launches,
                           cudaStream_t st, bool identity_values = false);
cudaError_t radix_sort_u16(void* tmp, size_t tmp_bytes, uint16_t* k0, uint16_t* k1, uint32_t* v0,
                           uint32_t* v1, int64_t n, int key_bits, int* which, int* launches,
                           cudaStream_t st);
// span binning (vg_span.cu): per-tile lists in depth order without a pair sort.
// begin (before the host sync): step-1 counts; span_info(scratch1) = {pairs, step-2 chunks}.
int span_max_buckets();
cudaError_t span_configure();
size_t span_scratch1_bytes(int64_t n, int nty);
cudaError_t span_rows_begin(int64_t n, const uint32_t* perm, const ushort4* rect, int nty,
                            void* scratch1, int* launches, cudaStream_t st);
const unsigned long long* span_info(const void* scratch1);
size_t span_scratch2_bytes(int64_t chunks2, int ntx, int n_tiles);
cudaError_t span_finish(int64_t n, const uint32_t* perm, const ushort4* rect, int ntx, int nty,
                        void* scratch1, int64_t chunks2, void* scratch2, uint2* ranges,
                        uint32_t* order, uint32_t* vals, int* launches, cudaStream_t st);

}  // namespace vg
