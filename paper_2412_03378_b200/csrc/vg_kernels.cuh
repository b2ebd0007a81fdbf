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
};

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
                       int vm_words, cudaStream_t st);
int debug_forward_stats(int n_tiles, const GRec* rec, const uint32_t* vals, const uint2* ranges,
                        const uint32_t* order, const BlendParams& p, float* color, float* final_t,
                        int* n_contrib, int* n_act, unsigned long long* out, cudaStream_t st);
void launch_render_bwd(int n_tiles, const GRec* rec, const uint32_t* vals, const uint2* ranges,
                       const uint32_t* order, const BlendParams& p, bool cut, int loss,
                       const BwdIO& io, const uint32_t* vmask, int vm_words, cudaStream_t st);
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
void launch_view_accumulate(int64_t n, const vg_scene& s, const CamK& c, const float* frame,
                            float* acc, float* lacc, float* cacc, float* dcol, double* center,
                            bool splat, cudaStream_t st);
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
