/*
 * volgauss_b200 -- C ABI of the B200-native (sm_100a) analytic-transmittance
 * Gaussian rasterizer (arXiv 2412.03378).
 *
 * This is the drop-in boundary for the reference package `volgauss` 0.1.0,
 * whose hot path is the Python API in pkg/src/volgauss/{raster,grad,tomo}.py.
 * The reference has no FFI of its own (it is pure numpy); each entry point
 * below replaces one reference call, cited as file:line relative to
 * /root/reference/pkg/src/volgauss/.  The Python facade
 * (paper_2412_03378_b200/{raster,grad,tomo}.py) binds these symbols through
 * ctypes and keeps the reference signatures; INTEGRATION.md shows the
 * binding.
 *
 * Conventions
 *  - All array arguments are DEVICE pointers (cudaMalloc / torch CUDA
 *    storage), float32 struct-of-arrays in the reference field order:
 *    means N*3, scales N*3, rotations N*4 (w,x,y,z; need not be unit),
 *    thetas N, colors N*3.  Images are row-major (H, W[, 3]).
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy stream).
 *    Every call is stream-ordered; nothing synchronises the host except
 *    vg_pair_count (which reads the pair count back).
 *  - Return codes: VG_OK, VG_EINVAL (bad argument -> the facade raises
 *    ValueError like raster.py:268-269, 293-294), VG_ECUDA (CUDA error ->
 *    RuntimeError), VG_ENOMEM.  vg_last_error() returns a thread-local
 *    message for the last failing call on this thread.
 *  - A context is not thread-safe; use one per (device, stream).  It owns
 *    the preprocessed records, the sorted tile lists and the per-pixel
 *    forward state that backward reuses (the reference's `prep`,
 *    raster.py:123-145, reused by optim.py:379-386).
 */
#ifndef VOLGAUSS_B200_H
#define VOLGAUSS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VG_ABI_VERSION 1

#define VG_OK 0
#define VG_EINVAL 1
#define VG_ECUDA 2
#define VG_ENOMEM 3

/* ray models */
#define VG_PINHOLE 0  /* camera.Camera pinhole rays from the centre (camera.py:57-64) */
#define VG_PARALLEL 1 /* orthographic detector of half-width `extent` (tomo.py:272-282) */

typedef struct vg_context vg_context;

/* camera.Camera (camera.py:14-48): x_view = R x_world + t */
typedef struct {
  int32_t width, height;
  int32_t projection; /* VG_PINHOLE or VG_PARALLEL */
  int32_t _pad;
  double fx, fy, cx, cy;
  double rotation[9]; /* row-major */
  double translation[3];
  double z_near;
  double extent; /* parallel detector half-width (world units) */
} vg_camera;

/* render()/backward() keyword flags (raster.py:26-35, 410-413) */
typedef struct {
  int32_t tile_size;   /* only 16 is supported (raster.TILE_SIZE) */
  int32_t _pad;
  double early_stop;   /* <= 0 disables early termination (early_stop=None) */
  double alpha_cut;    /* <= 0 disables the alpha skip (alpha_cut=0) */
  double alpha_clamp;  /* raster.ALPHA_CLAMP */
  double bin_cut;      /* alpha_cut used for bin radii: raster.prepare's
                          alpha_cut, or tomo.TOMO_BIN_CUT (tomo.py:28) */
  int32_t sort_by;     /* VG_SORT_DEPTH (default) or VG_SORT_GAMMA (raster.py:291-312) */
  int32_t deterministic; /* != 0: bitwise-reproducible backward (fixed-order reductions,
                            like the reference's tile-order sum, grad.py:188-204) */
  int32_t mode;        /* VG_MODE_ANALYTIC (default) or VG_MODE_SPLAT (the EWA comparator) */
  int32_t _pad3;
} vg_options;

/* render mode (raster.prepare's mode, raster.py:268-269) */
#define VG_MODE_ANALYTIC 0 /* analytic transmittance (the paper's method) */
#define VG_MODE_SPLAT 1    /* EWA splatting: opacity * exp(-maha/2) (raster.py:353-361) */

/* per-tile list order (raster.prepare's sort_by) */
#define VG_SORT_DEPTH 0 /* (tile, float32 view depth, index) */
#define VG_SORT_GAMMA 1 /* stable re-sort by gamma along each tile's central ray */

/* raster.Scene (raster.py:38-97) as device float32 SoA */
typedef struct {
  const float* means;
  const float* scales;
  const float* rotations;
  const float* thetas;
  const float* colors;  /* may be NULL for tomography */
  const float* sh;      /* optional N*16*3 SH-3 coefficients; when set, colors
                           are evaluated per view from sh (DC band = RGB) */
  int64_t n;
  double background[3];
  const float* splat_opacities; /* N, mode="splat" only (raster.Scene.splat_opacities) */
} vg_scene;

/* grad.SceneGrads (grad.py:41-69) as device pointers.  Any pointer may be
 * NULL to skip that output.  `accumulate` selects how a backward call writes:
 *   VG_OVERWRITE  this view's gradients overwrite every output;
 *   VG_ADD        this view's gradients are added to every output;
 *   VG_DEFER      multi-view accumulation: colour/SH gradients, d_background
 *                 and visible are added now, the per-Gaussian geometry chain
 *                 (means/scales/rotations/thetas/kappas) is summed over views
 *                 inside the context and written by vg_finalize_grads.  With
 *                 vg_options.deterministic, d_background and the fused-L2 loss
 *                 are also summed inside the context (in view order) and added
 *                 by vg_finalize_grads, so deferred views on different
 *                 contexts may run concurrently and stay bitwise reproducible. */
#define VG_OVERWRITE 0
#define VG_ADD 1
#define VG_DEFER 2
typedef struct {
  float* d_means;      /* N*3 */
  float* d_scales;     /* N*3 */
  float* d_rotations;  /* N*4 */
  float* d_thetas;     /* N   */
  float* d_colors;     /* N*3 */
  float* d_kappas;     /* N   */
  float* d_sh;         /* N*48, only with vg_scene.sh */
  float* d_background; /* 3   */
  uint8_t* visible;    /* N   (OR-accumulated) */
  int32_t accumulate;  /* VG_OVERWRITE, VG_ADD or VG_DEFER */
  int32_t _pad;
  float* d_splat_opacities; /* N, mode="splat" (zero in analytic mode) */
} vg_grads;

/* lifecycle */
int vg_abi_version(void);
const char* vg_last_error(void);
int vg_create(vg_context** out, int32_t device);
void vg_destroy(vg_context* ctx);

/* raster.prepare (raster.py:263-296) / bin_tiles (raster.py:315-319):
 * per-Gaussian projection, bounding radius and tile rectangle
 * (_project_all/_bounding_radii, raster.py:154-209), blend records, the
 * depth radix sort of the Gaussians and the span binning into per-tile lists
 * in (tile, depth, index) order with their ranges (_build_grid,
 * raster.py:222-260); with opt->sort_by == VG_SORT_GAMMA each list is then
 * re-sorted by gamma (_resort_by_gamma, raster.py:299-312).  The scene pointers must stay valid
 * until the matching backward has run. */
int vg_prepare(vg_context* ctx, const vg_scene* scene, const vg_camera* cam,
               const vg_options* opt, void* stream);

/* vg_prepare split in two for pipelining: _async enqueues projection, the
 * depth sort and the pair-count scan and returns without waiting; _finish
 * waits only for that count (an event, not the stream), then enqueues the
 * pair duplication, tile sort and ranges.  Issuing view v+1's _async on one
 * context before view v's blend on another hides the count read-back. */
int vg_prepare_async(vg_context* ctx, const vg_scene* scene, const vg_camera* cam,
                     const vg_options* opt, void* stream);
int vg_prepare_finish(vg_context* ctx, void* stream);

/* Update the blend flags (early_stop, alpha_cut, alpha_clamp) of a prepared
 * context without re-binning -- render(prep=...) may pass flags that differ
 * from prepare's (raster.py:410-418).  bin_cut and tile_size are ignored. */
int vg_set_options(vg_context* ctx, const vg_options* opt);

/* Number of (tile, primitive) pairs of the last vg_prepare (synchronises). */
int vg_pair_count(vg_context* ctx, int64_t* out_pairs);

/* TileGrid.tiles (raster.py:100-112): the sorted per-tile primitive lists,
 * flattened.  prims: device int32[pairs]; offsets: device int32[n_tiles+1]. */
int vg_tile_lists(vg_context* ctx, int32_t* prims, int32_t* offsets, void* stream);

/* raster.render (raster.py:410-439), analytic mode: color (H,W,3),
 * final_transmittance (H,W), n_contrib (H,W).  n_contrib may be NULL: the
 * per-pixel counts (n_contrib and the active-entry counts of vg_n_active) are
 * then not computed -- the training-step forward; the backward does not need
 * them. */
int vg_render_forward(vg_context* ctx, float* color, float* final_t, int32_t* n_contrib,
                      void* stream);

/* grad.backward (grad.py:107-213), analytic mode.  color/final_t are the
 * outputs of the matching vg_render_forward; d_color (H,W,3) and optional
 * d_transmittance (H,W) are dL/d(outputs). */
int vg_render_backward(vg_context* ctx, const float* color, const float* final_t,
                       const float* d_color, const float* d_transmittance, vg_grads* grads,
                       void* stream);

/* Fused L2 training step: grad.loss_and_grad(l2) (grad.py:346-348) folded
 * into the backward blend.  dL/dcolor = 2 (color - target) / (H*W*3) is
 * formed per pixel in the kernel and sum((color-target)^2) is ADDED to
 * *loss_sum (device float64). */
int vg_render_backward_l2(vg_context* ctx, const float* color, const float* final_t,
                          const float* target, double* loss_sum, vg_grads* grads,
                          void* stream);

/* Per-pixel count of composited (active) entries of the last forward,
 * int32 (H,W) -- the roofline's A count; needs a counting forward
 * (n_contrib != NULL). */
int vg_n_active(vg_context* ctx, int32_t* out, void* stream);

/* Number of (entry, 64-pixel warp block) pairs the last forward marked
 * visible -- the pairs the backward blend walks (its algorithmic unit count;
 * x 64 = visible pair-pixels).  Synchronises; 0 when the forward kept no
 * visibility mask (alpha_cut == 0 or splat mode).  Diagnostic, no reference
 * counterpart. */
int vg_visible_pairs(vg_context* ctx, int64_t* out);

/* tomo.tomo_forward (tomo.py:34-57): line-integral image (H,W).  Pass
 * intensity != NULL to also write exp(-image). */
int vg_tomo_forward(vg_context* ctx, float* image, float* intensity, void* stream);

/* tomo.tomo_backward (tomo.py:60-103): gradients of sum(d_image * image). */
int vg_tomo_backward(vg_context* ctx, const float* d_image, vg_grads* grads, void* stream);

/* Fused tomography L2 step: d_image = 2 (image - target) / (H*W) in-kernel,
 * sum((image-target)^2) added to *loss_sum. */
int vg_tomo_backward_l2(vg_context* ctx, const float* image, const float* target,
                        double* loss_sum, vg_grads* grads, void* stream);

/* tomo.voxelize (tomo.py:345-389): the mixture density sum_i kappa_i
 * exp(-q_i/2) at the cell centres of a shape[0] x shape[1] x shape[2] grid over
 * [bbox_min, bbox_max] (C order, float64, device `out`), each primitive culled
 * to a box of 5 largest standard deviations and q <= 25 like the reference. */
int vg_voxelize(const vg_scene* scene, const double* bbox_min, const double* bbox_max,
                const int32_t* shape, double* out, void* stream);

/* Copy `bytes` between device memory and pinned host memory (a mapped
 * pointer) with `ctas` CTAs of a streaming kernel (evict-first cache hints:
 * the transfer does not flush the L2 working set of concurrent kernels).
 * Either pointer may be device or mapped host memory. */
int vg_copy_streaming(void* dst, const void* src, size_t bytes, int32_t ctas, void* stream);

/* Move the VG_DEFER accumulators of `src` (same scene, same device) into `dst`
 * (src is left empty), so one vg_finalize_grads on dst covers the views of
 * both contexts: one parameter-chain pass per step instead of one per
 * context.  Ordered on `stream`. */
int vg_merge_deferred(vg_context* dst, vg_context* src, void* stream);

/* Write the geometry gradients accumulated by VG_DEFER backward calls
 * (analytic_param_chain, grad.py:242-259) into grads (overwrite when
 * grads->accumulate == VG_OVERWRITE, else add) and reset the accumulator. */
int vg_finalize_grads(vg_context* ctx, vg_grads* grads, void* stream);

/* Number of kernels this context launched since creation (bench accounting). */
int64_t vg_launch_count(vg_context* ctx);

/* Per-kernel device timing with CUDA events recorded on the launch stream.
 * vg_profile(ctx, 1) clears and enables, (ctx, 0) disables.  vg_profile_read
 * waits for the recorded events and returns, per kernel kind (VG_K_*),
 * the summed milliseconds and launch counts (arrays of VG_K_COUNT). */
#define VG_K_PREPROCESS 0
#define VG_K_SCAN 1
#define VG_K_DUPLICATE 2
#define VG_K_SORT 3
#define VG_K_RANGES 4
#define VG_K_RENDER_FWD 5
#define VG_K_RENDER_BWD 6
#define VG_K_FINALIZE 7
#define VG_K_TOMO_FWD 8
#define VG_K_TOMO_BWD 9
#define VG_K_COUNT 10
int vg_profile(vg_context* ctx, int32_t enable);
int vg_profile_read(vg_context* ctx, double* ms, int64_t* counts);

/* ---------------------------------------------------------------------------
 * Training-step caller: optim.Trainer.step + GradAccum
 * (optim.py:119-206) and the device half of densify_and_prune
 * (optim.py:218-317).  Scene arrays are updated in place. */

/* Trainer state on the device (float32).  moments: per primitive 14 Adam
 * first moments then 14 second moments, in the order position (3), scale (3),
 * rotation (4), colour (3, of the pre-softplus colour), density (1). */
typedef struct {
  float* means;
  float* scales;
  float* rotations;
  float* thetas;
  float* colors;
  float* color_raw;    /* N*3 pre-softplus colours (optim.py:128) */
  float* moments;      /* N*28 */
  float* accum_norm;   /* optional GradAccum (optim.py:194-206): N */
  float* accum_count;  /* N */
  int64_t n;
} vg_train_state;

/* optim.Adam (optim.py:84-107) hyper-parameters for one step; lr in group
 * order position (already scheduled: optim.py:140-144), scale, rotation,
 * colour, density; t = the step count after this step (>= 1). */
typedef struct {
  double lr[5];
  double beta1, beta2, eps;
  int64_t t;
} vg_adam_hparams;

/* One Trainer.step (optim.py:146-175) fused with GradAccum.update: Adam on
 * every group, then means -= u, scales floored at 1e-7, quaternions
 * renormalised, colours through softplus, thetas clipped to [0, 1].  The
 * gradients are a vg_grads (d_means, d_scales, d_rotations, d_thetas,
 * d_colors and visible are read).  bad: device int32[5], set to the first
 * primitive whose update is non-finite per group (INT32_MAX if none) -- the
 * caller raises DivergenceError (optim.py:159-164) after reading it. */
int vg_adam_step(vg_train_state* state, const vg_grads* grads, const vg_adam_hparams* hp,
                 int32_t* bad, void* stream);

/* densify_and_prune inputs (optim.TrainConfig fields, optim.py:24-53). */
typedef struct {
  int64_t n;
  const float* means;
  const float* scales;
  const float* rotations;
  const float* thetas;
  const float* colors;
  const float* color_raw;
  const float* moments;
  const float* accum_norm;
  const float* accum_count;
  double extent;
  double split_grad_threshold, clone_grad_threshold, prune_theta_min;
  double prune_scale_fraction, high_kappa_split_fraction;
  int64_t max_primitives;
} vg_densify_args;

/* Scratch for vg_densify_plan / vg_densify_apply (device bytes). */
size_t vg_densify_scratch_bytes(int64_t n);

/* Split / clone / prune decisions with the primitive budget
 * (optim.py:224-240, 292-297).  counts: device uint32[4] = {growing before
 * the budget, kept, splits, clones}; the per-primitive decisions stay in
 * scratch for vg_densify_apply. */
int vg_densify_plan(const vg_densify_args* args, void* scratch, uint32_t* counts, void* stream);

/* Write the densified state into `out` (sized kept + 2*(splits + clones)):
 * kept rows in order, then two children per split parent (means offset by
 * R diag(s) xi, scales / 1.6), then two per clone parent; children halve
 * kappa (theta clamped at the ceiling), copy rotation and colour, and start
 * with zero Adam moments.  counts_host: the counts of vg_densify_plan;
 * xi: device float64[splits*6], the standard normals the reference draws
 * per split parent (rng.standard_normal((2, 3)), optim.py:282). */
int vg_densify_apply(const vg_densify_args* args, const void* scratch,
                     const uint32_t* counts_host, const double* xi, vg_train_state* out,
                     void* stream);

/* oracle.raymarch_image (oracle.py:80-161): ground-truth midpoint-rule
 * quadrature of the volume rendering equation through the full mixture
 * density, independent of the closed-form path (validation tool; brute force
 * over all primitives, float64).  t_min / t_max: NaN = the reference's
 * auto-fitted bounds (support_sigmas beta around gamma, clipped to t >= 0).
 * color (H,W,3) and final_t (H,W) device float32. */
int vg_raymarch(const vg_scene* scene, const vg_camera* cam, int32_t n_steps,
                double support_sigmas, double t_min, double t_max, float* color, float* final_t,
                void* stream);

/* ---------------------------------------------------------------------------
 * Multi-GPU gradient exchange (SURVEY 8(b) vg_allreduce_grads, 8(e)).  The
 * reference sums per-view gradients one view per iteration
 * (optim.py:367-378); the view-sharded step renders each rank's views into
 * one flat float32 gradient buffer, then one NCCL group sums it over the
 * ranks.  NCCL is resolved at run time (the libnccl.so.2 already loaded in
 * the process, else VG_NCCL_LIB, else the loader path), so this library has
 * no link-time NCCL dependency.  Communicators are plain `ncclComm_t`
 * handles passed as void*: one from vg_nccl_comm_init, or any the caller
 * built with NCCL itself. */

/* 1 if NCCL could be resolved in this process, else 0 (vg_last_error says why). */
int vg_nccl_available(void);
/* ncclGetUniqueId: 128 bytes for rank 0 to broadcast to the other ranks. */
int vg_nccl_unique_id(void* out128);
/* ncclCommInitRank on `device` (collective over the nranks processes). */
int vg_nccl_comm_init(void** comm, int32_t nranks, const void* id128, int32_t rank, int32_t device);
int vg_nccl_comm_destroy(void* comm);
/* Stream-ordered, in place, in one NCCL group: flat[0..count) summed
 * (float32), visible[0..n_visible) OR-ed (uint8 max; NULL/0 to skip), *loss
 * summed (float64; NULL to skip).  Afterwards every rank holds the gradient
 * of all views, equal to the sum of the per-view reference SceneGrads. */
int vg_allreduce_grads(vg_context* ctx, void* nccl_comm, float* flat, int64_t count, uint8_t* visible,
                       int64_t n_visible, double* loss, void* stream);

/* Diagnostic (roofline counts, not on the hot path): re-run the forward of
 * the prepared view with counters and return out4 = {evaluated (list entry,
 * 8x8 warp block) pairs -- the pairs whose block the culling could not
 * exclude, each evaluated at 64 pixels --, of which any pixel was visible,
 * list entries walked per warp, 0}.  Writes color / final_t / n_contrib like
 * vg_render_forward.  Synchronises the stream. */
int vg_debug_forward_stats(vg_context* ctx, float* color, float* final_t, int32_t* n_contrib,
                           unsigned long long* out4, void* stream);

/* Diagnostic (load balance, tools/walk_stats.py; profiling build only,
 * -DVG_CTA_LOG=1, else VG_EINVAL): while log != NULL, every forward /
 * backward blend launch of this context writes, for CTA b < n, {start ns,
 * end ns, (SM id << 32) | tile} (globaltimer) and, for the forward, each
 * warp's chunk-walk and staging cycles to the device buffer log[16 b ..
 * 16 b + 10].  log = NULL turns it off. */
int vg_debug_cta_log(vg_context* ctx, unsigned long long* log, int n);

/* Diagnostic: the load-balance plan of the last forward of this context --
 * *segmented bit 0: its backward runs (tile, segment) work items
 * (vg_kernels.cuh, SegIO), *items = their count (else 0, one CTA per tile);
 * bit 1: its deepest tiles ran through the deep-tile forward.  Synchronises
 * the device. */
int vg_debug_segments(vg_context* ctx, int64_t* items, int32_t* segmented);

/* Roofline denominators measured at the live clock: FP32 FFMA lane-ops/s and
 * MUFU ex2 ops/s over all SMs of `device`. */
int vg_probe_peaks(int32_t device, double* fp32_per_s, double* mufu_per_s);

#ifdef __cplusplus
}
#endif

#endif /* VOLGAUSS_B200_H */
