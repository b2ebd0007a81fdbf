// The C ABI (include/volgauss_b200.h): context management and orchestration
// of the kernel pipeline  K1 preprocess -> scan -> K2 duplicate -> K3 radix
// sort -> K4 ranges -> K5/K6/K8 tile kernels -> K7 finalize.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "vg_kernels.cuh"

using namespace vg;

static thread_local std::string g_err;

static int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

namespace vg {
int set_error(int code, const char* msg) { return fail(code, msg); }
}  // namespace vg

#define VG_CUDA(call)                                                                      \
  do {                                                                                     \
    cudaError_t _e = (call);                                                               \
    if (_e != cudaSuccess)                                                                 \
      return fail(VG_ECUDA, std::string(#call) + ": " + cudaGetErrorString(_e));           \
  } while (0)

#define VG_LAUNCHED(ctx, k)                                                                \
  do {                                                                                     \
    (ctx)->launches += (k);                                                                \
    cudaError_t _e = cudaGetLastError();                                                   \
    if (_e != cudaSuccess) return fail(VG_ECUDA, std::string("launch: ") + cudaGetErrorString(_e)); \
  } while (0)

struct Buf {
  void* p = nullptr;
  size_t bytes = 0;
};

struct vg_context {
  int device = 0;
  int64_t launches = 0;
  // per-Gaussian
  Buf rec, depth, rect, offset, acc;
  // per-pair (double-buffered for the radix sort)
  Buf vals0;                         // per-tile Gaussian lists (depth order), P entries
  Buf ranges, n_act;
  Buf tord;                          // heavy-first tile launch order
  Buf span1, span2;                  // span-binning scratch (vg_span.cu)
  Buf dkey, perm, dsort_tmp;         // depth pre-sort of the Gaussians
  Buf frame, lacc;                   // per-view e-frames; view-independent grad accumulators
  Buf cacc;                          // RGB gradient accumulators, SoA [3][N]
  Buf gm, gscratch;                  // sort_by="gamma": per-Gaussian M, M delta; merge scratch
  Buf det_part, det_cnt, det_off, det_slot, det_bg, det_loss, det_scan;  // deterministic mode
  bool det_ready = false;            // det_cnt / det_off describe the lists of the last prepare
  bool det_slots_ready = false;      // ... and det_slot maps them (pair-major slots)
  Buf dcol, centers;                 // SH scenes: per-view dL/dRGB slabs [V][3][N] + centres
  int sh_views = 0;                  // views in dcol since the last parameter chain
  Buf tpart;                         // tomography forward: per-split partial images
  Buf det_gvis4, det_big;             // deterministic mode: warp bits per (Gaussian, tile); large-Gaussian queue
  // deterministic VG_DEFER: d_background (3 floats) and loss (double at +16 B)
  // partials summed per context in view order, added by vg_finalize_grads
  Buf det_sums;
  double* defer_loss = nullptr;
  float* defer_bg = nullptr;
  Buf vmask;                         // forward -> backward visibility bits (4 rows of P bits)
  Buf seg_state, seg_items;          // segmented backward (SegIO): boundary states, binned items
  bool seg_valid = false;            // the last forward recorded depth statistics (atomic mode)
  bool seg_on = false;               // ... and segmented its backward
  bool seg_next = false;             // decision for the next view (from the last statistics read)
  uint32_t seg_thr = 0;              // its split depth
  unsigned long long* seg_host = nullptr;  // mapped pinned: the last finished forward's decision
  unsigned long long* seg_host_dev = nullptr;
  cudaStream_t side = nullptr;       // deep-tile forward beside the regular launch
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  int last_deep = 0;                 // tiles the last forward ran through the deep variant
  int sm_count = 0;
  int vm_words = 0;
  bool vmask_valid = false;
  unsigned long long* total_host = nullptr;  // {pairs, step-2 span chunks}
  // state of the last prepare
  vg_scene scene{};
  CamK cam{};
  vg_options opt{};
  int64_t pairs = 0;
  int n_tiles = 0;
  uint32_t* vals = nullptr;
  bool prepared = false;
  bool have_fwd = false;
  bool have_counts = false;      // the last forward produced n_contrib / n_active
  bool pending = false;          // vg_prepare_async issued, finish outstanding
  uint32_t* perm_ptr = nullptr;  // depth order of the last prepare
  cudaEvent_t count_ready = nullptr;
  // event profiling (vg_profile)
  bool prof = false;
  std::vector<cudaEvent_t> pool;
  size_t pool_used = 0;
  struct Mark { int kind; cudaEvent_t a, b; };
  std::vector<Mark> marks;
  cudaEvent_t fence[2] = {nullptr, nullptr};   // launch fences (fence_mode)
  unsigned long long* dbg_cta = nullptr;       // vg_debug_cta_log
  int dbg_cta_n = 0;
};

static cudaEvent_t pool_event(vg_context* c) {
  if (c->pool_used == c->pool.size()) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
    c->pool.push_back(e);
  }
  return c->pool[c->pool_used++];
}

// Bracket a launch with events when profiling is on.  VG_FENCE brackets
// launches with timing events outside profiling too ("fences"): with the
// blends of consecutive views serialised on one stream, bracketing both the
// side-stream binning and the blend launches cut config 3 from 149.0 to 139.8
// ms per step (it kept the binning kernels from co-running with the blends in a
// way that slowed the blends more than it hid); with the two alternating blend
// streams of the multi-view step they cost 0.5-5 %, so they are off by
// default.  Bits: 0 = binning launches, 1 = blend launches, 2 = timing-free
// events (no gain).
static int fence_mode(const vg_context*) {
  static int m = -2;
  if (m == -2) {
    const char* e = getenv("VG_FENCE");
    m = e ? atoi(e) : 0;
  }
  return m;
}

struct ProfScope {
  vg_context* c;
  int kind;
  cudaStream_t st;
  cudaEvent_t a = nullptr;
  cudaEvent_t f = nullptr;
  ProfScope(vg_context* c_, int k, cudaStream_t s) : c(c_), kind(k), st(s) {
    if (c->prof) {
      if ((a = pool_event(c))) cudaEventRecord(a, st);
      return;
    }
    const int fm = fence_mode(c);
    const bool blend = k == VG_K_RENDER_FWD || k == VG_K_RENDER_BWD || k == VG_K_FINALIZE ||
                       k == VG_K_TOMO_FWD || k == VG_K_TOMO_BWD;
    if (fm & (blend ? 2 : 1)) {
      const int w = (fm & 4) ? 1 : 0;
      if (!c->fence[w])
        cudaEventCreateWithFlags(&c->fence[w], w ? cudaEventDisableTiming : cudaEventDefault);
      f = c->fence[w];
      cudaEventRecord(f, st);
    }
  }
  ~ProfScope() {
    if (f) {
      cudaEventRecord(f, st);
      return;
    }
    if (!a) return;
    cudaEvent_t b = pool_event(c);
    if (!b) return;
    cudaEventRecord(b, st);
    c->marks.push_back({kind, a, b});
  }
};

#ifdef VG_DEBUG
// Debug builds: every context buffer is allocated with exactly the requested
// size between two 4 KB guard bands, and the whole allocation is poisoned
// with 0xA5 bytes (reads of never-written memory then give NaN-like garbage
// that the parity checks see); vg_debug_guard_check finds writes past
// either end.
constexpr size_t VG_GUARD = 4096;
static int buf_alloc(Buf& b, size_t bytes, cudaStream_t st) {
  char* base = nullptr;
  VG_CUDA(cudaMallocAsync((void**)&base, bytes + 2 * VG_GUARD, st));
  VG_CUDA(cudaMemsetAsync(base, 0xA5, bytes + 2 * VG_GUARD, st));
  b.p = base + VG_GUARD;
  b.bytes = bytes;
  return VG_OK;
}
static void* buf_base(const Buf& b) { return (char*)b.p - VG_GUARD; }
#else
static int buf_alloc(Buf& b, size_t bytes, cudaStream_t st) {
  VG_CUDA(cudaMallocAsync(&b.p, bytes, st));
  b.bytes = bytes;
  return VG_OK;
}
static void* buf_base(const Buf& b) { return b.p; }
#endif

static int ensure(Buf& b, size_t bytes, cudaStream_t st, bool zero = false) {
#ifdef VG_DEBUG
  if (b.bytes == bytes && b.p) return VG_OK;  // exact sizes: the guards sit at the used end
  const size_t want = bytes;
#else
  if (b.bytes >= bytes && b.p) return VG_OK;
  const size_t want = bytes + bytes / 4 + 256;
#endif
  if (b.p) VG_CUDA(cudaFreeAsync(buf_base(b), st));
  { const int _r = buf_alloc(b, want, st); if (_r != VG_OK) return _r; }
  if (zero) VG_CUDA(cudaMemsetAsync(b.p, 0, want, st));
  return VG_OK;
}

#define VG_TRY(x)                 \
  do {                            \
    int _r = (x);                 \
    if (_r != VG_OK) return _r;   \
  } while (0)

extern "C" {

int vg_abi_version(void) { return VG_ABI_VERSION; }

const char* vg_last_error(void) { return g_err.c_str(); }

int vg_create(vg_context** out, int32_t device) {
  if (!out) return fail(VG_EINVAL, "vg_create: out is NULL");
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
    return fail(VG_ECUDA, "vg_create: no CUDA device");
  if (device < 0 || device >= count) return fail(VG_EINVAL, "vg_create: bad device index");
  VG_CUDA(cudaSetDevice(device));
  vg_context* c = new vg_context();
  c->device = device;
  // keep freed stream-ordered allocations cached in the device pool
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t keep = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  if (span_configure() != cudaSuccess) {
    delete c;
    return fail(VG_ECUDA, "vg_create: kernel attribute setup failed");
  }
  if (cudaMallocHost(&c->total_host, 2 * sizeof(unsigned long long)) != cudaSuccess) {
    delete c;
    return fail(VG_ENOMEM, "vg_create: pinned alloc failed");
  }
  if (cudaEventCreateWithFlags(&c->count_ready, cudaEventDisableTiming) != cudaSuccess) {
    cudaFreeHost(c->total_host);
    delete c;
    return fail(VG_ECUDA, "vg_create: event creation failed");
  }
  *out = c;
  return VG_OK;
}

static std::vector<Buf*> all_bufs(vg_context* c) {
  return {&c->rec,  &c->depth, &c->rect, &c->offset, &c->acc,
                &c->vals0, &c->ranges, &c->n_act, &c->tord, &c->span1,
                &c->span2, &c->dkey,  &c->perm,  &c->dsort_tmp, &c->frame, &c->lacc,
                &c->cacc, &c->vmask, &c->dcol, &c->centers, &c->gm, &c->gscratch, &c->det_part, &c->det_cnt, &c->det_off, &c->det_slot,
                &c->det_bg, &c->det_loss, &c->det_scan, &c->tpart, &c->det_gvis4, &c->det_big, &c->det_sums,
                &c->seg_state, &c->seg_items};
}

void vg_destroy(vg_context* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  for (Buf* b : all_bufs(c))
    if (b->p) cudaFree(buf_base(*b));
  if (c->total_host) cudaFreeHost(c->total_host);
  if (c->seg_host) cudaFreeHost(c->seg_host);
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  if (c->side) cudaStreamDestroy(c->side);
  for (cudaEvent_t e : c->pool) cudaEventDestroy(e);
  if (c->count_ready) cudaEventDestroy(c->count_ready);
  for (cudaEvent_t e : c->fence)
    if (e) cudaEventDestroy(e);
  delete c;
}

int64_t vg_launch_count(vg_context* c) { return c ? c->launches : 0; }

int vg_profile(vg_context* c, int32_t enable) {
  if (!c) return fail(VG_EINVAL, "vg_profile: NULL context");
  c->prof = enable != 0;
  if (enable) {
    c->marks.clear();
    c->pool_used = 0;
  }
  return VG_OK;
}

int vg_profile_read(vg_context* c, double* ms, int64_t* counts) {
  if (!c || !ms || !counts) return fail(VG_EINVAL, "vg_profile_read: NULL argument");
  for (int k = 0; k < VG_K_COUNT; ++k) { ms[k] = 0.0; counts[k] = 0; }
  for (const auto& m : c->marks) {
    VG_CUDA(cudaEventSynchronize(m.b));
    float t = 0.f;
    VG_CUDA(cudaEventElapsedTime(&t, m.a, m.b));
    ms[m.kind] += t;
    counts[m.kind] += 1;
  }
  return VG_OK;
}

static int make_cam(const vg_camera* cam, CamK& k) {
  if (!cam) return fail(VG_EINVAL, "camera is NULL");
  if (cam->width <= 0 || cam->height <= 0) return fail(VG_EINVAL, "camera size must be positive");
  if (cam->projection != VG_PINHOLE && cam->projection != VG_PARALLEL)
    return fail(VG_EINVAL, "unknown projection");
  if (cam->projection == VG_PINHOLE && (!(cam->fx > 0) || !(cam->fy > 0)))
    return fail(VG_EINVAL, "focal lengths must be positive");
  if (cam->projection == VG_PARALLEL && !(cam->extent > 0))
    return fail(VG_EINVAL, "parallel detector extent must be positive");
  k.width = cam->width;
  k.height = cam->height;
  k.ntx = (cam->width + TILE - 1) / TILE;
  k.nty = (cam->height + TILE - 1) / TILE;
  k.projection = cam->projection;
  k.fx = cam->fx; k.fy = cam->fy; k.cx = cam->cx; k.cy = cam->cy;
  k.z_near = cam->z_near;
  k.extent = cam->extent;
  for (int i = 0; i < 9; ++i) k.R[i] = cam->rotation[i];
  for (int i = 0; i < 3; ++i) k.t[i] = cam->translation[i];
  for (int j = 0; j < 3; ++j)  // centre = -R^T t
    k.center[j] = -(k.R[0 * 3 + j] * k.t[0] + k.R[1 * 3 + j] * k.t[1] + k.R[2 * 3 + j] * k.t[2]);
  return VG_OK;
}

int vg_prepare_async(vg_context* c, const vg_scene* s, const vg_camera* cam,
                     const vg_options* opt, void* stream) {
  if (!c || !s || !opt) return fail(VG_EINVAL, "vg_prepare: NULL argument");
  if (opt->tile_size != TILE) return fail(VG_EINVAL, "only tile_size=16 is supported");
  if (opt->sort_by != VG_SORT_DEPTH && opt->sort_by != VG_SORT_GAMMA)
    return fail(VG_EINVAL, "unknown sort key");
  if (opt->mode != VG_MODE_ANALYTIC && opt->mode != VG_MODE_SPLAT)
    return fail(VG_EINVAL, "unknown mode");
  if (opt->mode == VG_MODE_SPLAT && s && s->n > 0 && !s->splat_opacities)
    return fail(VG_EINVAL, "mode splat needs scene.splat_opacities");
  if (opt->mode == VG_MODE_SPLAT && cam && cam->projection != VG_PINHOLE)
    return fail(VG_EINVAL, "mode splat needs a pinhole camera");
  if (opt->sort_by == VG_SORT_GAMMA && cam && cam->projection != VG_PINHOLE)
    return fail(VG_EINVAL, "sort_by gamma needs a pinhole camera");
  if (s->n < 0) return fail(VG_EINVAL, "negative primitive count");
  if (s->n > 0x7fffffff) return fail(VG_EINVAL, "too many primitives (> 2^31-1)");
  if (s->n > 0 && (!s->means || !s->scales || !s->rotations || !s->thetas))
    return fail(VG_EINVAL, "scene arrays must be non-NULL");
  CamK k;
  VG_TRY(make_cam(cam, k));
  cudaStream_t st = (cudaStream_t)stream;
  VG_CUDA(cudaSetDevice(c->device));
  const int64_t n = s->n;
  if (n != c->scene.n) c->sh_views = 0;  // pending SH slabs belong to another scene
  c->scene = *s;
  c->cam = k;
  c->opt = *opt;
  c->n_tiles = k.ntx * k.nty;
  c->prepared = false;
  c->have_fwd = false;
  c->det_ready = false;
  c->det_slots_ready = false;
  const int64_t npix = (int64_t)k.width * k.height;
  VG_TRY(ensure(c->ranges, sizeof(uint2) * (size_t)c->n_tiles, st));
  VG_TRY(ensure(c->n_act, sizeof(int) * (size_t)npix, st));
  if (k.ntx > span_max_buckets() || k.nty > span_max_buckets())
    return fail(VG_EINVAL, "image too large: at most 1024 tile rows and columns (16384 px)");
  VG_CUDA(cudaMemsetAsync(c->ranges.p, 0, sizeof(uint2) * (size_t)c->n_tiles, st));
  c->pairs = 0;
  if (n > 0) {
    size_t accb = sizeof(float) * 16 * (size_t)n;
    bool grow_acc = c->acc.bytes < accb;
    VG_TRY(ensure(c->rec, sizeof(GRec) * (size_t)n, st));
    VG_TRY(ensure(c->depth, sizeof(float) * (size_t)n, st));
    VG_TRY(ensure(c->rect, sizeof(ushort4) * (size_t)n, st));
    VG_TRY(ensure(c->offset, sizeof(uint32_t) * (size_t)n, st));
    VG_TRY(ensure(c->dkey, sizeof(uint32_t) * (size_t)n, st));
    VG_TRY(ensure(c->perm, sizeof(uint32_t) * 2 * (size_t)n, st));
    if (grow_acc) VG_TRY(ensure(c->acc, accb, st, true));
    if (c->lacc.bytes < sizeof(float) * 12 * (size_t)n)
      VG_TRY(ensure(c->lacc, sizeof(float) * 12 * (size_t)n, st, true));
    VG_TRY(ensure(c->frame, sizeof(float) * 12 * (size_t)n, st));
    {
      const size_t cb = sizeof(float) * 3 * (size_t)n;
      if (c->cacc.bytes < cb) VG_TRY(ensure(c->cacc, cb, st, true));
    }
    double* gm = nullptr;
    if (opt->sort_by == VG_SORT_GAMMA) {
      VG_TRY(ensure(c->gm, sizeof(double) * 9 * (size_t)n, st));
      gm = (double*)c->gm.p;
    }
    {
      ProfScope ps(c, VG_K_PREPROCESS, st);
      launch_preprocess(n, *s, k, opt->bin_cut, (GRec*)c->rec.p, (float*)c->depth.p,
                        (ushort4*)c->rect.p, (float*)c->frame.p, gm, opt->mode == VG_MODE_SPLAT,
                        st);
    }
    VG_LAUNCHED(c, 1);
    // Gaussians in (float32 depth, index) order: hand-written radix sort of
    // the depth bits over the identity permutation (stable => index order)
    uint32_t* ids0 = (uint32_t*)c->perm.p + n;
    uint32_t* ids1 = (uint32_t*)c->perm.p;
    uint32_t* perm = ids1;
    {
      ProfScope ps(c, VG_K_SORT, st);
      VG_TRY(ensure(c->dsort_tmp, radix_temp_bytes(n, 32), st));
      int which = 0, nl = 0;
      VG_CUDA(radix_sort_u32(c->dsort_tmp.p, c->dsort_tmp.bytes, (uint32_t*)c->depth.p,
                             (uint32_t*)c->dkey.p, ids0, ids1, n, 32, &which, &nl, st,
                             /*identity_values=*/true));
      c->launches += nl;
      perm = which ? ids1 : ids0;
    }
    c->perm_ptr = perm;
    // step 1 of the span binning up to the pair count (vg_span.cu)
    VG_TRY(ensure(c->span1, span_scratch1_bytes(n, k.nty), st));
    {
      ProfScope ps(c, VG_K_SCAN, st);
      int nl = 0;
      VG_CUDA(span_rows_begin(n, perm, (const ushort4*)c->rect.p, k.nty, c->span1.p, &nl, st));
      VG_LAUNCHED(c, nl);
    }
    VG_CUDA(cudaMemcpyAsync(c->total_host, span_info(c->span1.p), 2 * sizeof(unsigned long long),
                            cudaMemcpyDeviceToHost, st));
    VG_CUDA(cudaEventRecord(c->count_ready, st));
  }
  c->pending = true;
  return VG_OK;
}

int vg_prepare_finish(vg_context* c, void* stream) {
  if (!c) return fail(VG_EINVAL, "vg_prepare_finish: NULL context");
  if (!c->pending) return fail(VG_EINVAL, "vg_prepare_finish: no vg_prepare_async pending");
  c->pending = false;
  cudaStream_t st = (cudaStream_t)stream;
  VG_CUDA(cudaSetDevice(c->device));
  const int64_t n = c->scene.n;
  const CamK& k = c->cam;
  c->pairs = 0;
  int64_t chunks2 = 0;
  if (n > 0) {
    // the only host synchronisation of the pipeline: the pair count sizes the lists
    VG_CUDA(cudaEventSynchronize(c->count_ready));
    const unsigned long long P = c->total_host[0];
    if (P > 0x7fffffffull) return fail(VG_EINVAL, "tile-pair count exceeds 2^31");
    c->pairs = (int64_t)P;
    chunks2 = (int64_t)c->total_host[1];
  }
  const int64_t P = c->pairs;
  const int nt = c->n_tiles;
  VG_TRY(ensure(c->tord, sizeof(uint32_t) * (size_t)nt, st));
  VG_TRY(ensure(c->span2, span_scratch2_bytes(chunks2, k.ntx, nt), st));
  if (P > 0) VG_TRY(ensure(c->vals0, sizeof(uint32_t) * (size_t)P, st));
  {
    // step 2: row spans -> per-tile lists, tile ranges, heavy-tiles-first order
    ProfScope ps(c, VG_K_DUPLICATE, st);
    int nl = 0;
    VG_CUDA(span_finish(n, c->perm_ptr, (const ushort4*)c->rect.p, k.ntx, k.nty, c->span1.p,
                        P > 0 ? chunks2 : 0, c->span2.p, (uint2*)c->ranges.p,
                        (uint32_t*)c->tord.p, (uint32_t*)c->vals0.p, &nl, st));
    VG_LAUNCHED(c, nl);
  }
  c->vals = P > 0 ? (uint32_t*)c->vals0.p : nullptr;
  if (c->opt.sort_by == VG_SORT_GAMMA && P > 1) {
    VG_TRY(ensure(c->gscratch, gamma_scratch_bytes(P), st));
    ProfScope ps(c, VG_K_SORT, st);
    launch_gamma_sort(nt, (const uint2*)c->ranges.p, c->vals, (const double*)c->gm.p, P,
                      c->gscratch.p, k, st);
    VG_LAUNCHED(c, 1);
  }
  c->prepared = true;
  return VG_OK;
}

int vg_prepare(vg_context* c, const vg_scene* s, const vg_camera* cam, const vg_options* opt,
               void* stream) {
  VG_TRY(vg_prepare_async(c, s, cam, opt, stream));
  return vg_prepare_finish(c, stream);
}

int vg_set_options(vg_context* c, const vg_options* opt) {
  if (!c || !opt) return fail(VG_EINVAL, "vg_set_options: NULL argument");
  if (opt->alpha_cut != c->opt.alpha_cut) c->vmask_valid = false;
  c->opt.early_stop = opt->early_stop;
  c->opt.alpha_cut = opt->alpha_cut;
  c->opt.alpha_clamp = opt->alpha_clamp;
  c->opt.deterministic = opt->deterministic;
  return VG_OK;
}

int vg_pair_count(vg_context* c, int64_t* out) {
  if (!c || !out) return fail(VG_EINVAL, "vg_pair_count: NULL argument");
  if (!c->prepared) return fail(VG_EINVAL, "vg_pair_count: call vg_prepare first");
  *out = c->pairs;
  return VG_OK;
}

__global__ void k_tile_lists(int64_t P, const uint32_t* vals,
                             const uint2* ranges, int n_tiles, int32_t* prims, int32_t* offsets) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < P) prims[i] = (int32_t)vals[i];
  if (i <= n_tiles) {
    // offsets[t] = start of tile t; empty tiles take the next non-empty start
    if (i == n_tiles) {
      offsets[i] = (int32_t)P;
    } else {
      uint2 r = ranges[i];
      if (r.y > r.x) {
        offsets[i] = (int32_t)r.x;
      } else {
        int64_t t = i + 1;
        uint32_t nxt = (uint32_t)P;
        while (t < n_tiles) {
          uint2 q = ranges[t];
          if (q.y > q.x) { nxt = q.x; break; }
          ++t;
        }
        offsets[i] = (int32_t)nxt;
      }
    }
  }
}

int vg_tile_lists(vg_context* c, int32_t* prims, int32_t* offsets, void* stream) {
  if (!c || !offsets) return fail(VG_EINVAL, "vg_tile_lists: NULL argument");
  if (!c->prepared) return fail(VG_EINVAL, "vg_tile_lists: call vg_prepare first");
  if (c->pairs > 0 && !prims) return fail(VG_EINVAL, "vg_tile_lists: prims is NULL");
  cudaStream_t st = (cudaStream_t)stream;
  int64_t work = c->pairs > c->n_tiles + 1 ? c->pairs : c->n_tiles + 1;
  k_tile_lists<<<(unsigned)((work + 255) / 256), 256, 0, st>>>(
      c->pairs, c->vals, (const uint2*)c->ranges.p, c->n_tiles, prims, offsets);
  VG_LAUNCHED(c, 1);
  return VG_OK;
}

// VG_SEG_BWD=0 turns the segmented backward off (one CTA per tile in list-length order)
static bool seg_enabled() {
  static int m = -1;
  if (m < 0) {
    const char* e = getenv("VG_SEG_BWD");
    m = e ? atoi(e) != 0 : 1;
  }
  return m != 0;
}

// VG_SEG_RATIO: segment a view when its deepest tile exceeds this multiple of
// the per-slot share of its work (default 1)
static float seg_ratio() {
  static float r = -1.f;
  if (r < 0.f) {
    const char* e = getenv("VG_SEG_RATIO");
    r = e ? (float)atof(e) : 1.f;
    if (!(r > 0.f)) r = 1.f;
  }
  return r;
}

// the segmented backward's buffers of the last forward (the bin counters
// follow the visibility mask, 16-byte aligned, and are cleared with it)
static SegIO seg_io(vg_context* c) {
  SegIO s;
  s.counts = (uint32_t*)((char*)c->vmask.p + ((sizeof(uint32_t) * 4 * (size_t)c->vm_words + 15) & ~(size_t)15));
  s.decision = c->seg_host_dev;
  s.slots = (uint32_t)(c->sm_count * VG_BWD_MINB);
  s.ratio = seg_ratio();
  s.on = c->seg_on;
  if (!s.on) return s;
  s.state = (float4*)c->seg_state.p;
  s.items = (uint2*)c->seg_items.p;
  s.budget = 2u * (uint32_t)(c->sm_count * VG_BWD_MINB);
  s.n_tiles = (uint32_t)c->n_tiles;
  s.cap = s.n_tiles + s.budget;
  s.thr = c->seg_thr;
  return s;
}

// This forward's segmentation: the decision the last finished forward on
// this context left in mapped host memory (a stale one while the device runs
// behind the host -- a heuristic either way).
// VG_DEEP_TILES: tiles the deep-tile forward takes (default: 2 per SM; 0: off).
// Config 4 step with the 63-register regular forward: 148: 30.9 ms, 222-370:
// 30.6, 444: 30.8, 592: 31.0, 888: 31.7 (with the 48-register one 4 per SM was best)
static int deep_tiles(const vg_context* c) {
  static int k = -2;
  if (k == -2) {
    const char* e = getenv("VG_DEEP_TILES");
    k = e ? std::max(0, atoi(e)) : -1;
  }
  return k < 0 ? 2 * c->sm_count : k;
}

// the context's side stream (highest priority) and fork / join events
static int side_stream(vg_context* c) {
  if (c->side) return VG_OK;
  int lo = 0, hi = 0;
  VG_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  VG_CUDA(cudaStreamCreateWithPriority(&c->side, cudaStreamNonBlocking, hi));
  VG_CUDA(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
  VG_CUDA(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
  return VG_OK;
}

static int seg_decide(vg_context* c) {
  if (!c->sm_count) {
    VG_CUDA(cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, c->device));
    if (c->sm_count < 1) c->sm_count = 1;
  }
  if (!c->seg_host) {
    if (cudaHostAlloc((void**)&c->seg_host, 64, cudaHostAllocMapped) != cudaSuccess)
      return fail(VG_ENOMEM, "segmented backward: mapped pinned alloc failed");
    *(volatile unsigned long long*)c->seg_host = 0ull;
    VG_CUDA(cudaHostGetDevicePointer((void**)&c->seg_host_dev, c->seg_host, 0));
  }
  const unsigned long long d = *(volatile unsigned long long*)c->seg_host;
  c->seg_next = (d & 1ull) != 0;
  c->seg_thr = (uint32_t)(d >> 32);
  return VG_OK;
}

static BlendParams blend_params(const vg_context* c) {
  BlendParams p;
  p.dbg_n = c->scene.n;
  p.dbg_pairs = c->pairs;
#ifdef VG_DEBUG
  if (const char* j = getenv("VG_DEBUG_JITTER")) p.dbg_jitter = (unsigned)atoi(j);
#endif
  p.width = c->cam.width;
  p.height = c->cam.height;
  p.ntx = c->cam.ntx;
  p.cx = (float)c->cam.cx;
  p.cy = (float)c->cam.cy;
  p.fx = (float)(c->cam.fx > 0 ? c->cam.fx : 1.0);
  p.fy = (float)(c->cam.fy > 0 ? c->cam.fy : 1.0);
  // An entry is active iff T_before >= early_stop (raster.py:384-385).  The
  // comparison carries a 2^-20 relative slack: products of exactly clamped
  // alphas, e.g. (1 - 0.99)^2 = 1.0000000000000018e-4 in float64, land just
  // above 1e-4 in the reference but just below it in float32 (0.99 is not
  // representable), which would systematically drop the next layer.
  p.stop = (float)(c->opt.early_stop * (1.0 - 9.5367431640625e-07));
  p.cut = (float)c->opt.alpha_cut;
  p.clamp = (float)c->opt.alpha_clamp;
  p.cc = (float)(1.0 - c->opt.alpha_clamp);
  // alpha_raw = 1 - exp(-e) < cut  <=>  e log2(e) < -log1p(-cut) log2(e):
  // cut entries get the factor 1 (eval_pinhole2), every other factor is
  // exp(-e) < 1 in float32 for cut >= 6e-8, so "cut" is om > nextafter(1, 0)
  p.omcut = 0.99999994f;
  p.e2cut = (float)(-log1p(-c->opt.alpha_cut) * 1.4426950408889634);
  p.ecut = c->opt.alpha_cut > 0 ? (float)(-log1p(-c->opt.alpha_cut) * (1.0 - 1e-3)) : 0.f;
  for (int i = 0; i < 3; ++i) p.bg[i] = (float)c->scene.background[i];
  p.dbg_cta = c->dbg_cta;
  p.dbg_cta_n = c->dbg_cta_n;
  return p;
}

int vg_render_forward(vg_context* c, float* color, float* final_t, int32_t* n_contrib,
                      void* stream) {
  if (!c || !color || !final_t) return fail(VG_EINVAL, "vg_render_forward: NULL argument");
  if (!c->prepared) return fail(VG_EINVAL, "vg_render_forward: call vg_prepare first");
  if (c->cam.projection != VG_PINHOLE) return fail(VG_EINVAL, "render needs a pinhole camera");
  cudaStream_t st = (cudaStream_t)stream;
  BlendParams p = blend_params(c);
  // with alpha_cut > 0, "live => not cut => visible": the forward records
  // which (entry, warp block) pairs had a visible pixel and the backward
  // walks exactly those
  const bool use_vm = c->opt.alpha_cut > 0 && c->pairs > 0 && c->opt.mode != VG_MODE_SPLAT;
  uint32_t* vm = nullptr;
  SegIO seg;
  // depth statistics in both modes; a tail-bound view (the previous view's
  // decision) gets the deep-tile forward, and in atomic mode the segmented backward
  c->seg_valid = use_vm && seg_enabled();
  c->seg_on = false;
  bool tail = false;
  if (c->seg_valid) {
    VG_TRY(seg_decide(c));
    tail = c->seg_next;
    c->seg_on = tail && !c->opt.deterministic;
  }
  if (use_vm) {
    c->vm_words = (int)((c->pairs + 31) / 32) + 1;
    // the visibility rows, then the segmented backward's bin counters
    const size_t bytes = ((sizeof(uint32_t) * 4 * (size_t)c->vm_words + 15) & ~(size_t)15) +
                         SEG_COUNT_BYTES;
    VG_TRY(ensure(c->vmask, bytes, st));
    VG_CUDA(cudaMemsetAsync(c->vmask.p, 0, bytes, st));
    vm = (uint32_t*)c->vmask.p;
    if (c->seg_on) {
      VG_TRY(ensure(c->seg_state, seg_state_bytes(c->pairs), st));
      VG_TRY(ensure(c->seg_items, sizeof(uint2) * SEG_BINS *
                                      ((size_t)c->n_tiles + 2 * (size_t)c->sm_count * VG_BWD_MINB), st));
    }
    if (c->seg_valid) seg = seg_io(c);
  }
  c->vmask_valid = use_vm;
  c->last_deep = 0;
  {
    ProfScope ps(c, VG_K_RENDER_FWD, st);
    if (c->opt.mode == VG_MODE_SPLAT) {
      launch_splat_fwd(c->n_tiles, (const GRec*)c->rec.p, c->vals, (const uint2*)c->ranges.p,
                       (const uint32_t*)c->tord.p, p, color, final_t, n_contrib,
                       n_contrib ? (int*)c->n_act.p : nullptr, st);
      VG_LAUNCHED(c, 1);
    } else {
      // the training forward of a tail-bound view: the deepest (longest-list)
      // tiles through the latency-bound variant on a side stream, beside the
      // regular launch over the others
      const int deep = tail && !n_contrib ? std::min(c->n_tiles, deep_tiles(c)) : 0;
      if (deep > 0) {
        VG_TRY(side_stream(c));
        VG_CUDA(cudaEventRecord(c->ev_fork, st));
        VG_CUDA(cudaStreamWaitEvent(c->side, c->ev_fork, 0));
        BlendParams pd = p;
        if (pd.dbg_cta) {  // profiling log: the deep CTAs after the regular ones
          pd.dbg_cta += (size_t)VG_CTA_LOG_STRIDE * (size_t)(c->n_tiles - deep);
          pd.dbg_cta_n = std::max(0, pd.dbg_cta_n - (c->n_tiles - deep));
        }
        launch_render_fwd_deep(deep, (const GRec*)c->rec.p, c->vals, (const uint2*)c->ranges.p,
                               (const uint32_t*)c->tord.p, pd, c->opt.early_stop > 0,
                               c->opt.alpha_cut > 0, color, final_t, vm, c->vm_words, c->side, seg);
        VG_LAUNCHED(c, 1);
      }
      if (c->n_tiles > deep) {
        launch_render_fwd(c->n_tiles - deep, (const GRec*)c->rec.p, c->vals, (const uint2*)c->ranges.p,
                          (const uint32_t*)c->tord.p + deep, p,
                          c->opt.early_stop > 0, c->opt.alpha_cut > 0, color, final_t, n_contrib,
                          (int*)c->n_act.p, vm, c->vm_words, st, seg);
        VG_LAUNCHED(c, 1);
      }
      if (deep > 0) {
        VG_CUDA(cudaEventRecord(c->ev_join, c->side));
        VG_CUDA(cudaStreamWaitEvent(st, c->ev_join, 0));
      }
      c->last_deep = deep;
    }
  }
  c->have_fwd = true;
  c->have_counts = n_contrib != nullptr;
  return VG_OK;
}

// Debug (not in the public header): forward-pass culling statistics.
int vg_debug_forward_stats(vg_context* c, float* color, float* final_t, int32_t* n_contrib,
                           unsigned long long* out4, void* stream) {
  if (!c || !c->prepared) return fail(VG_EINVAL, "vg_debug_forward_stats: not prepared");
  BlendParams p = blend_params(c);
  int e = debug_forward_stats(c->n_tiles, (const GRec*)c->rec.p, c->vals, (const uint2*)c->ranges.p,
                              (const uint32_t*)c->tord.p, p, color, final_t, n_contrib,
                              (int*)c->n_act.p, out4, (cudaStream_t)stream);
  return e ? fail(VG_ECUDA, "debug stats launch failed") : VG_OK;
}

// Diagnostic CTA log (volgauss_b200.h).
int vg_debug_cta_log(vg_context* c, unsigned long long* log, int n) {
  if (!c) return fail(VG_EINVAL, "vg_debug_cta_log: NULL context");
  if (!VG_CTA_LOG && log) return fail(VG_EINVAL, "vg_debug_cta_log: needs the profiling build (-DVG_CTA_LOG=1)");
  c->dbg_cta = log;
  c->dbg_cta_n = log ? n : 0;
  return VG_OK;
}

int vg_debug_segments(vg_context* c, int64_t* items, int32_t* segmented) {
  if (!c || !items || !segmented) return fail(VG_EINVAL, "vg_debug_segments: NULL argument");
  *items = 0;
  *segmented = 0;
  if (!c->have_fwd) return VG_OK;
  *segmented = c->last_deep > 0 ? 2 : 0;
  if (!c->seg_on) return VG_OK;
  uint32_t h[SEG_BINS];
  VG_CUDA(cudaDeviceSynchronize());
  VG_CUDA(cudaMemcpy(h, seg_io(c).counts, sizeof(h), cudaMemcpyDeviceToHost));
  *segmented |= 1;
  for (int b = 0; b < SEG_BINS; ++b) *items += h[b];
  return VG_OK;
}

int vg_n_active(vg_context* c, int32_t* out, void* stream) {
  if (!c || !out) return fail(VG_EINVAL, "vg_n_active: NULL argument");
  if (!c->have_fwd || !c->have_counts)
    return fail(VG_EINVAL, "vg_n_active: no counting forward (n_contrib != NULL) on this context");
  size_t bytes = sizeof(int32_t) * (size_t)c->cam.width * (size_t)c->cam.height;
  VG_CUDA(cudaMemcpyAsync(out, c->n_act.p, bytes, cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
  return VG_OK;
}

int vg_visible_pairs(vg_context* c, int64_t* out) {
  if (!c || !out) return fail(VG_EINVAL, "vg_visible_pairs: NULL argument");
  *out = 0;
  if (!c->have_fwd || !c->vmask_valid) return VG_OK;
  std::vector<uint32_t> h(4 * (size_t)c->vm_words);
  VG_CUDA(cudaMemcpy(h.data(), c->vmask.p, sizeof(uint32_t) * h.size(), cudaMemcpyDeviceToHost));
  int64_t n = 0;
  for (uint32_t w : h) n += __builtin_popcount(w);
  *out = n;
  return VG_OK;
}

static int prep_grads(vg_context* c, vg_grads* g, cudaStream_t st) {
  if (!g) return fail(VG_EINVAL, "grads is NULL");
  if (g->accumulate < VG_OVERWRITE || g->accumulate > VG_DEFER)
    return fail(VG_EINVAL, "grads.accumulate must be VG_OVERWRITE, VG_ADD or VG_DEFER");
  if (g->accumulate == VG_OVERWRITE) {
    const size_t n = (size_t)c->scene.n;
    if (g->d_background) VG_CUDA(cudaMemsetAsync(g->d_background, 0, 3 * sizeof(float), st));
    if (g->visible && n) VG_CUDA(cudaMemsetAsync(g->visible, 0, n, st));
  }
  return VG_OK;
}

// After a backward blend: rotate this view's accumulators into the
// view-independent ones (and add colour / SH gradients), then -- unless the
// caller defers -- run the float64 parameter chain.
// Grow a buffer to at least `bytes`, keeping its contents (stream ordered).
static int grow_keep(Buf& b, size_t bytes, cudaStream_t st) {
  if (b.bytes >= bytes && b.p) return VG_OK;
#ifdef VG_DEBUG
  const size_t want = bytes;
#else
  const size_t want = bytes * 2 + 256;
#endif
  Buf nb;
  VG_TRY(buf_alloc(nb, want, st));
  if (b.p) {
    VG_CUDA(cudaMemcpyAsync(nb.p, b.p, b.bytes, cudaMemcpyDeviceToDevice, st));
    VG_CUDA(cudaFreeAsync(buf_base(b), st));
  }
  b = nb;
  return VG_OK;
}

static int run_param_chain(vg_context* c, const vg_grads& g, cudaStream_t st) {
  int k = 0;
  {
    ProfScope ps(c, VG_K_FINALIZE, st);
    k = launch_finalize_params(c->scene.n, c->scene, (float*)c->lacc.p, (float*)c->cacc.p,
                               (const float*)c->dcol.p, (const double*)c->centers.p, c->sh_views,
                               g, c->opt.mode == VG_MODE_SPLAT, st);
  }
  c->sh_views = 0;
  VG_LAUNCHED(c, k);
  return VG_OK;
}

// publish: the render backward of an atomic-mode view that recorded depth
// statistics (the next view's segmentation decision, seg_publish)
static int finish_view(vg_context* c, vg_grads* g, cudaStream_t st, bool publish = false) {
  const int64_t n = c->scene.n;
  if (n <= 0) return VG_OK;
  float* dcol = nullptr;
  double* center = nullptr;
  if (c->scene.sh) {
    const int v = c->sh_views;
    VG_TRY(grow_keep(c->dcol, sizeof(float) * 3 * (size_t)n * (size_t)(v + 1), st));
    VG_TRY(grow_keep(c->centers, sizeof(double) * 3 * (size_t)(v + 1), st));
    dcol = (float*)c->dcol.p + (size_t)v * 3 * (size_t)n;
    center = (double*)c->centers.p + 3 * v;
    c->sh_views = v + 1;
  }
  {
    ProfScope ps(c, VG_K_FINALIZE, st);
    const SegIO seg = publish ? seg_io(c) : SegIO();
    launch_view_accumulate(n, c->scene, c->cam, (const float*)c->frame.p, (float*)c->acc.p,
                           (float*)c->lacc.p, (float*)c->cacc.p, dcol, center,
                           c->opt.mode == VG_MODE_SPLAT, st, publish ? &seg : nullptr);
  }
  VG_LAUNCHED(c, 1);
  if (g->accumulate != VG_DEFER) VG_TRY(run_param_chain(c, *g, st));
  return VG_OK;
}

int vg_merge_deferred(vg_context* dst, vg_context* src, void* stream) {
  if (!dst || !src) return fail(VG_EINVAL, "vg_merge_deferred: NULL context");
  if (dst == src) return VG_OK;
  if (!dst->prepared || !src->prepared) return fail(VG_EINVAL, "vg_merge_deferred: no scene on a context");
  if (dst->scene.n != src->scene.n || (dst->scene.sh == nullptr) != (src->scene.sh == nullptr))
    return fail(VG_EINVAL, "vg_merge_deferred: contexts hold different scenes");
  if (dst->device != src->device) return fail(VG_EINVAL, "vg_merge_deferred: contexts on different devices");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t n = dst->scene.n;
  if (n <= 0) return VG_OK;
  VG_CUDA(cudaSetDevice(dst->device));
  if (src->lacc.p && dst->lacc.p) launch_merge_acc(12 * n, (float*)dst->lacc.p, (float*)src->lacc.p, st);
  if (src->cacc.p && dst->cacc.p) launch_merge_acc(3 * n, (float*)dst->cacc.p, (float*)src->cacc.p, st);
  if (dst->scene.sh && src->sh_views > 0) {
    const int v0 = dst->sh_views, v1 = src->sh_views;
    VG_TRY(grow_keep(dst->dcol, sizeof(float) * 3 * (size_t)n * (size_t)(v0 + v1), st));
    VG_TRY(grow_keep(dst->centers, sizeof(double) * 3 * (size_t)(v0 + v1), st));
    VG_CUDA(cudaMemcpyAsync((float*)dst->dcol.p + (size_t)v0 * 3 * (size_t)n, src->dcol.p,
                            sizeof(float) * 3 * (size_t)n * (size_t)v1, cudaMemcpyDeviceToDevice, st));
    VG_CUDA(cudaMemcpyAsync((double*)dst->centers.p + 3 * (size_t)v0, src->centers.p,
                            sizeof(double) * 3 * (size_t)v1, cudaMemcpyDeviceToDevice, st));
    dst->sh_views = v0 + v1;
    src->sh_views = 0;
  }
  if (src->det_sums.p && (src->defer_bg || src->defer_loss)) {
    if (!dst->det_sums.p) VG_TRY(ensure(dst->det_sums, 64, st, true));
    launch_det_flush((float*)src->det_sums.p, (double*)((char*)src->det_sums.p + 16),
                     src->defer_bg ? (float*)dst->det_sums.p : nullptr,
                     src->defer_loss ? (double*)((char*)dst->det_sums.p + 16) : nullptr, st);
    if (src->defer_bg) dst->defer_bg = src->defer_bg;
    if (src->defer_loss) dst->defer_loss = src->defer_loss;
    src->defer_bg = nullptr;
    src->defer_loss = nullptr;
  }
  VG_LAUNCHED(dst, 2);
  return cudaGetLastError() == cudaSuccess ? VG_OK : fail(VG_ECUDA, "vg_merge_deferred: launch failed");
}

int vg_finalize_grads(vg_context* c, vg_grads* g, void* stream) {
  if (!c || !g) return fail(VG_EINVAL, "vg_finalize_grads: NULL argument");
  if (!c->prepared) return fail(VG_EINVAL, "vg_finalize_grads: no scene on this context");
  vg_grads gg = *g;
  gg.accumulate = g->accumulate == VG_OVERWRITE ? VG_OVERWRITE : VG_ADD;
  cudaStream_t st = (cudaStream_t)stream;
  if (c->scene.n > 0) VG_TRY(run_param_chain(c, gg, st));
  if (c->det_sums.p && (c->defer_bg || c->defer_loss)) {
    // the deterministic mode's deferred d_background / loss sums
    launch_det_flush((float*)c->det_sums.p, (double*)((char*)c->det_sums.p + 16), c->defer_bg,
                     c->defer_loss, st);
    VG_LAUNCHED(c, 1);
    c->defer_bg = nullptr;
    c->defer_loss = nullptr;
  }
  return VG_OK;
}

// Deterministic mode: the per-Gaussian tile counts / offsets of the current
// lists (once per prepare; plus the pair-major slot map unless `gmajor`), the
// slot array for one backward, and zeroed per-tile partials.  gmajor (render
// backward with a forward visibility mask): Gaussian-major slots, their warp
// bytes cleared (entries past a tile's early stop are never staged, so their
// bytes must read as "no warp visible").  Without list entries there are no
// slots, but the per-tile d_background / loss partials still take the
// fixed-order route (the blend selects it on det_part).
static int det_setup(vg_context* c, float*& part, float*& bg, double*& loss, cudaStream_t st,
                     BwdIO* gmajor = nullptr) {
  const int64_t n = c->scene.n, P = c->pairs;
  if (n > 0 && P > 0) {
    const bool need_slots = gmajor == nullptr;
    if (!c->det_ready || (need_slots && !c->det_slots_ready)) {
      VG_TRY(ensure(c->det_cnt, sizeof(uint32_t) * (size_t)n, st));
      VG_TRY(ensure(c->det_off, sizeof(uint32_t) * ((size_t)n + 1), st));
      VG_TRY(ensure(c->det_scan, scan_u32_scratch_bytes(n) + 16, st));
      if (need_slots) VG_TRY(ensure(c->det_slot, sizeof(uint32_t) * (size_t)P, st));
      VG_CUDA(det_prepare(n, (const ushort4*)c->rect.p, (const uint2*)c->ranges.p, c->vals,
                          c->n_tiles, c->cam.ntx, (uint32_t*)c->det_cnt.p, (uint32_t*)c->det_off.p,
                          need_slots ? (uint32_t*)c->det_slot.p : nullptr, c->det_scan.p,
                          (uint32_t*)c->det_off.p + n, st));
      c->det_ready = true;
      c->det_slots_ready = c->det_slots_ready || need_slots;
    }
    VG_TRY(ensure(c->det_part, det_part_bytes(P), st));
    if (gmajor) {
      VG_TRY(ensure(c->det_gvis4, (size_t)P, st));
      VG_TRY(ensure(c->det_big, sizeof(uint32_t) * ((size_t)n + 1), st));
      VG_CUDA(cudaMemsetAsync(c->det_gvis4.p, 0, (size_t)P, st));
      gmajor->det_off = (const uint32_t*)c->det_off.p;
      gmajor->det_rect = (const ushort4*)c->rect.p;
      gmajor->det_gvis4 = (uint8_t*)c->det_gvis4.p;
    } else {
      VG_CUDA(cudaMemsetAsync(c->det_part.p, 0, det_part_bytes(P), st));
    }
  } else {
    VG_TRY(ensure(c->det_part, 64, st));
  }
  VG_TRY(ensure(c->det_bg, sizeof(float) * 3 * (size_t)c->n_tiles, st));
  VG_TRY(ensure(c->det_loss, sizeof(double) * (size_t)c->n_tiles, st));
  VG_CUDA(cudaMemsetAsync(c->det_bg.p, 0, sizeof(float) * 3 * (size_t)c->n_tiles, st));
  part = (float*)c->det_part.p;
  bg = (float*)c->det_bg.p;
  loss = (double*)c->det_loss.p;
  return VG_OK;
}

// Deterministic mode: where the per-view tile-order d_background / loss sums
// go.  Deferred backward calls add them into the context's own sums (summed in
// view order; vg_merge_deferred / vg_finalize_grads add the contexts in a
// fixed order), so the views of different contexts may run concurrently.
static int det_targets(vg_context* c, const vg_grads* g, double* loss_sum, float*& bg,
                       double*& loss, cudaStream_t st) {
  bg = g->d_background;
  loss = loss_sum;
  if (g->accumulate != VG_DEFER) return VG_OK;
  if (!c->det_sums.p) VG_TRY(ensure(c->det_sums, 64, st, true));
  if (bg) {
    c->defer_bg = bg;
    bg = (float*)c->det_sums.p;
  }
  if (loss) {
    c->defer_loss = loss;
    loss = (double*)((char*)c->det_sums.p + 16);
  }
  return VG_OK;
}

static int render_bwd_common(vg_context* c, const float* color, const float* final_t,
                             const float* d_color, const float* d_t, const float* target,
                             double* loss_sum, vg_grads* g, void* stream) {
  if (!c || !color || !final_t) return fail(VG_EINVAL, "vg_render_backward: NULL argument");
  if (!c->prepared || !c->have_fwd)
    return fail(VG_EINVAL, "vg_render_backward: run vg_render_forward on this context first");
  cudaStream_t st = (cudaStream_t)stream;
  VG_TRY(prep_grads(c, g, st));
  BlendParams p = blend_params(c);
  BwdIO io;
  io.color = color;
  io.final_t = final_t;
  io.d_color = d_color;
  io.d_t = d_t;
  io.target = target;
  io.loss_scale = (float)(2.0 / (3.0 * (double)c->cam.width * (double)c->cam.height));
  io.loss_sum = loss_sum;
  io.acc = (float*)c->acc.p;
  io.visible = g->visible;
  io.d_background = g->d_background;
  if (!io.visible) {
    // visibility is always tracked; route it to scratch when not requested
    VG_TRY(ensure(c->offset, sizeof(uint32_t) * (size_t)(c->scene.n > 0 ? c->scene.n : 1), st));
    io.visible = (uint8_t*)c->offset.p;
  }
  const bool det = c->opt.deterministic != 0;
  const bool vm = c->vmask_valid && c->opt.alpha_cut > 0;
  if (det)
    VG_TRY(det_setup(c, io.det_part, io.det_bg, io.det_loss, st,
                     vm && c->opt.mode != VG_MODE_SPLAT ? &io : nullptr));
  if (c->scene.n > 0) {
    {
      ProfScope ps(c, VG_K_RENDER_BWD, st);
      if (c->opt.mode == VG_MODE_SPLAT)
        launch_splat_bwd(c->n_tiles, (const GRec*)c->rec.p, c->vals, (const uint2*)c->ranges.p,
                         (const uint32_t*)c->tord.p, p, target ? 1 : 0, io, st);
      else
      {
        // with the forward's visibility mask: (tile, segment) items, heaviest first
        // (atomic mode: the segment plan, and the next view's decision; a
        // deterministic backward after an atomic-mode forward: one CTA per tile)
        const SegIO seg = vm && c->seg_valid && !det ? seg_io(c) : SegIO();
        launch_render_bwd(c->n_tiles, (const GRec*)c->rec.p, c->vals, (const uint2*)c->ranges.p,
                          (const uint32_t*)c->tord.p, p, c->opt.alpha_cut > 0, target ? 1 : 0, io,
                          vm ? (const uint32_t*)c->vmask.p : nullptr, c->vm_words, st, seg);
      }
    }
    VG_LAUNCHED(c, 1);
    if (det) {
      float* bg_out;
      double* loss_out;
      VG_TRY(det_targets(c, g, loss_sum, bg_out, loss_out, st));
      VG_CUDA(det_reduce(c->pairs > 0 ? c->scene.n : 0, (const uint32_t*)c->det_cnt.p,
                         (const uint32_t*)c->det_off.p, (const uint32_t*)c->det_slot.p, (const float*)c->det_part.p,
                         (float*)c->acc.p, c->n_tiles, (const float*)c->det_bg.p,
                         target ? (const double*)c->det_loss.p : nullptr, bg_out,
                         loss_out, st, io.det_gvis4, (uint32_t*)c->det_big.p));
      VG_LAUNCHED(c, 2);
    }
    VG_TRY(finish_view(c, g, st, vm && c->seg_valid));
  } else {
    // empty scene: d_background = sum of d_color (grad.py:126-128) -- the
    // blend kernel still runs over the (empty) tiles to form it.
    launch_render_bwd(c->n_tiles, nullptr, nullptr, (const uint2*)c->ranges.p,
                      (const uint32_t*)c->tord.p, p, false, target ? 1 : 0, io, nullptr, 0, st);
    VG_LAUNCHED(c, 1);
    if (det) {
      float* bg_out;
      double* loss_out;
      VG_TRY(det_targets(c, g, loss_sum, bg_out, loss_out, st));
      VG_CUDA(det_reduce(0, nullptr, nullptr, nullptr, nullptr, nullptr, c->n_tiles,
                         (const float*)c->det_bg.p, target ? (const double*)c->det_loss.p : nullptr,
                         bg_out, loss_out, st));
      VG_LAUNCHED(c, 1);
    }
  }
  return VG_OK;
}

int vg_render_backward(vg_context* c, const float* color, const float* final_t,
                       const float* d_color, const float* d_t, vg_grads* g, void* stream) {
  if (!d_color) return fail(VG_EINVAL, "vg_render_backward: d_color is NULL");
  return render_bwd_common(c, color, final_t, d_color, d_t, nullptr, nullptr, g, stream);
}

int vg_render_backward_l2(vg_context* c, const float* color, const float* final_t,
                          const float* target, double* loss_sum, vg_grads* g, void* stream) {
  if (!target || !loss_sum) return fail(VG_EINVAL, "vg_render_backward_l2: NULL argument");
  return render_bwd_common(c, color, final_t, nullptr, nullptr, target, loss_sum, g, stream);
}

// Tomography CTAs per tile: enough to fill the GPU when a small detector has
// long per-tile lists (config 5: 1024 tiles x ~5k pairs).  The forward splits
// in batches of 256 entries (and sums partial images), the adjoint per pair.
static int tomo_splits(const vg_context* c, bool fwd) {
  static int env_f = -2, env_b = -2;
  int& e = fwd ? env_f : env_b;
  if (e == -2) {
    const char* v = getenv(fwd ? "VG_TOMO_SPLIT_F" : "VG_TOMO_SPLIT_B");
    e = v ? atoi(v) : -1;
  }
  if (e > 0) return e;
  if (c->n_tiles <= 0 || c->pairs <= 0) return 1;
  const int64_t avg = c->pairs / c->n_tiles;
  // forward: about one 256-entry batch per split; adjoint: about one pair
  // per thread (config 5 sweep: 383.7 ms/step unsplit -> 259-262 at 16-32 x 64)
  const int64_t s = fwd ? (avg + 255) / 256 : (avg + 127) / 128;
  return (int)(s < 1 ? 1 : s > 64 ? 64 : s);
}

int vg_tomo_forward(vg_context* c, float* image, float* intensity, void* stream) {
  if (!c || !image) return fail(VG_EINVAL, "vg_tomo_forward: NULL argument");
  if (!c->prepared) return fail(VG_EINVAL, "vg_tomo_forward: call vg_prepare first");
  if (c->opt.mode != VG_MODE_ANALYTIC) return fail(VG_EINVAL, "tomography is analytic-mode only");
  cudaStream_t st = (cudaStream_t)stream;
  BlendParams p = blend_params(c);
  {
    ProfScope ps(c, VG_K_TOMO_FWD, st);
    const int S = tomo_splits(c, true);
    if (S > 1)
      VG_TRY(ensure(c->tpart, sizeof(float) * (size_t)S * c->cam.width * c->cam.height, st));
    launch_tomo_fwd(c->n_tiles, c->cam.projection, (const GRec*)c->rec.p, c->vals,
                    (const uint2*)c->ranges.p, (const uint32_t*)c->tord.p, p, image, intensity, S,
                    (float*)c->tpart.p, st);
    if (S > 1) VG_LAUNCHED(c, 1);
  }
  VG_LAUNCHED(c, 1);
  return VG_OK;
}

static int tomo_bwd_common(vg_context* c, const float* d_image, const float* image,
                           const float* target, double* loss_sum, vg_grads* g, void* stream) {
  if (!c->prepared) return fail(VG_EINVAL, "vg_tomo_backward: call vg_prepare first");
  if (c->opt.mode != VG_MODE_ANALYTIC) return fail(VG_EINVAL, "tomography is analytic-mode only");
  cudaStream_t st = (cudaStream_t)stream;
  VG_TRY(prep_grads(c, g, st));
  BlendParams p = blend_params(c);
  uint8_t* vis = g->visible;
  if (!vis) {
    VG_TRY(ensure(c->offset, sizeof(uint32_t) * (size_t)(c->scene.n > 0 ? c->scene.n : 1), st));
    vis = (uint8_t*)c->offset.p;
  }
  float scale = (float)(2.0 / ((double)c->cam.width * (double)c->cam.height));
  const bool det = c->opt.deterministic != 0;
  float *dpart = nullptr, *dbg = nullptr;
  double* dloss = nullptr;
  if (det) VG_TRY(det_setup(c, dpart, dbg, dloss, st));
  {
    ProfScope ps(c, VG_K_TOMO_BWD, st);
    launch_tomo_bwd(c->n_tiles, tomo_splits(c, false), c->cam.projection, target ? 1 : 0,
                    (const GRec*)c->rec.p, c->vals,
                    (const uint2*)c->ranges.p, (const uint32_t*)c->tord.p, p, d_image, image,
                    target, scale, loss_sum, (float*)c->acc.p, vis, dpart, dloss, st);
  }
  VG_LAUNCHED(c, 1);
  if (det) {
    // tile loss partials exist only with the fused L2 (target); no d_background in tomography
    float* bg_out;
    double* loss_out;
    vg_grads gn = *g;
    gn.d_background = nullptr;
    VG_TRY(det_targets(c, &gn, loss_sum, bg_out, loss_out, st));
    VG_CUDA(det_reduce(c->pairs > 0 ? c->scene.n : 0, (const uint32_t*)c->det_cnt.p,
                       (const uint32_t*)c->det_off.p, (const uint32_t*)c->det_slot.p, (const float*)c->det_part.p,
                       (float*)c->acc.p, c->n_tiles, dbg, target ? dloss : nullptr, nullptr,
                       loss_out, st));
    VG_LAUNCHED(c, 2);
  }
  VG_TRY(finish_view(c, g, st));
  return VG_OK;
}

int vg_tomo_backward(vg_context* c, const float* d_image, vg_grads* g, void* stream) {
  if (!c || !d_image) return fail(VG_EINVAL, "vg_tomo_backward: NULL argument");
  return tomo_bwd_common(c, d_image, nullptr, nullptr, nullptr, g, stream);
}

int vg_tomo_backward_l2(vg_context* c, const float* image, const float* target, double* loss_sum,
                        vg_grads* g, void* stream) {
  if (!c || !image || !target || !loss_sum) return fail(VG_EINVAL, "vg_tomo_backward_l2: NULL argument");
  return tomo_bwd_common(c, nullptr, image, target, loss_sum, g, stream);
}

#ifdef VG_DEBUG
// Debug builds only (not in the public header): 0 if every guard band of the
// context's buffers still holds its 0xA5 poison, else the number of damaged
// buffers (first index in *first_bad, in all_bufs order).  Synchronises.
int vg_debug_guard_check(vg_context* c, int32_t* first_bad) {
  if (!c) return -1;
  VG_CUDA(cudaDeviceSynchronize());
  std::vector<unsigned char> h(VG_GUARD);
  int bad = 0, idx = 0;
  if (first_bad) *first_bad = -1;
  for (Buf* b : all_bufs(c)) {
    if (b->p) {
      for (int side = 0; side < 2; ++side) {
        const char* g = side ? (const char*)b->p + b->bytes : (const char*)b->p - VG_GUARD;
        VG_CUDA(cudaMemcpy(h.data(), g, VG_GUARD, cudaMemcpyDeviceToHost));
        bool ok = true;
        for (unsigned char x : h) ok &= x == 0xA5;
        if (!ok) {
          if (first_bad && *first_bad < 0) *first_bad = idx;
          ++bad;
          break;
        }
      }
    }
    ++idx;
  }
  return bad;
}
#endif

}  // extern "C"
