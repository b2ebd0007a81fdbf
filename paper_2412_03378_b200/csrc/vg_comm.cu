// Gradient exchange of the view-sharded multi-GPU step:
// vg_allreduce_grads sums the flat float32 gradient buffer and the float64
// loss over the ranks of an NCCL communicator and OR-reduces the per-primitive
// `visible` bytes (max over uint8), in one NCCL group on the caller's stream.
//
// NCCL is resolved at run time (dlopen / dlsym): the library binds to the
// libnccl.so.2 the process already has loaded (torch's), or to the one named
// by VG_NCCL_LIB, so libvolgauss_b200.so itself has no link-time NCCL
// dependency and loads on hosts without it.  The minimal declarations below
// follow nccl.h (NCCL 2.x ABI: ncclUniqueId is 128 bytes; ncclUint8 = 1,
// ncclFloat32 = 7, ncclFloat64 = 8; ncclSum = 0, ncclMax = 2).
#include <dlfcn.h>

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "vg_kernels.cuh"

namespace {

typedef int nccl_result;
typedef void* nccl_comm;
struct nccl_uid {
  char internal[128];
};
enum { NCCL_UINT8 = 1, NCCL_FLOAT32 = 7, NCCL_FLOAT64 = 8 };
enum { NCCL_SUM = 0, NCCL_MAX = 2 };

struct NcclApi {
  nccl_result (*get_unique_id)(nccl_uid*) = nullptr;
  nccl_result (*comm_init_rank)(nccl_comm*, int, nccl_uid, int) = nullptr;
  nccl_result (*comm_destroy)(nccl_comm) = nullptr;
  nccl_result (*all_reduce)(const void*, void*, size_t, int, int, nccl_comm, cudaStream_t) = nullptr;
  nccl_result (*group_start)() = nullptr;
  nccl_result (*group_end)() = nullptr;
  const char* (*error_string)(nccl_result) = nullptr;
  bool ok = false;
  std::string why;
};

NcclApi g_nccl;
std::once_flag g_nccl_once;

void load_nccl() {
  void* h = nullptr;
  const char* env = std::getenv("VG_NCCL_LIB");
  if (env && *env) h = dlopen(env, RTLD_NOW | RTLD_LOCAL);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // already in the process (torch)
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
  if (!h) {
    g_nccl.why = std::string("libnccl.so.2 not found (set VG_NCCL_LIB): ") + dlerror();
    return;
  }
  auto sym = [&](const char* name) { return dlsym(h, name); };
  g_nccl.get_unique_id = reinterpret_cast<decltype(g_nccl.get_unique_id)>(sym("ncclGetUniqueId"));
  g_nccl.comm_init_rank = reinterpret_cast<decltype(g_nccl.comm_init_rank)>(sym("ncclCommInitRank"));
  g_nccl.comm_destroy = reinterpret_cast<decltype(g_nccl.comm_destroy)>(sym("ncclCommDestroy"));
  g_nccl.all_reduce = reinterpret_cast<decltype(g_nccl.all_reduce)>(sym("ncclAllReduce"));
  g_nccl.group_start = reinterpret_cast<decltype(g_nccl.group_start)>(sym("ncclGroupStart"));
  g_nccl.group_end = reinterpret_cast<decltype(g_nccl.group_end)>(sym("ncclGroupEnd"));
  g_nccl.error_string = reinterpret_cast<decltype(g_nccl.error_string)>(sym("ncclGetErrorString"));
  g_nccl.ok = g_nccl.get_unique_id && g_nccl.comm_init_rank && g_nccl.comm_destroy &&
              g_nccl.all_reduce && g_nccl.group_start && g_nccl.group_end;
  if (!g_nccl.ok) g_nccl.why = "libnccl.so.2 lacks an expected symbol";
}

int need_nccl() {
  std::call_once(g_nccl_once, load_nccl);
  return g_nccl.ok ? VG_OK : vg::set_error(VG_ECUDA, g_nccl.why.c_str());
}

int nccl_fail(const char* what, nccl_result r) {
  std::string m = std::string(what) + ": NCCL error " + std::to_string(r);
  if (g_nccl.error_string) m += std::string(" (") + g_nccl.error_string(r) + ")";
  return vg::set_error(VG_ECUDA, m.c_str());
}

}  // namespace

extern "C" {

int vg_nccl_available(void) { return need_nccl() == VG_OK ? 1 : 0; }

int vg_nccl_unique_id(void* out128) {
  if (!out128) return vg::set_error(VG_EINVAL, "vg_nccl_unique_id: NULL output");
  if (int e = need_nccl()) return e;
  nccl_uid id;
  if (nccl_result r = g_nccl.get_unique_id(&id)) return nccl_fail("ncclGetUniqueId", r);
  std::memcpy(out128, id.internal, sizeof(id.internal));
  return VG_OK;
}

int vg_nccl_comm_init(void** comm, int32_t nranks, const void* id128, int32_t rank, int32_t device) {
  if (!comm || !id128) return vg::set_error(VG_EINVAL, "vg_nccl_comm_init: NULL argument");
  if (nranks < 1 || rank < 0 || rank >= nranks)
    return vg::set_error(VG_EINVAL, "vg_nccl_comm_init: bad rank / world size");
  if (int e = need_nccl()) return e;
  if (cudaSetDevice(device) != cudaSuccess) return vg::set_error(VG_EINVAL, "vg_nccl_comm_init: bad device");
  nccl_uid id;
  std::memcpy(id.internal, id128, sizeof(id.internal));
  nccl_comm c = nullptr;
  if (nccl_result r = g_nccl.comm_init_rank(&c, nranks, id, rank)) return nccl_fail("ncclCommInitRank", r);
  *comm = c;
  return VG_OK;
}

int vg_nccl_comm_destroy(void* comm) {
  if (!comm) return VG_OK;
  if (int e = need_nccl()) return e;
  if (nccl_result r = g_nccl.comm_destroy(comm)) return nccl_fail("ncclCommDestroy", r);
  return VG_OK;
}

int vg_allreduce_grads(vg_context* ctx, void* comm, float* flat, int64_t count, uint8_t* visible,
                       int64_t n_visible, double* loss, void* stream) {
  (void)ctx;  // the buffers belong to the caller; ctx is accepted for the 8(b) signature
  if (!comm) return vg::set_error(VG_EINVAL, "vg_allreduce_grads: NULL communicator");
  if (count < 0 || n_visible < 0 || (count > 0 && !flat) || (n_visible > 0 && !visible))
    return vg::set_error(VG_EINVAL, "vg_allreduce_grads: bad buffer");
  if (int e = need_nccl()) return e;
  cudaStream_t st = (cudaStream_t)stream;
  if (nccl_result r = g_nccl.group_start()) return nccl_fail("ncclGroupStart", r);
  nccl_result r = 0;
  if (count > 0) r = g_nccl.all_reduce(flat, flat, (size_t)count, NCCL_FLOAT32, NCCL_SUM, comm, st);
  if (!r && n_visible > 0)
    r = g_nccl.all_reduce(visible, visible, (size_t)n_visible, NCCL_UINT8, NCCL_MAX, comm, st);
  if (!r && loss) r = g_nccl.all_reduce(loss, loss, 1, NCCL_FLOAT64, NCCL_SUM, comm, st);
  nccl_result r2 = g_nccl.group_end();
  if (r) return nccl_fail("ncclAllReduce", r);
  if (r2) return nccl_fail("ncclGroupEnd", r2);
  return VG_OK;
}

}  // extern "C"
