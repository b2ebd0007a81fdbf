// sort_by="gamma" (raster.prepare + _resort_by_gamma, raster.py:291-312):
// every tile list (depth order, from the span binning) is re-sorted stably
// by gamma = (M delta) . d / (d^T M d), the centre of the Gaussian's 1D
// restriction to the tile's central ray d (the unit world direction through
// pixel (min(16 ty + 8, H-1), min(16 tx + 8, W-1)), camera.py:57-64).
//
// One CTA per tile.  gamma is evaluated in float64 from the per-Gaussian
// precision matrix M and M delta that preprocess wrote, and mapped to an
// order-preserving 64-bit key.  Lists of up to 2048 entries are bitonic-
// sorted in shared memory on (key, position) -- stable by construction;
// longer lists are sorted in 2048-entry runs and merged pairwise in global
// memory (merge path, ties take the earlier run), ping-ponging between two
// scratch buffers.
#include "vg_kernels.cuh"

namespace vg {
namespace gsort {

constexpr int NT = 256;
constexpr int CAP = 2048;  // entries per shared-memory run

__device__ __forceinline__ unsigned long long okey(double g) {
  unsigned long long b = (unsigned long long)__double_as_longlong(g);
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}

struct Args {
  const uint2* ranges;
  uint32_t* vals;
  const double* gm;  // per Gaussian: M (xx, xy, xz, yy, yz, zz), M delta (3)
  unsigned long long* k0;
  unsigned long long* k1;
  uint32_t* v0;
  uint32_t* v1;
  CamK cam;
};

__device__ __forceinline__ double gamma_of(const double* __restrict__ gm, uint32_t g, const double* d) {
  const double* q = gm + 9 * (size_t)g;
  const double a = q[0] * d[0] * d[0] + q[3] * d[1] * d[1] + q[5] * d[2] * d[2] +
                   2.0 * (q[1] * d[0] * d[1] + q[2] * d[0] * d[2] + q[4] * d[1] * d[2]);
  const double b = q[6] * d[0] + q[7] * d[1] + q[8] * d[2];
  return b / a;
}

// Bitonic sort of n <= CAP (key, pos) pairs in shared memory, padded to a
// power of two with (max, max) -- stable because positions break ties.
__device__ void bitonic(unsigned long long* key, uint32_t* pos, int n) {
  int m = 1;
  while (m < n) m <<= 1;
  for (int i = n + threadIdx.x; i < m; i += NT) {
    key[i] = ~0ull;
    pos[i] = 0xffffffffu;
  }
  __syncthreads();
  for (int k = 2; k <= m; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < m; i += NT) {
        const int l = i ^ j;
        if (l > i) {
          const bool up = (i & k) == 0;
          const unsigned long long ka = key[i], kb = key[l];
          const uint32_t pa = pos[i], pb = pos[l];
          const bool gt = ka > kb || (ka == kb && pa > pb);
          if (gt == up) {
            key[i] = kb; key[l] = ka;
            pos[i] = pb; pos[l] = pa;
          }
        }
      }
      __syncthreads();
    }
  }
}

__global__ void __launch_bounds__(NT) k_gamma_sort(Args a) {
  __shared__ unsigned long long skey[CAP];
  __shared__ uint32_t spos[CAP];
  __shared__ double sd[3];
  const int t = blockIdx.x;
  const uint2 r = a.ranges[t];
  const int L = (int)(r.y - r.x);
  if (L < 2) return;
  if (threadIdx.x == 0) {
    const int ty = t / a.cam.ntx, tx = t - ty * a.cam.ntx;
    const int row = min(ty * TILE + TILE / 2, a.cam.height - 1);
    const int col = min(tx * TILE + TILE / 2, a.cam.width - 1);
    double dv[3] = {((double)col + 0.5 - a.cam.cx) / a.cam.fx, ((double)row + 0.5 - a.cam.cy) / a.cam.fy, 1.0};
    const double nn = sqrt(dot3(dv, dv));
    for (int k = 0; k < 3; ++k) dv[k] /= nn;
    // d_world = R^T d_view (rows of R are the view axes)
    for (int j = 0; j < 3; ++j)
      sd[j] = a.cam.R[0 * 3 + j] * dv[0] + a.cam.R[1 * 3 + j] * dv[1] + a.cam.R[2 * 3 + j] * dv[2];
  }
  __syncthreads();
  const double d[3] = {sd[0], sd[1], sd[2]};
  uint32_t* vals = a.vals + r.x;
  // 1. runs of CAP sorted in shared memory
  for (int c0 = 0; c0 < L; c0 += CAP) {
    const int n = min(CAP, L - c0);
    for (int i = threadIdx.x; i < n; i += NT) {
      skey[i] = okey(gamma_of(a.gm, vals[c0 + i], d));
      spos[i] = (uint32_t)(c0 + i);
    }
    __syncthreads();
    bitonic(skey, spos, n);
    if (L <= CAP) {
      // single run: gather the ids (the original list is intact until here)
      uint32_t g[CAP / NT];
#pragma unroll
      for (int q = 0; q < CAP / NT; ++q) {
        const int i = threadIdx.x + q * NT;
        g[q] = i < n ? vals[spos[i]] : 0u;
      }
      __syncthreads();
#pragma unroll
      for (int q = 0; q < CAP / NT; ++q) {
        const int i = threadIdx.x + q * NT;
        if (i < n) vals[i] = g[q];
      }
      return;
    }
    for (int i = threadIdx.x; i < n; i += NT) {
      a.k0[r.x + c0 + i] = skey[i];
      a.v0[r.x + c0 + i] = vals[spos[i]];
    }
    __syncthreads();
  }
  // 2. pairwise merges of runs in global memory
  unsigned long long* ks = a.k0 + r.x;
  unsigned long long* kd = a.k1 + r.x;
  uint32_t* vs = a.v0 + r.x;
  uint32_t* vd = a.v1 + r.x;
  for (int w = CAP; w < L; w <<= 1) {
    for (int lo = 0; lo < L; lo += 2 * w) {
      const int mid = min(lo + w, L), hi = min(lo + 2 * w, L);
      const int na = mid - lo, nb = hi - mid, len = hi - lo;
      const unsigned long long* A = ks + lo;
      const unsigned long long* B = ks + mid;
      const int per = (len + NT - 1) / NT;
      const int k0 = min(len, (int)threadIdx.x * per), k1 = min(len, k0 + per);
      // merge path: number of A entries among the first k0 outputs (ties -> A first)
      int b0 = max(0, k0 - nb), e0 = min(k0, na);
      while (b0 < e0) {
        const int m = (b0 + e0) >> 1;
        if (A[m] <= B[k0 - 1 - m]) b0 = m + 1;
        else e0 = m;
      }
      int i = b0, j = k0 - b0;
      for (int k = k0; k < k1; ++k) {
        const bool takeA = j >= nb || (i < na && A[i] <= B[j]);
        if (takeA) {
          kd[lo + k] = A[i];
          vd[lo + k] = vs[lo + i];
          ++i;
        } else {
          kd[lo + k] = B[j];
          vd[lo + k] = vs[mid + j];
          ++j;
        }
      }
    }
    __syncthreads();
    unsigned long long* tk = ks; ks = kd; kd = tk;
    uint32_t* tv = vs; vs = vd; vd = tv;
  }
  for (int i = threadIdx.x; i < L; i += NT) vals[i] = vs[i];
}

}  // namespace gsort

size_t gamma_scratch_bytes(int64_t pairs) {
  return (size_t)pairs * 2 * (sizeof(unsigned long long) + sizeof(uint32_t));
}

void launch_gamma_sort(int n_tiles, const uint2* ranges, uint32_t* vals, const double* gm,
                       int64_t pairs, void* scratch, const CamK& cam, cudaStream_t st) {
  gsort::Args a;
  a.ranges = ranges;
  a.vals = vals;
  a.gm = gm;
  a.k0 = (unsigned long long*)scratch;
  a.k1 = a.k0 + pairs;
  a.v0 = (uint32_t*)(a.k1 + pairs);
  a.v1 = a.v0 + pairs;
  a.cam = cam;
  gsort::k_gamma_sort<<<n_tiles, gsort::NT, 0, st>>>(a);
}

}  // namespace vg
