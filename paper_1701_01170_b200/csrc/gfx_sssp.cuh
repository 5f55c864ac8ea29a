// Near/far pile phases shared by the single-GPU SSSP (gfx_sssp.cu: the
// host-driven loop's kernels and the device-resident persistent loop) and the
// partitioned SSSP engine (gfx_dsssp.cu).  Reference near_far.py:20-85.
// Kernels are `static` so each translation unit keeps its own copy (no -rdc);
// the phase bodies are device functions so the persistent loop runs them
// between grid barriers.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "gfx_internal.cuh"

namespace gfx {

// Block-staged appends for the near / far piles: each CTA collects its
// items in shared memory (block-local atomics) and appends them to the
// global pile with ONE atomicAdd per flush, instead of two same-address
// global atomics per warp and tile.
constexpr int kPileStage = 2048;
struct PileStage {
  int32_t nv[kPileStage];
  int32_t fv[kPileStage], fk[kPileStage];
  int nn, nfar;
  unsigned long long base;
};

static __device__ __forceinline__ void pile_flush(PileStage& S, int32_t* __restrict__ near,
                                                  unsigned long long* __restrict__ near_len,
                                                  int32_t* __restrict__ far,
                                                  int32_t* __restrict__ far_key,
                                                  unsigned long long* __restrict__ far_len) {
  __syncthreads();
  if (threadIdx.x == 0) S.base = S.nn ? atomicAdd(near_len, (unsigned long long)S.nn) : 0ull;
  __syncthreads();
  for (int i = threadIdx.x; i < S.nn; i += blockDim.x) near[S.base + i] = S.nv[i];
  __syncthreads();
  if (threadIdx.x == 0) S.base = S.nfar ? atomicAdd(far_len, (unsigned long long)S.nfar) : 0ull;
  __syncthreads();
  for (int i = threadIdx.x; i < S.nfar; i += blockDim.x) {
    far[S.base + i] = S.fv[i];
    far_key[S.base + i] = S.fk[i];
  }
  __syncthreads();
  if (threadIdx.x == 0) S.nn = S.nfar = 0;
  __syncthreads();
}

// split the improved vertices touched[0..n) against the threshold
// (near_far.py:40-57); every CTA of the grid calls it (block-uniform loop)
static __device__ __forceinline__ void sssp_split_phase(
    PileStage& S, const int32_t* __restrict__ touched, int64_t n, const uint32_t* __restrict__ dist,
    uint32_t* __restrict__ mark, double threshold, int32_t* __restrict__ near,
    unsigned long long* __restrict__ near_len, int32_t* __restrict__ far,
    int32_t* __restrict__ far_key, unsigned long long* __restrict__ far_len) {
  if (threadIdx.x == 0) S.nn = S.nfar = 0;
  __syncthreads();
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < n;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = base + threadIdx.x;
    if (i < n) {
      const int32_t v = touched[i];
      const int32_t key = (int32_t)dist[v];
      atomicAnd(&mark[v >> 5], ~(1u << (v & 31)));  // re-arm for the next iteration
      if ((double)key < threshold) {
        S.nv[atomicAdd(&S.nn, 1)] = v;
      } else {
        const int at = atomicAdd(&S.nfar, 1);
        S.fv[at] = v;
        S.fk[at] = key;
      }
    }
    __syncthreads();
    if (S.nn > kPileStage - (int)blockDim.x || S.nfar > kPileStage - (int)blockDim.x)
      pile_flush(S, near, near_len, far, far_key, far_len);
  }
  pile_flush(S, near, near_len, far, far_key, far_len);
}

// the same split over a touched list WITH duplicates: the first occurrence
// of a vertex in iteration `it` (stamp test-and-set) is split, the rest skip
static __device__ __forceinline__ void sssp_split_late_phase(
    PileStage& S, const int32_t* __restrict__ touched, int64_t n, const uint32_t* __restrict__ dist,
    int32_t* __restrict__ stamp, int32_t it, double threshold, int32_t* __restrict__ near,
    unsigned long long* __restrict__ near_len, int32_t* __restrict__ far,
    int32_t* __restrict__ far_key, unsigned long long* __restrict__ far_len) {
  if (threadIdx.x == 0) S.nn = S.nfar = 0;
  __syncthreads();
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < n;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = base + threadIdx.x;
    if (i < n) {
      const int32_t v = touched[i];
      if (atomicExch(&stamp[v], it) != it) {
        const int32_t key = (int32_t)dist[v];
        if ((double)key < threshold) {
          S.nv[atomicAdd(&S.nn, 1)] = v;
        } else {
          const int at = atomicAdd(&S.nfar, 1);
          S.fv[at] = v;
          S.fk[at] = key;
        }
      }
    }
    __syncthreads();
    if (S.nn > kPileStage - (int)blockDim.x || S.nfar > kPileStage - (int)blockDim.x)
      pile_flush(S, near, near_len, far, far_key, far_len);
  }
  pile_flush(S, near, near_len, far, far_key, far_len);
}

static __global__ void __launch_bounds__(256)
    k_sssp_split(const int32_t* __restrict__ touched, const unsigned long long* __restrict__ n_d,
                 const uint32_t* __restrict__ dist, uint32_t* __restrict__ mark, double threshold,
                 int32_t* __restrict__ near, unsigned long long* __restrict__ near_len,
                 int32_t* __restrict__ far, int32_t* __restrict__ far_key,
                 unsigned long long* __restrict__ far_len) {
  __shared__ PileStage S;
  sssp_split_phase(S, touched, (int64_t)*n_d, dist, mark, threshold, near, near_len, far, far_key,
                   far_len);
}

// advance_bucket (near_far.py:68-85): drop stale far entries, split the rest
// against the new threshold.  With split == false only the stale drop runs
// (capacity compaction; everything fresh stays far).
static __device__ __forceinline__ void sssp_refar_phase(
    PileStage& S, const int32_t* __restrict__ far, const int32_t* __restrict__ far_key, int64_t n,
    const uint32_t* __restrict__ dist, double threshold, int split, int32_t* __restrict__ near,
    unsigned long long* __restrict__ near_len, int32_t* __restrict__ far2,
    int32_t* __restrict__ far2_key, unsigned long long* __restrict__ far2_len) {
  if (threadIdx.x == 0) S.nn = S.nfar = 0;
  __syncthreads();
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < n;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = base + threadIdx.x;
    if (i < n) {
      const int32_t v = far[i];
      const int32_t key = far_key[i];
      if ((int32_t)dist[v] == key) {  // fresh
        if (split && (double)key < threshold) {
          S.nv[atomicAdd(&S.nn, 1)] = v;
        } else {
          const int at = atomicAdd(&S.nfar, 1);
          S.fv[at] = v;
          S.fk[at] = key;
        }
      }
    }
    __syncthreads();
    if (S.nn > kPileStage - (int)blockDim.x || S.nfar > kPileStage - (int)blockDim.x)
      pile_flush(S, near, near_len, far2, far2_key, far2_len);
  }
  pile_flush(S, near, near_len, far2, far2_key, far2_len);
}

// Two-level far pile (device-resident loop): `soon` holds far entries below
// the window bound fw, `later` the rest.  An advance re-splits only the soon
// pile; the later pile is re-split when the soon pile has run dry (with a new
// window), so a far entry is scanned about window/delta times at most instead
// of once per advance.  Same stale rule as near_far.py:68-85; every entry's
// route depends only on (dist, key, threshold, fw), so distances are those of
// the one-pile loop.
constexpr int kPileStage3 = 1024;
struct PileStage3 {
  int32_t nv[kPileStage3];
  int32_t fv[kPileStage3], fk[kPileStage3];
  int32_t lv[kPileStage3], lk[kPileStage3];
  int nn, nfar, nl, lmin;
  unsigned long long base;
};

static __device__ __forceinline__ void pile_append(int32_t* __restrict__ sv,
                                                   const int32_t* __restrict__ sk, int cnt,
                                                   unsigned long long& base,
                                                   int32_t* __restrict__ v,
                                                   int32_t* __restrict__ k,
                                                   unsigned long long* __restrict__ len) {
  __syncthreads();
  if (threadIdx.x == 0) base = cnt ? atomicAdd(len, (unsigned long long)cnt) : 0ull;
  __syncthreads();
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
    v[base + i] = sv[i];
    if (k) k[base + i] = sk[i];
  }
}

static __device__ __forceinline__ void pile_flush3(
    PileStage3& S, int32_t* __restrict__ near, unsigned long long* __restrict__ near_len,
    int32_t* __restrict__ soon, int32_t* __restrict__ soon_key,
    unsigned long long* __restrict__ soon_len, int32_t* __restrict__ later,
    int32_t* __restrict__ later_key, unsigned long long* __restrict__ later_len) {
  pile_append(S.nv, nullptr, S.nn, S.base, near, nullptr, near_len);
  pile_append(S.fv, S.fk, S.nfar, S.base, soon, soon_key, soon_len);
  pile_append(S.lv, S.lk, S.nl, S.base, later, later_key, later_len);
  __syncthreads();
  if (threadIdx.x == 0) S.nn = S.nfar = S.nl = 0;
  __syncthreads();
}

// fresh entries of in[0..n): key < threshold -> near, key < fw -> soon,
// else -> later (stale ones dropped); *later_max_inv = max(0xFFFFFFFF - key)
// over the entries sent to later (a running minimum of the later keys)
static __device__ __forceinline__ void sssp_refar2_phase(
    PileStage3& S, const int32_t* __restrict__ in, const int32_t* __restrict__ in_key, int64_t n,
    const uint32_t* __restrict__ dist, double threshold, double fw, int32_t* __restrict__ near,
    unsigned long long* __restrict__ near_len, int32_t* __restrict__ soon,
    int32_t* __restrict__ soon_key, unsigned long long* __restrict__ soon_len,
    int32_t* __restrict__ later, int32_t* __restrict__ later_key,
    unsigned long long* __restrict__ later_len, unsigned long long* __restrict__ later_max_inv) {
  if (threadIdx.x == 0) {
    S.nn = S.nfar = S.nl = 0;
    S.lmin = 0x7fffffff;
  }
  __syncthreads();
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < n;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = base + threadIdx.x;
    if (i < n) {
      const int32_t v = in[i];
      const int32_t key = in_key[i];
      if ((int32_t)dist[v] == key) {  // fresh
        if ((double)key < threshold) {
          S.nv[atomicAdd(&S.nn, 1)] = v;
        } else if ((double)key < fw) {
          const int at = atomicAdd(&S.nfar, 1);
          S.fv[at] = v;
          S.fk[at] = key;
        } else {
          const int at = atomicAdd(&S.nl, 1);
          S.lv[at] = v;
          S.lk[at] = key;
          atomicMin(&S.lmin, key);
        }
      }
    }
    __syncthreads();
    const int lim = kPileStage3 - (int)blockDim.x;
    if (S.nn > lim || S.nfar > lim || S.nl > lim)
      pile_flush3(S, near, near_len, soon, soon_key, soon_len, later, later_key, later_len);
  }
  pile_flush3(S, near, near_len, soon, soon_key, soon_len, later, later_key, later_len);
  if (threadIdx.x == 0 && S.lmin != 0x7fffffff)
    atomicMax(later_max_inv, 0xFFFFFFFFull - (unsigned long long)(uint32_t)S.lmin);
}

static __global__ void __launch_bounds__(256)
    k_sssp_refar(const int32_t* __restrict__ far, const int32_t* __restrict__ far_key, int64_t n,
                 const uint32_t* __restrict__ dist, double threshold, int split,
                 int32_t* __restrict__ near, unsigned long long* __restrict__ near_len,
                 int32_t* __restrict__ far2, int32_t* __restrict__ far2_key,
                 unsigned long long* __restrict__ far2_len) {
  __shared__ PileStage S;
  sssp_refar_phase(S, far, far_key, n, dist, threshold, split, near, near_len, far2, far2_key,
                   far2_len);
}

// (dist | pred) words -> the two int32 outputs; two vertices per thread with
// 16-byte loads and 8-byte stores when the outputs are 8-byte aligned
static __device__ __forceinline__ void sssp_unpack_phase(const unsigned long long* __restrict__ dp,
                                                         int64_t n, int32_t* __restrict__ dist,
                                                         int32_t* __restrict__ preds, int vec,
                                                         int64_t t0, int64_t stride) {
  int64_t done = 0;
  if (vec) {
    const int64_t pairs = n >> 1;
    for (int64_t p = t0; p < pairs; p += stride) {
      const ulonglong2 x = reinterpret_cast<const ulonglong2*>(dp)[p];
      const uint32_t d0 = (uint32_t)(x.x >> 32), d1 = (uint32_t)(x.y >> 32);
      reinterpret_cast<int2*>(dist)[p] =
          make_int2(d0 == 0xFFFFFFFFu ? GFX_UNVISITED : (int32_t)d0,
                    d1 == 0xFFFFFFFFu ? GFX_UNVISITED : (int32_t)d1);
      reinterpret_cast<int2*>(preds)[p] = make_int2((int32_t)(uint32_t)x.x, (int32_t)(uint32_t)x.y);
    }
    done = pairs << 1;
  }
  for (int64_t v = done + t0; v < n; v += stride) {
    const unsigned long long x = dp[v];
    const uint32_t d = (uint32_t)(x >> 32);
    dist[v] = d == 0xFFFFFFFFu ? GFX_UNVISITED : (int32_t)d;
    preds[v] = (int32_t)(uint32_t)x;
  }
}

static __global__ void k_sssp_unpack(const unsigned long long* __restrict__ dp, int64_t n,
                                     int32_t* __restrict__ dist, int32_t* __restrict__ preds,
                                     int vec) {
  sssp_unpack_phase(dp, n, dist, preds, vec, blockIdx.x * (int64_t)blockDim.x + threadIdx.x,
                    (int64_t)gridDim.x * blockDim.x);
}

}  // namespace gfx
