// Triangle counting: degree orientation + sorted-list intersection.
//
// Reference: primitives/tc.py:27-86 keeps slot s -> d iff deg[s] > deg[d] or
// (deg[s] == deg[d] and s < d) (tc.py:57-59), rebuilds a canonical oriented
// CSR with coo_to_csr (tc.py:53-56), then counts |N+(u) ∩ N+(v)| for every
// oriented edge in that CSR order (segmented_intersect, operators.py:485-525).
//
// Device: orientation keeps each row's surviving slots in order, so the
// compacted rows ARE the canonical oriented CSR (sorted by (src, dst)).
// Counting (default): every triangle {x, y, z} with rank x < y < z (rank =
// the reference's orientation order: degree, then smaller id higher) is
// found ONCE from the rank-increasing side -- for the edge x => y of the
// REVERSED orientation, z is a common element of the two (short) reversed
// rows x and y -- and credited to the reference's oriented edge z -> y, the
// only one of its three edges whose endpoints' out-lists both hold the third
// vertex (tc.py:57-59: x is a common out-neighbour of z and y).  The
// reversed CSR and the map from its slots to the reference's oriented slots
// are built once with the orientation (preprocessing, like the reference's
// oriented-adjacency build).  Reversed rows are bounded by O(sqrt(m)), so
// the work is the optimal sum over vertices of d+(v)^2 instead of the
// reference orientation's hub-sized out-lists.  Counts stay exact int32, in
// the reference's oriented CSR order.  GFX_TC_LEGACY=1 selects the direct
// intersection of the reference orientation (below) for comparison:
// one thread merges both lists when they are short; longer pairs go to a
// list handled warp-cooperatively (each lane binary-searches elements of the
// shorter list in the longer one), hub rows through per-CTA bitmaps.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "gfx_device.cuh"
#include "gfx_internal.cuh"

namespace gfx {

__device__ __forceinline__ bool keep_slot(const int64_t* row, int64_t ds, int32_t s, int32_t d) {
  const int64_t dd = row[d + 1] - row[d];
  return ds > dd || (ds == dd && s < d);
}

// pass 0: count kept slots per row; pass 1: write them (ordered compaction)
template <bool WRITE>
__global__ void __launch_bounds__(256)
    k_tc_orient(const int64_t* __restrict__ row, const int32_t* __restrict__ col, int64_t n,
                int64_t* __restrict__ ocnt, const int64_t* __restrict__ orow,
                int32_t* __restrict__ ocol, int32_t* __restrict__ osrc) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t grp = gw; grp * 32 < n; grp += nw) {
    const int64_t v = grp * 32 + lane;
    int64_t b = 0, e = 0;
    if (v < n) {
      b = row[v];
      e = row[v + 1];
    }
    const bool heavy = (e - b) > 32;
    if (v < n && !heavy) {
      // 8 neighbours' ids, then their row bounds, in flight per batch
      int64_t k = WRITE ? orow[v] : 0;
      for (int64_t p0 = b; p0 < e; p0 += 8) {
        int32_t d[8];
        int64_t dd[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) d[t] = p0 + t < e ? col[p0 + t] : -1;
#pragma unroll
        for (int t = 0; t < 8; ++t) dd[t] = d[t] >= 0 ? row[d[t] + 1] - row[d[t]] : 0;
        const int64_t ds = e - b;
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          if (d[t] < 0) continue;
          if (ds > dd[t] || (ds == dd[t] && (int32_t)v < d[t])) {  // keep_slot
            if (WRITE) {
              ocol[k] = d[t];
              osrc[k] = (int32_t)v;
            }
            ++k;
          }
        }
      }
      if (!WRITE) ocnt[v] = k;
    }
    unsigned hm = __ballot_sync(0xffffffffu, heavy);
    while (hm) {
      const int k = __ffs(hm) - 1;
      hm &= hm - 1;
      const int64_t kv = grp * 32 + k;
      const int64_t kb = __shfl_sync(0xffffffffu, b, k), ke = __shfl_sync(0xffffffffu, e, k);
      int64_t pos = WRITE ? orow[kv] : 0;
      // 8 rows of 32 slots per step: ids, then their row bounds, in flight
      for (int64_t p0 = kb; p0 < ke; p0 += 256) {
        int32_t d[8];
        int64_t dd[8];
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const int64_t p = p0 + t * 32 + lane;
          d[t] = p < ke ? col[p] : -1;
        }
#pragma unroll
        for (int t = 0; t < 8; ++t) dd[t] = d[t] >= 0 ? row[d[t] + 1] - row[d[t]] : 0;
        const int64_t ds = ke - kb;
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const bool keep = d[t] >= 0 && (ds > dd[t] || (ds == dd[t] && (int32_t)kv < d[t]));
          const unsigned km = __ballot_sync(0xffffffffu, keep);
          if (WRITE && keep) {
            const int64_t at = pos + __popc(km & ((1u << lane) - 1));
            ocol[at] = d[t];
            osrc[at] = (int32_t)kv;
          }
          pos += __popc(km);
        }
      }
      if (!WRITE && lane == 0) ocnt[kv] = pos;
    }
  }
}

// short lists: one thread merges; long: queued for the warp kernel
__global__ void __launch_bounds__(256)
    k_tc_small(const int32_t* __restrict__ us, const int32_t* __restrict__ vs, int64_t npairs,
               const int64_t* __restrict__ rows, const int32_t* __restrict__ cols,
               int32_t* __restrict__ counts, int32_t* __restrict__ heavy,
               unsigned long long* __restrict__ nheavy, unsigned long long* __restrict__ total,
               int64_t hub_deg = 0) {
  const int lane = threadIdx.x & 31;
  unsigned long long sum = 0;
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < npairs;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = base + threadIdx.x;
    bool big = false;
    if (i < npairs) {
      const int32_t u = us[i], v = vs[i];
      int64_t a = rows[u], ae = rows[u + 1], b = rows[v], be = rows[v + 1];
      if (hub_deg && ae - a > hub_deg) {
        // a hub source: counted by k_tc_hubs
      } else if (ae - a + be - b > 64) {
        big = true;
      } else {
        int c = 0;
        while (a < ae && b < be) {
          const int32_t x = cols[a], y = cols[b];
          c += (x == y);
          a += (x <= y);
          b += (y <= x);
        }
        counts[i] = c;
        sum += (unsigned long long)c;
      }
    }
    const unsigned hm = __ballot_sync(0xffffffffu, big);
    if (hm) {
      unsigned long long at = 0;
      if (lane == 0) at = atomicAdd(nheavy, (unsigned long long)__popc(hm));
      at = __shfl_sync(0xffffffffu, at, 0);
      if (big) heavy[at + __popc(hm & ((1u << lane) - 1))] = (int32_t)i;
    }
  }
  sum = warp_sum_u64(sum);
  if (lane == 0 && sum) atomicAdd(total, sum);
}

__global__ void __launch_bounds__(256)
    k_tc_heavy(const int32_t* __restrict__ us, const int32_t* __restrict__ vs,
               const int32_t* __restrict__ heavy, const unsigned long long* __restrict__ nheavy_d,
               const int64_t* __restrict__ rows, const int32_t* __restrict__ cols,
               int32_t* __restrict__ counts, unsigned long long* __restrict__ total) {
  const int lane = threadIdx.x & 31;
  const int64_t nheavy = (int64_t)*nheavy_d;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long sum = 0;
  for (int64_t h = gw; h < nheavy; h += nw) {
    const int32_t i = heavy[h];
    const int32_t u = us[i], v = vs[i];
    int64_t a = rows[u], ae = rows[u + 1], b = rows[v], be = rows[v + 1];
    if (ae - a > be - b) {  // a = shorter list
      int64_t t = a; a = b; b = t;
      t = ae; ae = be; be = t;
    }
    int c = 0;
    for (int64_t p = a + lane; p < ae; p += 32) {
      const int32_t x = cols[p];
      int64_t lo = b, hi = be;
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (cols[mid] < x) lo = mid + 1; else hi = mid;
      }
      c += (lo < be && cols[lo] == x);
    }
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) {
      counts[i] = c;
      sum += (unsigned long long)c;
    }
  }
  if (lane == 0 && sum) atomicAdd(total, sum);
}

// Hub rows of the oriented CSR (out-degree > kTcHub): one CTA per hub at a
// time keeps N+(u) as bits of its own bitmap slot (n bits, L2-resident for
// the scales benchmarked), then each warp counts, for one out-neighbour v,
// the elements of N+(v) whose bit is set -- one bitmap probe per element
// instead of a binary search over the hub's long list -- and clears the
// bits again.  Hubs are handed out dynamically.
constexpr int64_t kTcHub = 512;
__global__ void k_tc_hub_list(const int64_t* __restrict__ orow, int64_t n, int32_t* __restrict__ hubs,
                              unsigned long long* __restrict__ nhubs) {
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n;
       u += (int64_t)gridDim.x * blockDim.x)
    if (orow[u + 1] - orow[u] > kTcHub) hubs[atomicAdd(nhubs, 1ull)] = (int32_t)u;
}

// work item k: hub hub_of[k], its out-neighbours [j0[k], j1[k]) (a hub's
// pairs are cut into kTcHubChunk-pair items so the largest hubs spread over
// many CTAs; every item rebuilds the hub's bits in its CTA's slot)
constexpr int64_t kTcHubChunk = 4096;
__global__ void __launch_bounds__(256)
    k_tc_hubs(const int64_t* __restrict__ orow, const int32_t* __restrict__ ocol,
              const int32_t* __restrict__ hub_of, const int64_t* __restrict__ j0s,
              const int64_t* __restrict__ j1s, int64_t nitems, uint32_t* __restrict__ bitmaps,
              int64_t words, int32_t* __restrict__ counts, unsigned long long* __restrict__ total,
              unsigned long long* __restrict__ cursor) {
  __shared__ long long s_h;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  uint32_t* bm = bitmaps + (int64_t)blockIdx.x * words;
  unsigned long long sum = 0;
  for (;;) {
    if (threadIdx.x == 0) s_h = (long long)atomicAdd(cursor, 1ull);
    __syncthreads();
    const int64_t h = s_h;
    __syncthreads();
    if (h >= nitems) break;
    const int32_t u = hub_of[h];
    const int64_t ub = orow[u], ue = orow[u + 1];
    for (int64_t p = ub + threadIdx.x; p < ue; p += blockDim.x) {
      const int32_t x = ocol[p];
      atomicOr(&bm[x >> 5], 1u << (x & 31));
    }
    __syncthreads();
    for (int64_t j = j0s[h] + warp; j < j1s[h]; j += nwarp) {
      const int32_t v = ocol[j];
      const int64_t vb = orow[v], ve = orow[v + 1];
      int c = 0;
      for (int64_t p = vb + lane; p < ve; p += 32) {
        const int32_t w = ocol[p];
        c += (__ldcg(&bm[w >> 5]) >> (w & 31)) & 1u;  // L2: the bits were set by atomics
      }
      for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
      if (lane == 0) {
        counts[j] = c;
        sum += (unsigned long long)c;
      }
    }
    __syncthreads();
    for (int64_t p = ub + threadIdx.x; p < ue; p += blockDim.x) bm[ocol[p] >> 5] = 0u;
    __syncthreads();
  }
  sum = warp_sum_u64(sum);
  if (lane == 0 && sum) atomicAdd(total, sum);
}

int intersect_pairs(gfx_graph* g, const int32_t* us, const int32_t* vs, int64_t npairs,
                    const int64_t* rows, const int32_t* cols, int32_t* counts, int64_t* total) {
  gfx_ctx* ctx = g->ctx;
  int32_t* heavy = nullptr;
  GFX_TRY(scratch_t(g, "tc_heavy", npairs + 1, &heavy));
  Counters* C = g->counters + 3;
  GFX_CK(cudaMemsetAsync(C, 0, sizeof(Counters), ctx->stream));
  const int grid = ctx->sm_count * 8;
  GFX_LAUNCH(k_tc_small, grid_for(npairs, 256, grid), 256, 0, ctx->stream, us, vs, npairs, rows,
             cols, counts, heavy, &C->aux0, &C->total);
  GFX_LAUNCH(k_tc_heavy, grid, 256, 0, ctx->stream, us, vs, heavy, &C->aux0, rows, cols, counts,
             &C->total);
  GFX_CK(cudaGetLastError());
  auto* pin = static_cast<Counters*>(ctx->pinned);
  GFX_CK(cudaMemcpyAsync(pin, C, sizeof(Counters), cudaMemcpyDeviceToHost, ctx->stream));
  GFX_CK(cudaStreamSynchronize(ctx->stream));
  *total = (int64_t)pin->total;
  return GFX_OK;
}

// reversed-orientation build: (dst << 32 | src) keys of the oriented slots
__global__ void k_tc_rev_keys(const int32_t* __restrict__ osrc, const int32_t* __restrict__ ocol,
                              int64_t mo, unsigned long long* __restrict__ keys,
                              int32_t* __restrict__ slot, int64_t* __restrict__ rcnt) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < mo;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int32_t d = ocol[j];
    keys[j] = ((unsigned long long)(uint32_t)d << 32) | (uint32_t)osrc[j];
    slot[j] = (int32_t)j;
    atomicAdd(reinterpret_cast<unsigned long long*>(&rcnt[d]), 1ull);
  }
}

__global__ void k_tc_rev_split(const unsigned long long* __restrict__ keys, int64_t mo,
                               int32_t* __restrict__ rsrc, int32_t* __restrict__ rcol) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < mo;
       j += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long k = keys[j];
    rsrc[j] = (int32_t)(k >> 32);
    rcol[j] = (int32_t)(uint32_t)k;
  }
}

__device__ __forceinline__ int64_t lower_bound_i32(const int32_t* __restrict__ a, int64_t lo,
                                                   int64_t hi, int32_t v) {
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (a[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// reversed edge x => y: common elements z of rows x and y; each credits the
// reference slot of z -> y (xslot of (y => z)).  Short pairs (both rows
// together <= kRevShort) are merged by one thread; longer ones are appended
// to a list that k_tc_rev_heavy takes a warp per pair.
constexpr int kRevShort = 64;

__global__ void __launch_bounds__(256)
    k_tc_rev_count(const int32_t* __restrict__ rsrc, const int32_t* __restrict__ rcol, int64_t mo,
                   const int64_t* __restrict__ rrow, const int32_t* __restrict__ xslot,
                   int32_t* __restrict__ counts, unsigned long long* __restrict__ total,
                   int32_t* __restrict__ heavy, unsigned long long* __restrict__ nheavy) {
  const int lane = threadIdx.x & 31;
  unsigned long long local = 0;
  for (int64_t base = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) & ~31ll; base < mo;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = base + lane;
    bool is_heavy = false;
    if (p < mo) {
      const int32_t x = rsrc[p], y = rcol[p];
      int64_t i = rrow[x];
      const int64_t ie = rrow[x + 1];
      int64_t j = rrow[y];
      const int64_t je = rrow[y + 1];
      if (j < je) {
        if ((ie - i) + (je - j) > kRevShort) {
          is_heavy = true;
        } else {
          int32_t a = rcol[i], b = rcol[j];
          for (;;) {
            if (a < b) {
              if (++i == ie) break;
              a = rcol[i];
            } else if (a > b) {
              if (++j == je) break;
              b = rcol[j];
            } else {
              atomicAdd(&counts[xslot[j]], 1);
              ++local;
              if (++i == ie || ++j == je) break;
              a = rcol[i];
              b = rcol[j];
            }
          }
        }
      }
    }
    const unsigned hm = __ballot_sync(0xffffffffu, is_heavy);
    if (hm) {
      unsigned long long at = 0;
      if (lane == 0) at = atomicAdd(nheavy, (unsigned long long)__popc(hm));
      at = __shfl_sync(0xffffffffu, at, 0);
      if (is_heavy) heavy[at + __popc(hm & ((1u << lane) - 1))] = (int32_t)p;
    }
  }
  for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
  if (lane == 0 && local) atomicAdd(total, local);
}

// warp per heavy pair.  Rows of similar length: a warp-wide merge, 32
// elements of each row per step -- every lane locates its element of x's
// chunk in y's chunk with a 5-step binary search over shuffles, and the
// chunk with the smaller last element advances.  Very uneven rows (one more
// than kRevSkew times the other): lanes take elements of the shorter row
// and binary-search them in the longer one.
constexpr int kRevSkew = 2;
constexpr int64_t kRevGrab = 16;  // heavy pairs per dynamic hand-out

__global__ void __launch_bounds__(256)
    k_tc_rev_heavy(const int32_t* __restrict__ rsrc, const int32_t* __restrict__ rcol,
                   const int64_t* __restrict__ rrow, const int32_t* __restrict__ xslot,
                   const int32_t* __restrict__ heavy, const unsigned long long* __restrict__ nheavy,
                   int32_t* __restrict__ counts, unsigned long long* __restrict__ total,
                   int skew, unsigned long long* __restrict__ grab, int64_t grab_chunk) {
  const int lane = threadIdx.x & 31;
  const int64_t nh = (int64_t)*nheavy;
  unsigned long long local = 0;
  // pairs handed out dynamically in chunks of kRevGrab (their costs vary
  // by orders of magnitude; one counter update per chunk)
  int64_t w = 0, wend = 0;
  for (;;) {
    if (w == wend) {
      if (lane == 0) w = (int64_t)atomicAdd(grab, (unsigned long long)grab_chunk);
      w = __shfl_sync(0xffffffffu, w, 0);
      wend = min(w + grab_chunk, nh);
    }
    if (w >= nh) break;
    const int64_t p = heavy[w];
    const int32_t x = rsrc[p], y = rcol[p];
    const int64_t i0 = rrow[x], ie = rrow[x + 1], j0 = rrow[y], je = rrow[y + 1];
    const int64_t la = ie - i0, lb = je - j0;
    if (la > skew * lb || lb > skew * la) {
      // (each lane's elements increase, so its search starts where the
      // previous one ended)
      if (la <= lb) {  // elements of x searched in y's row
        int64_t jl = j0;
        for (int64_t i = i0 + lane; i < ie; i += 32) {
          const int32_t z = rcol[i];
          jl = lower_bound_i32(rcol, jl, je, z);
          if (jl == je) break;
          if (rcol[jl] == z) {
            atomicAdd(&counts[xslot[jl]], 1);
            ++local;
          }
        }
      } else {  // elements of y searched in x's row
        int64_t il = i0;
        for (int64_t j = j0 + lane; j < je; j += 32) {
          const int32_t z = rcol[j];
          il = lower_bound_i32(rcol, il, ie, z);
          if (il == ie) break;
          if (rcol[il] == z) {
            atomicAdd(&counts[xslot[j]], 1);
            ++local;
          }
        }
      }
      ++w;
      continue;
    }
    int64_t i = i0, j = j0;
    // the next chunk of each row is loaded one step ahead: a step's loads
    // are in flight while the previous step's chunks are compared (s22:
    // 100-102 -> 96-98 ms; the kernel is issue-bound at 85 % SM throughput)
    int32_t a_nx = i + lane < ie ? rcol[i + lane] : 0x7fffffff;
    int32_t b_nx = j + lane < je ? rcol[j + lane] : 0x7fffffff;
    int32_t a2 = i + 32 + lane < ie ? rcol[i + 32 + lane] : 0x7fffffff;
    int32_t b2 = j + 32 + lane < je ? rcol[j + 32 + lane] : 0x7fffffff;
    while (i < ie && j < je) {  // warp-uniform
      const bool va = i + lane < ie, vb = j + lane < je;
      const int32_t a = a_nx, b = b_nx;
      const int32_t amax = __shfl_sync(0xffffffffu, a, (int)min((int64_t)31, ie - i - 1));
      const int32_t bmax = __shfl_sync(0xffffffffu, b, (int)min((int64_t)31, je - j - 1));
      int lo = 0;
#pragma unroll
      for (int step = 16; step > 0; step >>= 1) {  // first lane of b's chunk with b >= a
        const int32_t bm = __shfl_sync(0xffffffffu, b, lo + step - 1);
        if (bm < a) lo += step;
      }
      const int32_t bv = __shfl_sync(0xffffffffu, b, lo & 31);
      if (va && lo < 32 && bv == a && j + lo < je) {
        atomicAdd(&counts[xslot[j + lo]], 1);
        ++local;
      }
      if (amax <= bmax) {
        i += 32;
        a_nx = a2;
        a2 = i + 32 + lane < ie ? rcol[i + 32 + lane] : 0x7fffffff;
      }
      if (bmax <= amax) {
        j += 32;
        b_nx = b2;
        b2 = j + 32 + lane < je ? rcol[j + 32 + lane] : 0x7fffffff;
      }
    }
    ++w;
  }
  for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
  if (lane == 0 && local) atomicAdd(total, local);
}

// reversed CSR of the oriented graph + slot map (graph constant, cached)
static int build_reverse(gfx_graph* g, int64_t mo) {
  gfx_ctx* ctx = g->ctx;
  const int64_t n = g->n;
  int64_t *rcnt, *rrow;
  int32_t *rsrc, *rcol, *xslot;
  GFX_TRY(scratch_t(g, "tc_rcnt", n + 1, &rcnt));
  GFX_TRY(scratch_t(g, "tc_rrow", n + 1, &rrow));
  GFX_TRY(scratch_t(g, "tc_rsrc", mo + 1, &rsrc));
  GFX_TRY(scratch_t(g, "tc_rcol", mo + 1, &rcol));
  GFX_TRY(scratch_t(g, "tc_xslot", mo + 1, &xslot));
  const int32_t* osrc = static_cast<const int32_t*>(g->scratch["tc_osrc"].ptr);
  const int32_t* ocol = static_cast<const int32_t*>(g->scratch["tc_ocol"].ptr);
  unsigned long long *k0 = nullptr, *k1 = nullptr;
  int32_t* v0 = nullptr;
  void* tmp = nullptr;
  size_t tb = 0;
  int end_bit = 32;
  while (end_bit < 64 && (1ll << (end_bit - 32)) < n) ++end_bit;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, k0, k1, v0, xslot, mo, 0, end_bit, ctx->stream);
  GFX_CK(cudaMallocAsync(&k0, (mo + 1) * 8, ctx->stream));
  GFX_CK(cudaMallocAsync(&k1, (mo + 1) * 8, ctx->stream));
  GFX_CK(cudaMallocAsync(&v0, (mo + 1) * 4, ctx->stream));
  GFX_CK(cudaMallocAsync(&tmp, tb + 16, ctx->stream));
  GFX_CK(cudaMemsetAsync(rcnt, 0, (n + 1) * 8, ctx->stream));
  const int grid = grid_for(mo, 256, ctx->sm_count * 16);
  GFX_LAUNCH(k_tc_rev_keys, grid, 256, 0, ctx->stream, osrc, ocol, mo, k0, v0, rcnt);
  cub::DeviceRadixSort::SortPairs(tmp, tb, k0, k1, v0, xslot, mo, 0, end_bit, ctx->stream);
  GFX_LAUNCH(k_tc_rev_split, grid, 256, 0, ctx->stream, k1, mo, rsrc, rcol);
  size_t sb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, sb, rcnt, rrow, n + 1, ctx->stream);
  void* stmp = nullptr;
  GFX_TRY(scratch(g, "tc_scan_tmp2", sb, &stmp));
  cub::DeviceScan::ExclusiveSum(stmp, sb, rcnt, rrow, n + 1, ctx->stream);
  GFX_CK(cudaFreeAsync(k0, ctx->stream));
  GFX_CK(cudaFreeAsync(k1, ctx->stream));
  GFX_CK(cudaFreeAsync(v0, ctx->stream));
  GFX_CK(cudaFreeAsync(tmp, ctx->stream));
  GFX_CK(cudaGetLastError());
  GFX_CK(cudaStreamSynchronize(ctx->stream));
  return GFX_OK;
}

}  // namespace gfx

using namespace gfx;

extern "C" int gfx_tc_orient(gfx_graph* g, int64_t* m_oriented) {
  GFX_NVTX("gfx_tc_orient");
  GFX_REQUIRE(g && m_oriented, "gfx_tc_orient: null argument");
  GFX_REQUIRE(g->flags & GFX_GRAPH_UNDIRECTED, "tc expects a canonical undirected graph");
  gfx_ctx* ctx = g->ctx;
  GFX_CK(cudaSetDevice(ctx->device));
  if (g->m_oriented >= 0) {  // graph constant, already built (gfx_graph_refresh resets it)
    *m_oriented = g->m_oriented;
    return GFX_OK;
  }
  const int64_t n = g->n;
  int64_t *ocnt, *orow;
  int32_t *ocol, *osrc;
  GFX_TRY(scratch_t(g, "tc_ocnt", n + 1, &ocnt));
  GFX_TRY(scratch_t(g, "tc_orow", n + 1, &orow));
  const int grid = grid_for(n, 256, ctx->sm_count * 16);
  GFX_LAUNCH((k_tc_orient<false>), grid, 256, 0, ctx->stream, g->row, g->col, n, ocnt, nullptr,
             nullptr, nullptr);
  GFX_CK(cudaMemsetAsync(ocnt + n, 0, 8, ctx->stream));
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, ocnt, orow, n + 1, ctx->stream);
  void* tmp = nullptr;
  GFX_TRY(scratch(g, "tc_scan_tmp", tb, &tmp));
  cub::DeviceScan::ExclusiveSum(tmp, tb, ocnt, orow, n + 1, ctx->stream);
  int64_t mo = 0;
  GFX_CK(cudaMemcpyAsync(&mo, orow + n, 8, cudaMemcpyDeviceToHost, ctx->stream));
  GFX_CK(cudaStreamSynchronize(ctx->stream));
  GFX_TRY(scratch_t(g, "tc_ocol", mo + 1, &ocol));
  GFX_TRY(scratch_t(g, "tc_osrc", mo + 1, &osrc));
  GFX_LAUNCH((k_tc_orient<true>), grid, 256, 0, ctx->stream, g->row, g->col, n, nullptr, orow,
             ocol, osrc);
  GFX_CK(cudaGetLastError());
  GFX_CK(cudaStreamSynchronize(ctx->stream));
  if (mo > 0) GFX_TRY(build_reverse(g, mo));
  g->m_oriented = mo;
  *m_oriented = mo;
  return GFX_OK;
}

extern "C" int gfx_tc_count(gfx_graph* g, int32_t* osrc_d, int32_t* odst_d, int32_t* counts_d,
                            int64_t* total, gfx_stats* stats) {
  GFX_NVTX("gfx_tc_count");
  GFX_REQUIRE(g && total, "gfx_tc_count: null argument");
  GFX_REQUIRE(g->m_oriented >= 0, "gfx_tc_count: call gfx_tc_orient first");
  gfx_ctx* ctx = g->ctx;
  GFX_CK(cudaSetDevice(ctx->device));
  const int64_t mo = g->m_oriented;
  int64_t* orow = static_cast<int64_t*>(g->scratch["tc_orow"].ptr);
  int32_t* ocol = static_cast<int32_t*>(g->scratch["tc_ocol"].ptr);
  int32_t* osrc = static_cast<int32_t*>(g->scratch["tc_osrc"].ptr);
  int32_t* counts = counts_d;
  if (!counts) GFX_TRY(scratch_t(g, "tc_counts", mo + 1, &counts));
  if (!getenv("GFX_TC_LEGACY")) {
    Counters* C = g->counters + 3;
    GFX_CK(cudaEventRecord(ctx->ev0, ctx->stream));
    GFX_CK(cudaMemsetAsync(C, 0, sizeof(Counters), ctx->stream));
    GFX_CK(cudaMemsetAsync(counts, 0, (mo + 1) * 4, ctx->stream));
    if (mo > 0) {
      auto* rrow = static_cast<const int64_t*>(g->scratch["tc_rrow"].ptr);
      auto* rsrc = static_cast<const int32_t*>(g->scratch["tc_rsrc"].ptr);
      auto* rcol = static_cast<const int32_t*>(g->scratch["tc_rcol"].ptr);
      auto* xslot = static_cast<const int32_t*>(g->scratch["tc_xslot"].ptr);
      int32_t* heavy = nullptr;
      GFX_TRY(scratch_t(g, "tc_heavy", mo + 1, &heavy));
      GFX_LAUNCH(k_tc_rev_count, grid_for(mo, 256, ctx->sm_count * 8), 256, 0, ctx->stream, rsrc,
                 rcol, mo, rrow, xslot, counts, &C->total, heavy, &C->aux0);
      const int skew = getenv("GFX_TC_SKEW") ? atoi(getenv("GFX_TC_SKEW")) : kRevSkew;
      const int64_t grab = getenv("GFX_TC_GRAB") ? atoi(getenv("GFX_TC_GRAB")) : kRevGrab;
      GFX_LAUNCH(k_tc_rev_heavy, ctx->sm_count * 8, 256, 0, ctx->stream, rsrc, rcol, rrow, xslot,
                 heavy, &C->aux0, counts, &C->total, skew, &C->aux1, grab);
    }
    GFX_CK(cudaGetLastError());
    GFX_CK(cudaEventRecord(ctx->ev1, ctx->stream));
    auto* pin = static_cast<Counters*>(ctx->pinned);
    GFX_CK(cudaMemcpyAsync(pin, C, sizeof(Counters), cudaMemcpyDeviceToHost, ctx->stream));
    GFX_CK(cudaStreamSynchronize(ctx->stream));
    *total = (int64_t)pin->total;
    if (osrc_d)
      GFX_CK(cudaMemcpyAsync(osrc_d, osrc, mo * 4, cudaMemcpyDeviceToDevice, ctx->stream));
    if (odst_d)
      GFX_CK(cudaMemcpyAsync(odst_d, ocol, mo * 4, cudaMemcpyDeviceToDevice, ctx->stream));
    GFX_CK(cudaStreamSynchronize(ctx->stream));
    float ms = 0.f;
    GFX_CK(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
    if (stats) {
      *stats = gfx_stats{};
      stats->iterations = 1;
      stats->device_ms = ms;
    }
    return GFX_OK;
  }
  // legacy: hub rows first (bitmap counting), then every other pair
  int32_t *hubs = nullptr, *heavy = nullptr;
  GFX_TRY(scratch_t(g, "tc_hubs", g->n + 1, &hubs));
  GFX_TRY(scratch_t(g, "tc_heavy", mo + 1, &heavy));
  const int hub_ctas = ctx->sm_count;
  uint32_t* bitmaps = nullptr;
  GFX_TRY(scratch_t(g, "tc_hub_bm", (size_t)hub_ctas * g->words, &bitmaps));
  Counters* C = g->counters + 3;
  GFX_CK(cudaEventRecord(ctx->ev0, ctx->stream));
  GFX_CK(cudaMemsetAsync(C, 0, sizeof(Counters), ctx->stream));
  GFX_CK(cudaMemsetAsync(bitmaps, 0, (size_t)hub_ctas * g->words * 4, ctx->stream));
  GFX_LAUNCH(k_tc_hub_list, grid_for(g->n, 256, ctx->sm_count * 8), 256, 0, ctx->stream, orow,
             g->n, hubs, &C->aux2);
  {
    // items: each hub's pairs in chunks of kTcHubChunk (host-built, small)
    auto* pin = static_cast<Counters*>(ctx->pinned);
    GFX_CK(cudaMemcpyAsync(pin, C, sizeof(Counters), cudaMemcpyDeviceToHost, ctx->stream));
    GFX_CK(cudaStreamSynchronize(ctx->stream));
    const int64_t nh = (int64_t)pin->aux2;
    std::vector<int32_t> hh((size_t)nh);
    std::vector<int64_t> rows((size_t)g->n + 1);
    if (nh) {
      GFX_CK(cudaMemcpy(hh.data(), hubs, nh * 4, cudaMemcpyDeviceToHost));
      GFX_CK(cudaMemcpy(rows.data(), orow, (g->n + 1) * 8, cudaMemcpyDeviceToHost));
    }
    std::vector<int32_t> item_hub;
    std::vector<int64_t> item_j0, item_j1;
    for (int32_t u : hh)
      for (int64_t j = rows[u]; j < rows[u + 1]; j += kTcHubChunk) {
        item_hub.push_back(u);
        item_j0.push_back(j);
        item_j1.push_back(std::min(j + kTcHubChunk, rows[u + 1]));
      }
    const int64_t ni = (int64_t)item_hub.size();
    if (ni) {
      int32_t* ih = nullptr;
      int64_t *ij0 = nullptr, *ij1 = nullptr;
      GFX_TRY(scratch_t(g, "tc_item_hub", ni, &ih));
      GFX_TRY(scratch_t(g, "tc_item_j0", ni, &ij0));
      GFX_TRY(scratch_t(g, "tc_item_j1", ni, &ij1));
      GFX_CK(cudaMemcpyAsync(ih, item_hub.data(), ni * 4, cudaMemcpyHostToDevice, ctx->stream));
      GFX_CK(cudaMemcpyAsync(ij0, item_j0.data(), ni * 8, cudaMemcpyHostToDevice, ctx->stream));
      GFX_CK(cudaMemcpyAsync(ij1, item_j1.data(), ni * 8, cudaMemcpyHostToDevice, ctx->stream));
      GFX_LAUNCH(k_tc_hubs, hub_ctas, 256, 0, ctx->stream, orow, ocol, ih, ij0, ij1, ni, bitmaps,
                 g->words, counts, &C->total, &C->aux3);
      GFX_CK(cudaStreamSynchronize(ctx->stream));  // host item vectors go out of scope
    }
  }
  const int grid = ctx->sm_count * 8;
  GFX_LAUNCH(k_tc_small, grid_for(mo, 256, grid), 256, 0, ctx->stream, osrc, ocol, mo, orow, ocol,
             counts, heavy, &C->aux0, &C->total, kTcHub);
  GFX_LAUNCH(k_tc_heavy, grid, 256, 0, ctx->stream, osrc, ocol, heavy, &C->aux0, orow, ocol,
             counts, &C->total);
  GFX_CK(cudaGetLastError());
  GFX_CK(cudaEventRecord(ctx->ev1, ctx->stream));
  {
    auto* pin = static_cast<Counters*>(ctx->pinned);
    GFX_CK(cudaMemcpyAsync(pin, C, sizeof(Counters), cudaMemcpyDeviceToHost, ctx->stream));
    GFX_CK(cudaStreamSynchronize(ctx->stream));
    *total = (int64_t)pin->total;
  }
  if (osrc_d)
    GFX_CK(cudaMemcpyAsync(osrc_d, osrc, mo * 4, cudaMemcpyDeviceToDevice, ctx->stream));
  if (odst_d)
    GFX_CK(cudaMemcpyAsync(odst_d, ocol, mo * 4, cudaMemcpyDeviceToDevice, ctx->stream));
  GFX_CK(cudaStreamSynchronize(ctx->stream));
  float ms = 0.f;
  GFX_CK(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
  if (stats) {
    *stats = gfx_stats{};
    stats->iterations = 1;
    stats->device_ms = ms;
  }
  return GFX_OK;
}

extern "C" int gfx_segmented_intersect(gfx_graph* g, const int32_t* u_d, const int32_t* v_d,
                                       int64_t num_pairs, int32_t* counts_d, int64_t* total) {
  GFX_NVTX("gfx_segmented_intersect");
  GFX_REQUIRE(g && total && (num_pairs == 0 || (u_d && v_d && counts_d)),
              "gfx_segmented_intersect: null argument");
  GFX_CK(cudaSetDevice(g->ctx->device));
  if (num_pairs == 0) {
    *total = 0;
    return GFX_OK;
  }
  return intersect_pairs(g, u_d, v_d, num_pairs, g->row, g->col, counts_d, total);
}
