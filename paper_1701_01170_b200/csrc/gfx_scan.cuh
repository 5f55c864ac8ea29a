// Fused degree scan + LB tile partition: one decoupled look-back tile.
//
// Replaces reference load_balance.py:105-113 (compute_scan_offsets) and
// load_balance.py:157-176 (plan_lb_output: ceil(total/N) chunks of N output
// slots, each chunk's first source found by searchsorted).  Here the
// partition falls out of the scan: the item whose units cover k*kTile writes
// part[k] directly, so no search is needed.  Units: every item weighs
// kItemUnits plus its degree (merge-path over items and slots), so a tile
// holds at most kTile slots AND about kTile/kItemUnits items.
// Tile status word: [63:62] flag (1 aggregate, 2 inclusive prefix),
// [61:48] epoch tag, [47:0] value.  Used by the standalone scan kernel
// (dynamic tile ids) and by the persistent BFS kernel (static tile ids; all
// CTAs co-resident, so the look-back always makes progress).
#pragma once

#include "gfx_device.cuh"
#include "gfx_internal.cuh"

namespace gfx {

constexpr unsigned long long kFlagAgg = 1ull << 62;
constexpr unsigned long long kFlagPre = 2ull << 62;
constexpr unsigned long long kValMask = (1ull << 48) - 1;

__device__ __forceinline__ unsigned long long pack_status(unsigned long long flag, unsigned epoch,
                                                          unsigned long long v) {
  return flag | ((unsigned long long)(epoch & 0x3FFF) << 48) | (v & kValMask);
}

constexpr int kLongFill = 16;  // items owning more tiles than this are filled by the whole block
struct ScanSmem {
  int64_t warp[kScanBlock / 32];
  int64_t prefix;
  int64_t lk0[kLongFill], lk1[kLongFill];  // long partition ranges [k0, k1] of item li
  int32_t li[kLongFill];
  int nlong;
};

// one tile of kScanTileItems frontier items (blockDim == kScanBlock)
__device__ __forceinline__ void scan_tile(int64_t tile, int64_t ntiles,
                                          const int32_t* __restrict__ F, int64_t nf,
                                          const int64_t* __restrict__ row,
                                          int64_t* __restrict__ scan,
                                          int64_t* __restrict__ rowbase,
                                          int32_t* __restrict__ part, unsigned long long* status,
                                          unsigned ep, Counters* __restrict__ ctr, ScanSmem& sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) sm.nlong = 0;
  const int64_t base = tile * kScanTileItems + (int64_t)threadIdx.x * kScanItems;
  int64_t deg[kScanItems];
  int64_t rb[kScanItems];
  int64_t tsum = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int64_t i = base + k;
    deg[k] = 0;
    rb[k] = 0;
    if (i < nf) {
      const int32_t v = F[i];
      const int64_t a = row[v], b = row[v + 1];
      rb[k] = a;
      deg[k] = b - a;
    }
    tsum += deg[k];
  }
  // block exclusive scan of per-thread sums
  int64_t incl = tsum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) sm.warp[warp] = incl;
  __syncthreads();
  int64_t warp_off = 0, agg = 0;
#pragma unroll
  for (int w = 0; w < kScanBlock / 32; ++w) {
    const int64_t x = sm.warp[w];
    if (w < warp) warp_off += x;
    agg += x;
  }
  // decoupled look-back (warp 0)
  if (warp == 0) {
    int64_t excl = 0;
    if (tile == 0) {
      if (lane == 0) atomicExch(&status[0], pack_status(kFlagPre, ep, (unsigned long long)agg));
    } else {
      if (lane == 0) atomicExch(&status[tile], pack_status(kFlagAgg, ep, (unsigned long long)agg));
      int64_t pred = tile - 1;
      for (;;) {
        const int64_t idx = pred - lane;
        unsigned long long s = 0;
        unsigned flag = 0;
        if (idx >= 0) {
          do {
            s = ld_volatile_u64(&status[idx]);
            flag = (unsigned)(s >> 62);
            if (((s >> 48) & 0x3FFF) != (ep & 0x3FFF)) flag = 0;
          } while (flag == 0);
        } else {
          flag = 2;  // virtual prefix of zero before tile 0
          s = 0;
        }
        const unsigned pre_mask = __ballot_sync(0xffffffffu, flag == 2);
        int64_t val = (int64_t)(s & kValMask);
        if (pre_mask) {
          const int first = __ffs(pre_mask) - 1;
          if (lane > first) val = 0;
          excl += warp_sum_i64(val);
          break;
        }
        excl += warp_sum_i64(val);
        pred -= 32;
      }
      if (lane == 0)
        atomicExch(&status[tile], pack_status(kFlagPre, ep, (unsigned long long)(excl + agg)));
    }
    if (lane == 0) sm.prefix = excl;
  }
  __syncthreads();
  int64_t run = sm.prefix + warp_off + incl - tsum;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    const int64_t i = base + k;
    if (i < nf) {
      scan[i] = run;
      rowbase[i] = rb[k];
      // item i occupies units [ub, ub + kItemUnits + deg) of the merged
      // (items + slots) sequence; it owns every tile starting inside them
      const int64_t ub = run + (int64_t)kItemUnits * i;
      const int64_t k0 = (ub + kTile - 1) / kTile;
      const int64_t k1 = (ub + kItemUnits + deg[k] - 1) / kTile;
      int slot = -1;
      if (k1 - k0 >= kLongFill) {  // a hub: the block fills its range below
        slot = atomicAdd(&sm.nlong, 1);
        if (slot < kLongFill) {
          sm.lk0[slot] = k0;
          sm.lk1[slot] = k1;
          sm.li[slot] = (int32_t)i;
        }
      }
      if (slot < 0 || slot >= kLongFill)
        for (int64_t t = k0; t <= k1; ++t) part[t] = (int32_t)i;
    }
    run += deg[k];
  }
  __syncthreads();
  for (int j = 0; j < min(sm.nlong, kLongFill); ++j)
    for (int64_t t = sm.lk0[j] + threadIdx.x; t <= sm.lk1[j]; t += kScanBlock) part[t] = sm.li[j];
  if (tile == ntiles - 1 && threadIdx.x == kScanBlock - 1) {
    // the last thread of the last tile holds the grand total
    scan[nf] = run;
    ctr->total = (unsigned long long)run;
    const int64_t units = run + (int64_t)kItemUnits * nf;
    ctr->ntiles = (unsigned long long)((units + kTile - 1) / kTile);
  }
  __syncthreads();
}

}  // namespace gfx
