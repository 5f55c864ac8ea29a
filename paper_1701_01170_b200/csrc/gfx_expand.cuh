// Load-balanced push expansion (the device `advance`), warp-centric.
//
// Reference semantics: operators.py:218-266 (advance, push) with the LB plan
// of load_balance.py:157-176.  The fused degree scan (gfx_scan.cuh) cuts the
// frontier's expansion into tiles of kTile = 512 consecutive OUTPUT slots and
// records the item owning each tile's first slot, so hub vertices are split
// across many tiles and every tile is the same amount of work.
//
// One WARP owns one tile at a time -- no CTA barriers anywhere:
//   items : lanes load up to 32 overlapping items (scan, delta = row[v] -
//           scan, v) into the warp's shared-memory slice and mark each
//           item's first slot;
//   owner : chunks whose items average >= kItemModeSlots slots are walked
//           item by item (no lookup); otherwise a warp-wide inclusive
//           max-scan over the markers (16 per lane + shuffles) gives every
//           slot its owning item;
//   visit : lane l handles slots l, l+32, ... -- consecutive lanes read
//           consecutive column ids (coalesced) -- with Op::kBatch column
//           loads in flight per lane before the functor runs;
//   emit  : survivors are compacted with ballot/popc into the warp's
//           shared-memory staging buffer and appended to the global queue
//           with ONE atomicAdd per flush (frontier queues in shared-memory
//           staged buffers).
//
// Functor interface (gfx_bfs.cu / gfx_sssp.cu / gfx_cc.cu / gfx_operators.cu):
//   static constexpr bool kWeights;    load w[e]
//   static constexpr bool kSrcVal;     per-item src_value(v)
//   static constexpr bool kEmitEdge;   emit edge ids instead of dst ids
//   static constexpr int  kBatch;      slots in flight per lane (divides 16)
//   static constexpr int  kMinBlocks;  CTAs per SM the register budget targets
//   __device__ int32_t src_value(int32_t v) const;
//   __device__ void prefetch(const int32_t* d);       // d[kBatch]
//   __device__ bool visit(int u, int32_t dst, int32_t src, int32_t w,
//                         int32_t sval, int64_t edge);  // u = prefetch slot
#pragma once

#include <type_traits>

#include "gfx_device.cuh"
#include "gfx_internal.cuh"

namespace gfx {

// element type of the weight stream an Op reads (Op::WeightT, default int32)
template <class Op, class = void>
struct WeightOf {
  using T = int32_t;
};
template <class Op>
struct WeightOf<Op, std::void_t<typename Op::WeightT>> {
  using T = typename Op::WeightT;
};
template <class T>
__device__ __forceinline__ int32_t ld_weight(const T* p, unsigned long long pol);
template <>
__device__ __forceinline__ int32_t ld_weight<int32_t>(const int32_t* p, unsigned long long pol) {
  return ld_stream_i32(p, pol);
}
template <>
__device__ __forceinline__ int32_t ld_weight<uint8_t>(const uint8_t* p, unsigned long long pol) {
  unsigned short v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u8 %0, [%1], %2;"
               : "=h"(v)
               : "l"(p), "l"(pol));
  return (int32_t)v;
}

// Op::kPipeline (default false): software-pipelined adjacency loads in the
// expansion (measured: BFS claims gain, the SSSP relax loses to spills)
template <class Op, class = void>
struct PipelineOf {
  static constexpr bool value = false;
};
template <class Op>
struct PipelineOf<Op, std::void_t<decltype(Op::kPipeline)>> {
  static constexpr bool value = Op::kPipeline;
};

constexpr int kExpandBlock = 256;
constexpr int kWarpsPerBlock = kExpandBlock / 32;
constexpr int kLaneSlots = kTile / 32;  // 16 slots per lane per tile
constexpr int kOutCap = 640;            // per-warp staged output (flushed past kOutCap - 32*kBatch)
constexpr int kVisitBatch = 8;          // default Op::kBatch
constexpr int kItemModeSlots = 128;     // chunks averaging >= this many slots per item walk items

struct WarpSmem {
  int64_t delta[32];     // row[v] - scan[i]: col index = delta + global slot
  int32_t src[32];
  int32_t sval[32];
  int8_t owner[kTile];   // slot -> item lane (within the 32-item chunk)
  int32_t obuf[kOutCap];
};

__device__ __forceinline__ WarpSmem& warp_smem(unsigned char* base) {
  return reinterpret_cast<WarpSmem*>(base)[threadIdx.x >> 5];
}

// flush the warp's staged output (count is warp-uniform)
__device__ __forceinline__ void warp_flush(WarpSmem& W, int& ocnt, int32_t* __restrict__ out,
                                           unsigned long long* __restrict__ out_len) {
  const int lane = threadIdx.x & 31;
  if (ocnt == 0) return;
  unsigned long long base = 0;
  if (lane == 0) base = atomicAdd(out_len, (unsigned long long)ocnt);
  base = __shfl_sync(0xffffffffu, base, 0);
  __syncwarp();
  for (int j = lane; j < ocnt; j += 32) out[base + j] = W.obuf[j];
  __syncwarp();
  ocnt = 0;
}

// Per-CTA aggregation of the level counters and queue reservations.  All
// counters of a level share one 64-byte line, so per-warp atomics on them
// serialise in one L2 slice (~3500 warps per level); the persistent loop
// sums per CTA in shared memory and issues one atomic per CTA instead, and
// one thread per CTA reads the counters back after a grid barrier.
struct CtaAgg {
  unsigned long long ctr[8];  // shared mirror of Counters (summed, then flushed)
  unsigned long long rd[8];   // Counters as read after the last grid barrier
  unsigned long long base;
  int woff[kWarpsPerBlock + 1];
};
static_assert(sizeof(Counters) == 8 * sizeof(unsigned long long), "Counters layout");

// every thread of the CTA: add the CTA's sums to the global counters and
// clear them (callers separate this from the next use by a barrier)
__device__ __forceinline__ void cta_flush_ctrs(CtaAgg& g, Counters* cur) {
  __syncthreads();
  if (threadIdx.x < 8) {
    const unsigned long long v = g.ctr[threadIdx.x];
    if (v) atomicAdd(reinterpret_cast<unsigned long long*>(cur) + threadIdx.x, v);
    g.ctr[threadIdx.x] = 0ull;
  }
}

// every thread of the CTA: read the 8 counters once per CTA into g.rd
__device__ __forceinline__ void cta_read_ctrs(CtaAgg& g, const Counters* cur) {
  if (threadIdx.x < 8)
    g.rd[threadIdx.x] =
        ld_volatile_u64(reinterpret_cast<const unsigned long long*>(cur) + threadIdx.x);
  __syncthreads();
}

// every thread of the CTA: append every warp's staged output (ocnt entries
// in W.obuf) to the queue with ONE reservation per CTA
__device__ __forceinline__ void cta_flush(WarpSmem& W, int& ocnt, int32_t* __restrict__ out,
                                          unsigned long long* __restrict__ out_len, CtaAgg& g) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (lane == 0) g.woff[wid + 1] = ocnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    g.woff[0] = 0;
    for (int k = 1; k <= kWarpsPerBlock; ++k) g.woff[k] += g.woff[k - 1];
    const int tot = g.woff[kWarpsPerBlock];
    g.base = tot ? atomicAdd(out_len, (unsigned long long)tot) : 0ull;
  }
  __syncthreads();
  const unsigned long long b = g.base + g.woff[wid];
  for (int j = lane; j < ocnt; j += 32) out[b + j] = W.obuf[j];
  ocnt = 0;
}

// All tiles t = task0, task0 + ntasks, ... of one expansion, processed by the
// calling warp.  Shared by the standalone kernel and the persistent BFS.
template <class Op>
__device__ __forceinline__ void expand_tasks(WarpSmem& W, Op& o, const int32_t* __restrict__ F,
                                             int64_t nf, const int64_t* __restrict__ scan,
                                             const int64_t* __restrict__ rowbase,
                                             const int32_t* __restrict__ part, int64_t ntiles,
                                             int64_t total, const int32_t* __restrict__ col,
                                             const typename WeightOf<Op>::T* __restrict__ wgt,
                                             int32_t* __restrict__ out,
                                             unsigned long long* __restrict__ out_len,
                                             int64_t task0, int64_t ntasks,
                                             CtaAgg* cta = nullptr) {
  // cta: every thread of the CTA calls this (the persistent loops); the last
  // flush then takes one queue reservation per CTA instead of one per warp
  constexpr int B = Op::kBatch;
  const int lane = threadIdx.x & 31;
  const unsigned long long pol = l2_evict_first_policy();
  int ocnt = 0;
  // software pipeline: the next tile's partition entry and first 32 items
  // are loaded while the current tile's column loads are in flight
  int64_t p_i0 = 0, p_i1 = -1, p_sc = 0, p_sc1 = 0, p_rb = 0;
  int32_t p_v = 0;
  auto prefetch_tile = [&](int64_t t) {
    if (t >= ntiles) return;
    p_i0 = part[t];
    p_i1 = (t + 1 < ntiles) ? (int64_t)part[t + 1] : nf - 1;
    const int64_t i = p_i0 + lane;
    if (i <= p_i1) {
      p_sc = scan[i];
      p_sc1 = scan[i + 1];
      p_rb = rowbase[i];
      p_v = F[i];
    }
  };
  prefetch_tile(task0);
  const int64_t units = total + (int64_t)kItemUnits * nf;
  for (int64_t t = task0; t < ntiles; t += ntasks) {
    const int64_t u0 = t * kTile;
    const int64_t u1 = min(u0 + (int64_t)kTile, units);
    const int64_t i0 = p_i0, i1 = p_i1;
    const int64_t f_sc = p_sc, f_sc1 = p_sc1, f_rb = p_rb;
    const int32_t f_v = p_v;
    prefetch_tile(t + ntasks);
    int64_t s0 = 0;  // first slot of the tile (set by the first chunk)
    for (int64_t ib = i0; ib <= i1; ib += 32) {
      const int64_t i = ib + lane;
      const bool valid = i <= i1;
      int64_t sc = 0, sc1 = 0, rb = 0;
      int32_t v = 0;
      if (valid) {
        if (ib == i0) {
          sc = f_sc;
          sc1 = f_sc1;
          rb = f_rb;
          v = f_v;
        } else {
          sc = scan[i];
          sc1 = scan[i + 1];
          rb = rowbase[i];
          v = F[i];
        }
      }
      // clip the item's slots to the tile's unit range
      const int64_t ub = sc + (int64_t)kItemUnits * i + kItemUnits;  // unit of slot sc
      const int64_t deg = sc1 - sc;
      const int64_t lo = sc + min(max(u0 - ub, (int64_t)0), deg);
      const int64_t hi = sc + min(max(u1 - ub, (int64_t)0), deg);
      const bool has = valid && hi > lo;
      if (ib == i0) s0 = __shfl_sync(0xffffffffu, lo, 0);
      // chunk slot range [cl, ch) relative to s0
      const int cl = (int)(__shfl_sync(0xffffffffu, lo, 0) - s0);
      const unsigned vm = __ballot_sync(0xffffffffu, valid);
      const int last = 31 - __clz(vm);
      const int ch = (int)(__shfl_sync(0xffffffffu, hi, last) - s0);
      if (ch <= cl) continue;
      const unsigned hm = __ballot_sync(0xffffffffu, has);
      if ((ch - cl) >= kItemModeSlots * __popc(hm)) {
        // long segments: walk the items one by one, lanes over consecutive
        // slots -- no owner lookup at all (the common case on hub frontiers)
        const int32_t my_sv = (Op::kSrcVal && has) ? o.src_value(v) : 0;
        const int64_t my_del = rb - sc;
        unsigned rem = hm;
        while (rem) {
          const int k = __ffs(rem) - 1;
          rem &= rem - 1;
          const int64_t klo = __shfl_sync(0xffffffffu, lo, k);
          const int64_t khi = __shfl_sync(0xffffffffu, hi, k);
          const int64_t kdel = __shfl_sync(0xffffffffu, my_del, k);
          const int32_t ksrc = __shfl_sync(0xffffffffu, v, k);
          const int32_t ksv = Op::kSrcVal ? __shfl_sync(0xffffffffu, my_sv, k) : 0;
          const int32_t* cbase = col + kdel + klo + lane;
          const typename WeightOf<Op>::T* wbase = Op::kWeights ? wgt + kdel + klo + lane : nullptr;
          const int klen = (int)(khi - klo);
          // Op::kPipeline: two-stage software pipeline -- the next batch's
          // column (and weight) loads are issued before this batch's probes,
          // so the adjacency stream's latency overlaps the probe / claim chain
          constexpr bool kPipe = PipelineOf<Op>::value;
          int32_t dn[B];
          int32_t wn[Op::kWeights ? B : 1];
          if constexpr (kPipe) {
#pragma unroll
            for (int q = 0; q < B; ++q) {
              dn[q] = -1;
              if (Op::kWeights) wn[Op::kWeights ? q : 0] = 0;
              if (q * 32 < klen - lane) {
                dn[q] = ld_stream_i32(cbase + q * 32, pol);
                if (Op::kWeights) wn[Op::kWeights ? q : 0] = ld_weight(wbase + q * 32, pol);
              }
            }
          }
          for (int jb = 0; jb < klen; jb += 32 * B) {
            int32_t d[B];
            int32_t w[Op::kWeights ? B : 1];
            if constexpr (kPipe) {
#pragma unroll
              for (int q = 0; q < B; ++q) {
                d[q] = dn[q];
                if (Op::kWeights) w[Op::kWeights ? q : 0] = wn[Op::kWeights ? q : 0];
              }
              const int lim = klen - (jb + 32 * B) - lane;
#pragma unroll
              for (int q = 0; q < B; ++q) {
                dn[q] = -1;
                if (q * 32 < lim) {
                  dn[q] = ld_stream_i32(cbase + jb + 32 * B + q * 32, pol);
                  if (Op::kWeights)
                    wn[Op::kWeights ? q : 0] = ld_weight(wbase + jb + 32 * B + q * 32, pol);
                }
              }
            } else {
              const int lim = klen - jb - lane;  // this lane's slots remaining
#pragma unroll
              for (int q = 0; q < B; ++q) {
                d[q] = -1;
                if (Op::kWeights) w[Op::kWeights ? q : 0] = 0;
                if (q * 32 < lim) {
                  d[q] = ld_stream_i32(cbase + jb + q * 32, pol);
                  if (Op::kWeights) w[Op::kWeights ? q : 0] = ld_weight(wbase + jb + q * 32, pol);
                }
              }
            }
            o.prefetch(d);
#pragma unroll
            for (int q = 0; q < B; ++q) {
              bool emit = false;
              const int64_t e = Op::kEmitEdge ? kdel + klo + jb + q * 32 + lane : 0;
              if (d[q] >= 0)
                emit = o.visit(q, d[q], ksrc, Op::kWeights ? w[Op::kWeights ? q : 0] : 1, ksv, e);
              const unsigned em = __ballot_sync(0xffffffffu, emit);
              if (emit)
                W.obuf[ocnt + __popc(em & ((1u << lane) - 1))] = Op::kEmitEdge ? (int32_t)e : d[q];
              ocnt += __popc(em);
            }
            if (ocnt > kOutCap - 32 * B) warp_flush(W, ocnt, out, out_len);
          }
        }
        continue;
      }
      __syncwarp();
      for (int j = cl + lane; j < ch; j += 32) W.owner[j] = -1;
      __syncwarp();
      if (has) {
        W.owner[lo - s0] = (int8_t)lane;
        W.delta[lane] = rb - sc;
        W.src[lane] = v;
        if (Op::kSrcVal) W.sval[lane] = o.src_value(v);
      }
      __syncwarp();
      // inclusive max-scan of owner[cl, ch): 16 consecutive entries per lane
      {
        const int base = cl + lane * kLaneSlots;
        int run = -1;
        int8_t loc[kLaneSlots];
#pragma unroll
        for (int k = 0; k < kLaneSlots; ++k) {
          const int j = base + k;
          const int x = j < ch ? W.owner[j] : -1;
          run = x > run ? x : run;
          loc[k] = (int8_t)run;
        }
        int incl = run;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, off);
          if (lane >= off) incl = y > incl ? y : incl;
        }
        int pre = __shfl_up_sync(0xffffffffu, incl, 1);
        if (lane == 0) pre = -1;
        __syncwarp();
#pragma unroll
        for (int k = 0; k < kLaneSlots; ++k) {
          const int j = base + k;
          if (j < ch) W.owner[j] = (int8_t)(loc[k] > pre ? loc[k] : pre);
        }
      }
      __syncwarp();
      // visit in batches of B slots per lane (not pipelined: measured slower,
      // the extra live registers spill)
      for (int jb = cl; jb < ch; jb += 32 * B) {
        int32_t d[B];
        int32_t w[Op::kWeights ? B : 1];
#pragma unroll
        for (int k = 0; k < B; ++k) {
          const int j = jb + k * 32 + lane;
          d[k] = -1;
          if (Op::kWeights) w[Op::kWeights ? k : 0] = 0;
          if (j < ch) {
            const int it = W.owner[j];
            const int64_t e = W.delta[it] + s0 + j;
            d[k] = ld_stream_i32(col + e, pol);
            if (Op::kWeights) w[Op::kWeights ? k : 0] = ld_weight(wgt + e, pol);
          }
        }
        o.prefetch(d);
#pragma unroll
        for (int k = 0; k < B; ++k) {
          const int j = jb + k * 32 + lane;
          bool emit = false;
          int32_t outv = d[k];
          if (d[k] >= 0) {
            const int it = W.owner[j];
            const int64_t e = Op::kEmitEdge ? W.delta[it] + s0 + j : 0;
            emit = o.visit(k, d[k], W.src[it], Op::kWeights ? w[Op::kWeights ? k : 0] : 1,
                           Op::kSrcVal ? W.sval[it] : 0, e);
            if (Op::kEmitEdge) outv = (int32_t)e;
          }
          const unsigned em = __ballot_sync(0xffffffffu, emit);
          if (emit) W.obuf[ocnt + __popc(em & ((1u << lane) - 1))] = outv;
          ocnt += __popc(em);
        }
        if (ocnt > kOutCap - 32 * B) warp_flush(W, ocnt, out, out_len);
      }
    }
  }
  if (cta) cta_flush(W, ocnt, out, out_len, *cta);
  else warp_flush(W, ocnt, out, out_len);
}

// Expansion of at most 32 items held one per lane (v, row base, degree; 0
// for empty lanes) without any scan pass: the degrees are scanned with
// shuffles, the exclusive offsets parked in the warp's shared memory, and
// the slots [c0, c0 + 32 * Op::kBatch) for c0 = chunk0, chunk0 + stride, ...
// expanded by this warp; a slot's item comes from a binary search over the
// <= 32 offsets.  Returns the item set's slot count.  Output and claims as
// expand_tasks (staged in the warp buffer, ocnt carried by the caller).
template <class Op>
__device__ __forceinline__ int64_t expand_items32(WarpSmem& W, Op& o, int32_t v, int64_t rb,
                                                  int64_t deg, const int32_t* __restrict__ col,
                                                  int32_t* __restrict__ out,
                                                  unsigned long long* __restrict__ out_len,
                                                  int& ocnt, int64_t chunk0, int64_t stride) {
  constexpr int B = Op::kBatch;
  const int lane = threadIdx.x & 31;
  int64_t* ex = reinterpret_cast<int64_t*>(W.owner);  // exclusive offsets
  int64_t incl = deg;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, incl, off);
    if (lane >= off) incl += y;
  }
  const int64_t total = __shfl_sync(0xffffffffu, incl, 31);
  __syncwarp();
  ex[lane] = incl - deg;
  W.delta[lane] = rb - (incl - deg);
  W.src[lane] = v;
  __syncwarp();
  const unsigned long long pol = l2_evict_first_policy();
  for (int64_t c0 = chunk0; c0 < total; c0 += stride) {
    int32_t d[B];
    int it[B];
#pragma unroll
    for (int q = 0; q < B; ++q) {
      const int64_t sl = c0 + q * 32 + lane;
      d[q] = -1;
      it[q] = 0;
      if (sl < total) {
        int lo = 0, hi = 31;  // last item with ex[item] <= sl (empty items repeat offsets)
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (ex[mid] <= sl) lo = mid; else hi = mid - 1;
        }
        it[q] = lo;
        d[q] = ld_stream_i32(col + W.delta[lo] + sl, pol);
      }
    }
    o.prefetch(d);
#pragma unroll
    for (int q = 0; q < B; ++q) {
      const bool emit = d[q] >= 0 && o.visit(q, d[q], W.src[it[q]], 1, 0, 0);
      const unsigned em = __ballot_sync(0xffffffffu, emit);
      if (emit) W.obuf[ocnt + __popc(em & ((1u << lane) - 1))] = d[q];
      ocnt += __popc(em);
    }
    if (ocnt > kOutCap - 32 * B) warp_flush(W, ocnt, out, out_len);
  }
  __syncwarp();
  return total;
}

// A frontier of <= 32 items: every warp derives the whole plan and takes
// its own slot chunks (the hub's level, the last levels).
template <class Op>
__device__ __forceinline__ void push_tiny(WarpSmem& W, Op& o, const int32_t* __restrict__ F,
                                          int64_t nf, const int64_t* __restrict__ row,
                                          const int32_t* __restrict__ col,
                                          int32_t* __restrict__ out,
                                          unsigned long long* __restrict__ out_len,
                                          unsigned long long* __restrict__ total_out, int64_t gw,
                                          int64_t nw, CtaAgg& agg) {
  const int lane = threadIdx.x & 31;
  int32_t v = 0;
  int64_t rb = 0, deg = 0;
  if (lane < nf) {
    v = F[lane];
    rb = row[v];
    deg = row[v + 1] - rb;
  }
  int ocnt = 0;
  const int64_t total = expand_items32(W, o, v, rb, deg, col, out, out_len, ocnt,
                                       gw * 32 * Op::kBatch, nw * 32 * Op::kBatch);
  cta_flush(W, ocnt, out, out_len, agg);
  if (gw == 0 && lane == 0) *total_out = (unsigned long long)total;
}

// A frontier of up to kMidItems items: each warp expands 32 consecutive
// items by itself (no scan pass, no plan barrier); items with more than
// kHeavyDeg slots are set aside in `heavy` (count in *nheavy) for a second,
// cooperative pass after the caller's barrier.
constexpr int64_t kMidItems = 1 << 16;
constexpr int64_t kHeavyDeg = 1024;
template <class Op>
__device__ __forceinline__ void push_mid(WarpSmem& W, Op& o, const int32_t* __restrict__ F,
                                         int64_t nf, const int64_t* __restrict__ row,
                                         const int32_t* __restrict__ col,
                                         int32_t* __restrict__ out,
                                         unsigned long long* __restrict__ out_len,
                                         int32_t* __restrict__ heavy,
                                         unsigned long long* __restrict__ nheavy, int64_t gw,
                                         int64_t nw, CtaAgg& agg) {
  const int lane = threadIdx.x & 31;
  int ocnt = 0;
  unsigned long long tot = 0;
  for (int64_t base = gw * 32; base < nf; base += nw * 32) {
    const int64_t i = base + lane;
    int32_t v = 0;
    int64_t rb = 0, deg = 0;
    if (i < nf) {
      v = F[i];
      rb = row[v];
      deg = row[v + 1] - rb;
    }
    const bool hv = deg > kHeavyDeg;
    const unsigned hm = __ballot_sync(0xffffffffu, hv);
    if (hm) {
      unsigned long long at = 0;
      if (lane == __ffs(hm) - 1) at = atomicAdd(nheavy, (unsigned long long)__popc(hm));
      at = __shfl_sync(0xffffffffu, at, __ffs(hm) - 1);
      if (hv) heavy[at + __popc(hm & ((1u << lane) - 1))] = i;
    }
    tot += (unsigned long long)expand_items32(W, o, v, rb, hv ? 0 : deg, col, out, out_len, ocnt,
                                              0, 32 * Op::kBatch);
  }
  cta_flush(W, ocnt, out, out_len, agg);
  if (lane == 0 && tot) atomicAdd(&agg.ctr[2], tot);  // Counters::total, flushed by the caller
}

template <class Op>
__global__ void __launch_bounds__(kExpandBlock, Op::kMinBlocks)
    k_lb_expand(const int32_t* __restrict__ F, const unsigned long long* __restrict__ nf_d,
                const int64_t* __restrict__ scan, const int64_t* __restrict__ rowbase,
                const int32_t* __restrict__ part, const Counters* __restrict__ plan,
                const int32_t* __restrict__ col, const typename WeightOf<Op>::T* __restrict__ wgt,
                Op op,
                int32_t* __restrict__ out, unsigned long long* __restrict__ out_len) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  WarpSmem& W = warp_smem(smem_raw);
  Op o = op;  // mutable copy: functors keep per-thread prefetch registers
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  expand_tasks(W, o, F, (int64_t)*nf_d, scan, rowbase, part, (int64_t)plan->ntiles,
               (int64_t)plan->total, col, wgt, out, out_len, gw, nw);
}

constexpr int expand_smem_bytes() { return (int)sizeof(WarpSmem) * kWarpsPerBlock; }

template <class Op>
int set_expand_smem() {
  static bool done = false;
  if (done) return GFX_OK;
  GFX_CK(cudaFuncSetAttribute(k_lb_expand<Op>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              expand_smem_bytes()));
  done = true;
  return GFX_OK;
}

// scan + expand over queue F (size at *nf_d), emitting into out / *out_len
template <class Op>
int lb_advance(gfx_graph* g, const int32_t* F, const unsigned long long* nf_d, int64_t nf_max,
               Counters* plan_ctr, int64_t* scan, int64_t* rowbase, int32_t* part, const Op& op,
               int32_t* out, unsigned long long* out_len, const void* wgt = nullptr) {
  gfx_ctx* ctx = g->ctx;
  GFX_TRY(launch_degree_scan(g, F, nf_d, nf_max, g->row, scan, rowbase, part, plan_ctr));
  GFX_TRY(set_expand_smem<Op>());
  static int per_sm = 0;
  if (per_sm == 0) {
    GFX_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_lb_expand<Op>, kExpandBlock,
                                                         expand_smem_bytes()));
    if (per_sm < 1) per_sm = 1;
  }
  const int grid = ctx->sm_count * per_sm;
  GFX_LAUNCH((k_lb_expand<Op>), grid, kExpandBlock, expand_smem_bytes(), ctx->stream, F, nf_d,
             scan, rowbase, part, plan_ctr, g->col,
             reinterpret_cast<const typename WeightOf<Op>::T*>(wgt ? wgt : g->w), op, out, out_len);
  GFX_CK(cudaGetLastError());
  return GFX_OK;
}

}  // namespace gfx
