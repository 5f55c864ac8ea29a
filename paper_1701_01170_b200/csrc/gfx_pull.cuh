// Pull (bottom-up) level body shared by the single-GPU BFS (gfx_bfs.cu) and
// the partitioned multi-GPU BFS (gfx_dist.cu).
#pragma once

#include "gfx_device.cuh"
#include "gfx_expand.cuh"
#include "gfx_internal.cuh"

namespace gfx {

// frontier = one bitmap over global ids (single GPU)
struct BitmapFront {
  const uint32_t* bm;
  __device__ __forceinline__ uint32_t word(int32_t s) const { return bm[s >> 5]; }
  __device__ __forceinline__ bool bit(uint32_t w, int32_t s) const { return (w >> (s & 31)) & 1u; }
};

// Where a discovered vertex's depth goes: straight into the int32 label
// array, or (deferred output) into a byte-per-vertex depth array that stays
// L2-resident; the persistent BFS writes the int32 labels once, coalesced,
// after the last level.
struct LabelOut {
  int32_t* labels;
  uint8_t* lvl8;  // non-null: deferred mode
  __device__ __forceinline__ void set(int32_t v, int32_t d) const {
    if (lvl8) lvl8[v] = (uint8_t)d;
    else labels[v] = d;
  }
};

constexpr int kPullBatch = 8;   // candidates per lane in flight
constexpr int kSweepBatch = 8;  // head probes per lane in flight in the sweep

// per-warp scratch of the pull phase (aliases the expansion's WarpSmem)
constexpr int kPullStage = 256;  // staged list appends per warp (flushed with one atomic)
struct PullSmem {
  int32_t cand[1024];    // compacted candidate vertices of the warp's 32 words
  uint32_t newbits[32];  // found bits per word of the group
  int32_t stage[kPullStage];  // unfound candidates awaiting their append
};
static_assert(sizeof(PullSmem) <= sizeof(WarpSmem) + 2048, "pull scratch must fit the warp slice");
constexpr int kWarpScratch = sizeof(PullSmem) > sizeof(WarpSmem) ? sizeof(PullSmem) : sizeof(WarpSmem);

// Pull (bottom-up) level.  One warp owns 32 consecutive bitmap words (1024
// vertices).  Candidates (unvisited & in-degree > 0) are first compacted
// into the warp's shared-memory list, so every lane always works on a real
// candidate however sparse the unvisited set is.  Each candidate's first
// probe reads head[u] -- the graph-constant copy of its first in-neighbour,
// stored densely -- and only misses fetch their row bounds and scan on in
// ascending order (reference pull_expand, operators.py:269-307, scans every
// in-edge; labels are identical, only the work differs).  Found bits are
// gathered per word in shared memory and written with plain coalesced
// stores (the warp owns its words).
// counters: out_len += |new frontier|, edges += sum of in-degree(U) (only
//           when count_in_edges; for undirected graphs the per-level degree
//           post-pass derives it), aux0 += early-exit probes S(U),
//           aux1 += |U| with in-degree > 0.
// FrontT: frontier membership of an in-neighbour s (global id):
//   uint32_t word(s) loads the bitmap word holding s; bool bit(w, s) tests it.
template <class FrontT>
__device__ __forceinline__ void pull_groups(
    int64_t words, const uint32_t* __restrict__ nz_in, uint32_t* __restrict__ visited,
    const FrontT front, uint32_t* __restrict__ next,
    const int32_t* __restrict__ head, const int64_t* __restrict__ rrow,
    const int32_t* __restrict__ rcol, int count_in_edges, int32_t* __restrict__ labels,
    int32_t* __restrict__ preds, int32_t depth, Counters* __restrict__ ctr, int64_t gw,
    int64_t nwarps, PullSmem& P) {
  const int lane = threadIdx.x & 31;
  unsigned long long found_cnt = 0, in_edges = 0, probes = 0, cands = 0;
  for (int64_t grp = gw; grp * 32 < words; grp += nwarps) {
    const int64_t w = grp * 32 + lane;
    uint32_t vis = 0xffffffffu, cand = 0;
    if (w < words) {
      vis = visited[w];
      cand = ~vis & nz_in[w];
    }
    int total;
    const int off = warp_excl_scan(__popc(cand), lane, &total);
    if (total == 0) {
      if (w < words) next[w] = 0u;  // the frontier buffer is reused across levels
      continue;
    }
    P.newbits[lane] = 0u;
    {
      uint32_t x = cand;
      int k = off;
      while (x) {
        const int b = __ffs(x) - 1;
        x &= x - 1;
        P.cand[k++] = (int32_t)(w * 32 + b);
      }
    }
    __syncwarp();
    cands += (unsigned long long)(lane == 0 ? total : 0);
    // phase 1: first probe of every candidate from the dense head array;
    // misses are compacted in place to the front of the list
    int nmiss = 0;
    for (int base = 0; base < total; base += 32 * kPullBatch) {
      int32_t u[kPullBatch], h[kPullBatch];
      uint32_t fw[kPullBatch];
#pragma unroll
      for (int q = 0; q < kPullBatch; ++q) {
        const int k = base + q * 32 + lane;
        u[q] = k < total ? P.cand[k] : -1;
        h[q] = u[q] >= 0 ? head[u[q]] : -1;
      }
#pragma unroll
      for (int q = 0; q < kPullBatch; ++q) fw[q] = h[q] >= 0 ? front.word(h[q]) : 0u;
      __syncwarp();
#pragma unroll
      for (int q = 0; q < kPullBatch; ++q) {
        const bool hit = h[q] >= 0 && front.bit(fw[q], h[q]);
        const bool miss = h[q] >= 0 && !hit;
        if (hit) {
          labels[u[q]] = depth;
          preds[u[q]] = h[q];
          atomicOr(&P.newbits[(u[q] >> 5) - grp * 32], 1u << (u[q] & 31));
          ++found_cnt;
          ++probes;
          if (count_in_edges) in_edges += (unsigned long long)(rrow[u[q] + 1] - rrow[u[q]]);
        }
        const unsigned mm = __ballot_sync(0xffffffffu, miss);
        if (miss) P.cand[nmiss + __popc(mm & ((1u << lane) - 1))] = u[q];
        nmiss += __popc(mm);
      }
    }
    __syncwarp();
    // phase 2: misses, one per lane, scanning on from the second in-neighbour
    // with four column loads in flight (early-exit count stays exact)
    for (int base = 0; base < nmiss; base += 32) {
      const int k = base + lane;
      if (k >= nmiss) continue;
      const int32_t uu = P.cand[k];
      const int64_t b = rrow[uu], e = rrow[uu + 1];
      bool found = false;
      int32_t par = -1;
      int64_t p = b + 1;
      while (p < e && !found) {
        int32_t sv[4];
        uint32_t wv[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) sv[t] = (p + t < e) ? ld_stream_i32(rcol + p + t) : -1;
#pragma unroll
        for (int t = 0; t < 4; ++t) wv[t] = sv[t] >= 0 ? front.word(sv[t]) : 0u;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          if (!found && sv[t] >= 0 && front.bit(wv[t], sv[t])) {
            found = true;
            par = sv[t];
            p = p + t;
          }
        }
        if (!found) p += 4;
      }
      probes += (unsigned long long)(found ? p - b + 1 : e - b);
      in_edges += (unsigned long long)(e - b);
      if (found) {
        labels[uu] = depth;
        preds[uu] = par;
        atomicOr(&P.newbits[(uu >> 5) - grp * 32], 1u << (uu & 31));
        ++found_cnt;
      }
    }
    __syncwarp();
    if (w < words) {
      const uint32_t nb = P.newbits[lane];
      next[w] = nb;
      if (nb) visited[w] = vis | nb;
    } else {
      (void)0;
    }
    __syncwarp();
  }
  found_cnt = warp_sum_u64(found_cnt);
  in_edges = warp_sum_u64(in_edges);
  probes = warp_sum_u64(probes);
  cands = warp_sum_u64(cands);
  if (lane == 0) {
    if (found_cnt) atomicAdd(&ctr->out_len, found_cnt);
    if (in_edges) atomicAdd(&ctr->edges, in_edges);
    if (probes) atomicAdd(&ctr->aux0, probes);
    if (cands) atomicAdd(&ctr->aux1, cands);
  }
}

// Per-warp staged list appends: items are compacted into a shared-memory
// buffer and appended to the global list with ONE atomicAdd per flush, so
// the level's emits do not serialise on a single counter address.
struct WarpStage {
  int32_t* buf;
  int cap, cnt;
  __device__ __forceinline__ void flush(int32_t* __restrict__ list,
                                        unsigned long long* __restrict__ len) {
    const int lane = threadIdx.x & 31;
    if (cnt == 0) return;
    __syncwarp();
    unsigned long long b = 0;
    if (lane == 0) b = atomicAdd(len, (unsigned long long)cnt);
    b = __shfl_sync(0xffffffffu, b, 0);
    for (int j = lane; j < cnt; j += 32) list[b + j] = buf[j];
    __syncwarp();
    cnt = 0;
  }
  // warp-uniform call; flushes first when the buffer could overflow
  __device__ __forceinline__ void push(bool want, int32_t v, int32_t* __restrict__ list,
                                       unsigned long long* __restrict__ len) {
    const int lane = threadIdx.x & 31;
    const unsigned m = __ballot_sync(0xffffffffu, want);
    if (!m) return;
    if (cnt + 32 > cap) flush(list, len);
    if (want) buf[cnt + __popc(m & ((1u << lane) - 1))] = v;
    cnt += __popc(m);
  }
};

// warp-aggregated append of this lane's `want` item to list[*len]
__device__ __forceinline__ void warp_append(bool want, int32_t v, int32_t* __restrict__ list,
                                            unsigned long long* __restrict__ len) {
  const int lane = threadIdx.x & 31;
  const unsigned m = __ballot_sync(0xffffffffu, want);
  if (!m) return;
  unsigned long long b = 0;
  if (lane == __ffs(m) - 1) b = atomicAdd(len, (unsigned long long)__popc(m));
  b = __shfl_sync(0xffffffffu, b, __ffs(m) - 1);
  if (want) list[b + __popc(m & ((1u << lane) - 1))] = v;
}

// Scan the in-neighbours of u from position p0 (ascending) for the first one
// in the frontier; 4 column loads in flight.  Returns the parent or -1 and
// adds the sequential early-exit probe count (reference pull_expand scans
// in-edges in CSC order, operators.py:269-307) to *probes.
template <class FrontT>
__device__ __forceinline__ int32_t scan_in_edges(const FrontT& front,
                                                 const int32_t* __restrict__ rcol, int64_t b,
                                                 int64_t p0, int64_t e,
                                                 unsigned long long* probes) {
  int64_t p = p0;
  int32_t par = -1;
  while (p < e && par < 0) {
    int32_t sv[4];
    uint32_t wv[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) sv[t] = (p + t < e) ? ld_stream_i32(rcol + p + t) : -1;
#pragma unroll
    for (int t = 0; t < 4; ++t) wv[t] = sv[t] >= 0 ? front.word(sv[t]) : 0u;
    int hitt = -1;
#pragma unroll
    for (int t = 3; t >= 0; --t)
      if (sv[t] >= 0 && front.bit(wv[t], sv[t])) hitt = t;
    if (hitt >= 0) {
      par = sv[hitt];
      p += hitt;
    } else {
      p += 4;
    }
  }
  *probes += (unsigned long long)(par >= 0 ? p - b + 1 : e - b);
  return par;
}

// Resolve the misses list[0..cnt) -- candidates whose head probe missed --
// by scanning each one's in-neighbours on from the second, ascending: first
// kMissPerLane misses per lane and 2 probes per miss in flight per round (a
// group's misses cost a few dependent round trips instead of one scan chain
// per 32).
// The early-exit probe count stays the sequential one.  found(want, u, par)
// and unfound(want, u) are called warp-uniformly (every lane, with a flag).
constexpr int kMissPerLane = 4;
template <class FrontT, class Found, class Unfound>
__device__ __forceinline__ void resolve_misses(const int32_t* list, int cnt, const FrontT& front,
                                               const int64_t* __restrict__ rrow,
                                               const int32_t* __restrict__ rcol,
                                               int count_in_edges, unsigned long long& probes,
                                               unsigned long long& in_edges, Found found,
                                               Unfound unfound) {
  constexpr int MB = kMissPerLane;
  const int lane = threadIdx.x & 31;
  for (int mb = 0; mb < cnt; mb += 32 * MB) {
    int32_t u[MB], par[MB], done[MB], deg[MB];
    int64_t b[MB];
#pragma unroll
    for (int q = 0; q < MB; ++q) {
      const int k = mb + q * 32 + lane;
      u[q] = k < cnt ? list[k] : -1;
      par[q] = -1;
      done[q] = 1;  // the head (position b) already missed
      b[q] = 0;
      deg[q] = 0;
    }
#pragma unroll
    for (int q = 0; q < MB; ++q) {
      if (u[q] >= 0) {
        b[q] = rrow[u[q]];
        deg[q] = (int32_t)(rrow[u[q] + 1] - b[q]);
      }
    }
    for (;;) {
      int32_t sv[MB][2];
      uint32_t wv[MB][2];
#pragma unroll
      for (int q = 0; q < MB; ++q)
#pragma unroll
        for (int t = 0; t < 2; ++t)
          sv[q][t] = (par[q] < 0 && done[q] + t < deg[q]) ? ld_stream_i32(rcol + b[q] + done[q] + t)
                                                          : -1;
#pragma unroll
      for (int q = 0; q < MB; ++q)
#pragma unroll
        for (int t = 0; t < 2; ++t) wv[q][t] = sv[q][t] >= 0 ? front.word(sv[q][t]) : 0u;
      bool pending = false;
#pragma unroll
      for (int q = 0; q < MB; ++q) {
        if (par[q] >= 0 || done[q] >= deg[q]) continue;
        if (front.bit(wv[q][0], sv[q][0])) {
          par[q] = sv[q][0];
          done[q] += 1;
        } else if (sv[q][1] >= 0 && front.bit(wv[q][1], sv[q][1])) {
          par[q] = sv[q][1];
          done[q] += 2;
        } else {
          done[q] = min(done[q] + 2, deg[q]);
          pending |= done[q] < deg[q];
        }
      }
      if (!__any_sync(0xffffffffu, pending)) break;
    }
#pragma unroll
    for (int q = 0; q < MB; ++q) {
      if (u[q] >= 0) {
        b[q] = rrow[u[q]];
        deg[q] = (int32_t)(rrow[u[q] + 1] - b[q]);
      }
    }
    {  // first round: 2 probes per miss, all misses of the lane in flight
      int32_t sv[MB][2];
      uint32_t wv[MB][2];
#pragma unroll
      for (int q = 0; q < MB; ++q)
#pragma unroll
        for (int t = 0; t < 2; ++t)
          sv[q][t] = (u[q] >= 0 && done[q] + t < deg[q]) ? ld_stream_i32(rcol + b[q] + done[q] + t)
                                                         : -1;
#pragma unroll
      for (int q = 0; q < MB; ++q)
#pragma unroll
        for (int t = 0; t < 2; ++t) wv[q][t] = sv[q][t] >= 0 ? front.word(sv[q][t]) : 0u;
#pragma unroll
      for (int q = 0; q < MB; ++q) {
        if (u[q] < 0 || done[q] >= deg[q]) continue;
        if (front.bit(wv[q][0], sv[q][0])) {
          par[q] = sv[q][0];
          done[q] += 1;
        } else if (sv[q][1] >= 0 && front.bit(wv[q][1], sv[q][1])) {
          par[q] = sv[q][1];
          done[q] += 2;
        } else {
          done[q] = min(done[q] + 2, deg[q]);
        }
      }
    }
    // the rest (rare: long in-lists without an early hit) is scanned by the
    // whole warp, one vertex at a time, 32 coalesced probes per step; the
    // first hit in ascending order gives the exact early-exit count
#pragma unroll
    for (int q = 0; q < MB; ++q) {
      unsigned pend = __ballot_sync(0xffffffffu, u[q] >= 0 && par[q] < 0 && done[q] < deg[q]);
      while (pend) {
        const int src = __ffs(pend) - 1;
        pend &= pend - 1;
        const int64_t bb = __shfl_sync(0xffffffffu, b[q], src);
        const int32_t dg = __shfl_sync(0xffffffffu, deg[q], src);
        int32_t pos = __shfl_sync(0xffffffffu, done[q], src);
        int32_t found = -1;
        while (pos < dg) {
          const int32_t p = pos + lane;
          const int32_t sv = p < dg ? ld_stream_i32(rcol + bb + p) : -1;
          const bool hit = sv >= 0 && front.bit(front.word(sv), sv);
          const unsigned hm = __ballot_sync(0xffffffffu, hit);
          if (hm) {
            const int first = __ffs(hm) - 1;
            found = __shfl_sync(0xffffffffu, sv, first);
            pos += first + 1;
            break;
          }
          pos = min(pos + 32, dg);
        }
        if (lane == src) {
          par[q] = found;
          done[q] = pos;
        }
      }
    }
#pragma unroll
    for (int q = 0; q < MB; ++q) {
      if (u[q] >= 0) {
        b[q] = rrow[u[q]];
        deg[q] = (int32_t)(rrow[u[q] + 1] - b[q]);
      }
    }
    for (;;) {
      int32_t sv[MB][2];
      uint32_t wv[MB][2];
#pragma unroll
      for (int q = 0; q < MB; ++q)
#pragma unroll
        for (int t = 0; t < 2; ++t)
          sv[q][t] = (par[q] < 0 && done[q] + t < deg[q]) ? ld_stream_i32(rcol + b[q] + done[q] + t)
                                                          : -1;
#pragma unroll
      for (int q = 0; q < MB; ++q)
#pragma unroll
        for (int t = 0; t < 2; ++t) wv[q][t] = sv[q][t] >= 0 ? front.word(sv[q][t]) : 0u;
      bool pending = false;
#pragma unroll
      for (int q = 0; q < MB; ++q) {
        if (par[q] >= 0 || done[q] >= deg[q]) continue;
        if (front.bit(wv[q][0], sv[q][0])) {
          par[q] = sv[q][0];
          done[q] += 1;
        } else if (sv[q][1] >= 0 && front.bit(wv[q][1], sv[q][1])) {
          par[q] = sv[q][1];
          done[q] += 2;
        } else {
          done[q] = min(done[q] + 2, deg[q]);
          pending |= done[q] < deg[q];
        }
      }
      if (!__any_sync(0xffffffffu, pending)) break;
    }
#pragma unroll
    for (int q = 0; q < MB; ++q) {
      if (u[q] >= 0) {
        probes += (unsigned long long)done[q];
        if (count_in_edges) in_edges += (unsigned long long)deg[q];
      }
      found(u[q] >= 0 && par[q] >= 0, u[q], par[q]);
      unfound(u[q] >= 0 && par[q] < 0, u[q]);
    }
  }
}

// Pull level, SWEEP form (the first pull level of a traversal): like
// pull_groups, but groups of 32 bitmap words are handed out dynamically
// (one atomic grab per group, issued a group ahead) so the level's tail is
// not set by the densest static slice, and every candidate that stays
// unvisited is appended to `unext` -- the candidate list the following pull
// levels walk instead of sweeping the whole bitmap again.
// counters: out_len |new frontier|, aux0 probes S(U), aux1 |U|, aux2 group
// grab cursor (zero on entry), aux3 |unext|; edges (directed only).
template <class FrontT>
__device__ __forceinline__ void pull_sweep(
    int64_t words, const uint32_t* __restrict__ nz_in, uint32_t* __restrict__ visited,
    const FrontT front, uint32_t* __restrict__ next, const int32_t* __restrict__ head,
    const int64_t* __restrict__ rrow, const int32_t* __restrict__ rcol, int count_in_edges,
    const LabelOut lab, int32_t* __restrict__ preds, int32_t depth,
    Counters* __restrict__ ctr, int32_t* __restrict__ unext, int64_t gw, int64_t nwarps,
    PullSmem& P, int knobs = 0) {
  const int lane = threadIdx.x & 31;
  const int64_t ngroups = (words + 31) / 32;
  unsigned long long found_cnt = 0, in_edges = 0, probes = 0, cands = 0;
  WarpStage st{P.stage, kPullStage, 0};
  // the next group's bitmap words are loaded while this group is processed
  // (static assignment: only this warp writes them during the level)
  uint32_t vis_n = 0xffffffffu, nz_n = 0u;
  if (gw < ngroups && gw * 32 + lane < words) {
    vis_n = visited[gw * 32 + lane];
    nz_n = nz_in[gw * 32 + lane];
  }
  for (int64_t grp = gw; grp < ngroups; grp += nwarps) {
    const int64_t w = grp * 32 + lane;
    const uint32_t vis = vis_n, cand = ~vis_n & nz_n;
    {
      const int64_t w2 = (grp + nwarps) * 32 + lane;
      vis_n = 0xffffffffu;
      nz_n = 0u;
      if (w2 < words) {
        vis_n = visited[w2];
        nz_n = nz_in[w2];
      }
    }
    int total;
    const int off = warp_excl_scan(__popc(cand), lane, &total);
    if (total == 0) {
      if (w < words) next[w] = 0u;
    } else {
      P.newbits[lane] = 0u;
      {
        uint32_t x = cand;
        int k = off;
        while (x) {
          const int b = __ffs(x) - 1;
          x &= x - 1;
          P.cand[k++] = (int32_t)(w * 32 + b);
        }
      }
      __syncwarp();
      cands += (unsigned long long)(lane == 0 ? total : 0);
      int nmiss = 0;
      // consecutive lanes probe consecutive candidates (their label / pred
      // stores coalesce); kSweepBatch head probes per lane in flight, the
      // candidate ids re-read from shared memory instead of held in registers
      for (int base = 0; base < total; base += 32 * kSweepBatch) {
        int32_t h[kSweepBatch];
        uint32_t fw[kSweepBatch];
#pragma unroll
        for (int q = 0; q < kSweepBatch; ++q) {
          const int k = base + q * 32 + lane;
          h[q] = k < total ? head[P.cand[k]] : -1;
        }
#pragma unroll
        for (int q = 0; q < kSweepBatch; ++q)
          fw[q] = h[q] >= 0 ? ((knobs & 4) ? __ldg(front.bm + (h[q] >> 5)) : front.word(h[q])) : 0u;
        __syncwarp();
#pragma unroll
        for (int q = 0; q < kSweepBatch; ++q) {
          const int k = base + q * 32 + lane;
          const int32_t u = k < total ? P.cand[k] : -1;
          const bool hit = h[q] >= 0 && front.bit(fw[q], h[q]);
          const bool miss = h[q] >= 0 && !hit;
          if (hit) {
            if (!(knobs & 2)) {
              lab.set(u, depth);
              preds[u] = h[q];
            }
            atomicOr(&P.newbits[(u >> 5) - grp * 32], 1u << (u & 31));
            ++found_cnt;
            ++probes;
            if (count_in_edges) in_edges += (unsigned long long)(rrow[u + 1] - rrow[u]);
          }
          const unsigned mm = __ballot_sync(0xffffffffu, miss);
          if (miss) P.cand[nmiss + __popc(mm & ((1u << lane) - 1))] = u;
          nmiss += __popc(mm);
        }
      }
      __syncwarp();
      if (knobs & 1) nmiss = 0;
      resolve_misses(P.cand, nmiss, front, rrow, rcol, count_in_edges, probes, in_edges,
                     [&](bool want, int32_t uu, int32_t par) {
                       if (want) {
                         lab.set(uu, depth);
                         preds[uu] = par;
                         atomicOr(&P.newbits[(uu >> 5) - grp * 32], 1u << (uu & 31));
                         ++found_cnt;
                       }
                     },
                     [&](bool want, int32_t uu) {
                       if (unext) st.push(want, uu, unext, &ctr->aux3);
                     });
      __syncwarp();
      if (w < words) {
        const uint32_t nb = P.newbits[lane];
        next[w] = nb;
        if (nb) visited[w] = vis | nb;
      }
      __syncwarp();
    }
  }
  if (unext) st.flush(unext, &ctr->aux3);
  found_cnt = warp_sum_u64(found_cnt);
  in_edges = warp_sum_u64(in_edges);
  probes = warp_sum_u64(probes);
  cands = warp_sum_u64(cands);
  if (lane == 0) {
    if (found_cnt) atomicAdd(&ctr->out_len, found_cnt);
    if (in_edges) atomicAdd(&ctr->edges, in_edges);
    if (probes) atomicAdd(&ctr->aux0, probes);
    if (cands) atomicAdd(&ctr->aux1, cands);
  }
}

// Pull level, LIST form: walk the candidate list U[0..nu) left by the
// previous pull level (entries visited since, by a push level, are stale and
// dropped).  Found vertices set their bit in `next` (pre-zeroed) and in
// `visited`, and are appended to the frontier queue `qout` (so a following
// push level needs no bitmap-to-queue pass); unfound candidates go to
// `unext`.  Both appends are staged per warp in shared memory.  Same
// counters as pull_sweep (out_len doubles as the queue cursor).
template <class FrontT>
__device__ __forceinline__ void pull_list(
    const int32_t* __restrict__ U, int64_t nu, uint32_t* __restrict__ visited,
    const FrontT front, uint32_t* __restrict__ next, const int32_t* __restrict__ head,
    const int64_t* __restrict__ rrow, const int32_t* __restrict__ rcol, int count_in_edges,
    const LabelOut lab, int32_t* __restrict__ preds, int32_t depth,
    Counters* __restrict__ ctr, int32_t* __restrict__ qout, int32_t* __restrict__ unext,
    int64_t gw, int64_t nwarps, PullSmem& P) {
  constexpr int B = kPullBatch;
  static_assert(32 * B <= kPullStage, "miss scratch");
  const int lane = threadIdx.x & 31;
  WarpStage fq{P.cand, 512, 0};
  WarpStage uq{P.cand + 512, 512, 0};
  unsigned long long in_edges = 0, probes = 0, cands = 0;
  for (int64_t base = gw * 32 * B; base < nu; base += nwarps * 32 * B) {
    int32_t u[B], h[B];
    uint32_t vw[B], fw[B];
#pragma unroll
    for (int q = 0; q < B; ++q) {
      const int64_t i = base + q * 32 + lane;
      u[q] = i < nu ? U[i] : -1;
    }
#pragma unroll
    for (int q = 0; q < B; ++q) {
      vw[q] = u[q] >= 0 ? visited[u[q] >> 5] : 0u;
      h[q] = u[q] >= 0 ? head[u[q]] : -1;
    }
#pragma unroll
    for (int q = 0; q < B; ++q) {
      if (u[q] >= 0 && ((vw[q] >> (u[q] & 31)) & 1u)) u[q] = -1;  // stale
      fw[q] = (u[q] >= 0 && h[q] >= 0) ? front.word(h[q]) : 0u;
    }
    // head probes; every candidate that misses is staged for the scan
    int nmiss = 0;
    int32_t* miss = P.stage;  // 32 * B entries
#pragma unroll
    for (int q = 0; q < B; ++q) {
      const bool live = u[q] >= 0;
      const bool hit = live && h[q] >= 0 && front.bit(fw[q], h[q]);
      if (live) ++cands;
      if (hit) {
        lab.set(u[q], depth);
        preds[u[q]] = h[q];
        const uint32_t bit = 1u << (u[q] & 31);
        atomicOr(&next[u[q] >> 5], bit);
        atomicOr(&visited[u[q] >> 5], bit);
        ++probes;
        if (count_in_edges) in_edges += (unsigned long long)(rrow[u[q] + 1] - rrow[u[q]]);
      }
      fq.push(hit, u[q], qout, &ctr->out_len);
      const unsigned mm = __ballot_sync(0xffffffffu, live && !hit);
      if (live && !hit) miss[nmiss + __popc(mm & ((1u << lane) - 1))] = u[q];
      nmiss += __popc(mm);
    }
    __syncwarp();
    resolve_misses(miss, nmiss, front, rrow, rcol, count_in_edges, probes, in_edges,
                   [&](bool want, int32_t uu, int32_t par) {
                     if (want) {
                       lab.set(uu, depth);
                       preds[uu] = par;
                       const uint32_t bit = 1u << (uu & 31);
                       atomicOr(&next[uu >> 5], bit);
                       atomicOr(&visited[uu >> 5], bit);
                     }
                     fq.push(want, uu, qout, &ctr->out_len);
                   },
                   [&](bool want, int32_t uu) { uq.push(want, uu, unext, &ctr->aux3); });
    __syncwarp();
  }
  fq.flush(qout, &ctr->out_len);
  uq.flush(unext, &ctr->aux3);
  in_edges = warp_sum_u64(in_edges);
  probes = warp_sum_u64(probes);
  cands = warp_sum_u64(cands);
  if (lane == 0) {
    if (in_edges) atomicAdd(&ctr->edges, in_edges);
    if (probes) atomicAdd(&ctr->aux0, probes);
    if (cands) atomicAdd(&ctr->aux1, cands);
  }
}

}  // namespace gfx
