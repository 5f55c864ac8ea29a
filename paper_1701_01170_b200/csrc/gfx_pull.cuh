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
// array, or (deferred labels, the single-GPU persistent BFS) into a
// byte-per-vertex depth array that stays L2-resident; the int32 labels are
// then written once, coalesced, after the last level.
struct LabelOut {
  int32_t* labels;
  uint8_t* lvl8;  // non-null: deferred mode
  __device__ __forceinline__ void set(int32_t v, int32_t d) const {
    if (lvl8) lvl8[v] = (uint8_t)d;
    else labels[v] = d;
  }
};

constexpr int kPullBatch = 8;  // candidates per lane in flight

// Diagnostic (-DGFX_BFS_TIMELINE only): SM cycles per pull phase summed over
// warps, per depth: [0] bitmap words + candidate list, [1] head probes,
// [2] found-bit rebuild, [3] misses, [4] stores, [5] groups, [6] misses count
#ifdef GFX_BFS_TIMELINE
static __device__ unsigned long long g_pull_ph[64][8];
#define PULL_T(k)                                   \
  do {                                              \
    const long long t_ = clock64();                 \
    ph[k] += (unsigned long long)(t_ - t_last);     \
    t_last = t_;                                    \
  } while (0)
#else
#define PULL_T(k) \
  do {            \
  } while (0)
#endif

// per-warp scratch of the pull phase (aliases the expansion's WarpSmem)
struct PullSmem {
  int32_t cand[1024];    // compacted candidate vertices of the warp's 32 words
  uint32_t newbits[32];  // found bits per word of the group
  uint32_t hitmask[32];  // head-probe hits, one ballot per 32 consecutive candidates
};
static_assert(sizeof(PullSmem) <= sizeof(WarpSmem) + 1024, "pull scratch must fit the warp slice");
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
template <class FrontT, int kPB = kPullBatch>
__device__ __forceinline__ void pull_groups(
    int64_t words, const uint32_t* __restrict__ nz_in, uint32_t* __restrict__ visited,
    const FrontT front, uint32_t* __restrict__ next,
    const int32_t* __restrict__ head, const int64_t* __restrict__ rrow,
    const int32_t* __restrict__ rcol, int count_in_edges, const LabelOut labels,
    int32_t* __restrict__ preds, int32_t depth, Counters* __restrict__ ctr, int64_t gw,
    int64_t nwarps, PullSmem& P, const int32_t* __restrict__ head2 = nullptr,
    unsigned long long* __restrict__ grab = nullptr, int32_t* __restrict__ qout = nullptr,
    unsigned long long* __restrict__ qlen = nullptr) {
  // qout (optional): the found vertices are also appended to a queue, one
  // reservation per 1024-vertex group (*qlen counts them)
  const int lane = threadIdx.x & 31;
  // head / head2 are streamed once per level: no L1 allocation (the L1
  // keeps the frontier words the probes hit), evict-first in L2
  const unsigned long long pol = l2_evict_first_policy();
  unsigned long long found_cnt = 0, in_edges = 0, probes = 0, cands = 0;
  // groups are dealt out statically for all but the last ~1.5 rounds; the
  // rest are handed out dynamically when `grab` (a zeroed counter) is given
  // -- the next group is claimed while this one is processed -- so warps
  // with slow groups do not set the level's tail
  const int64_t ngroups = (words + 31) / 32;
  // (every warp's first group is static: the dynamic range starts after them)
  const int64_t nstatic = grab ? max(ngroups / nwarps - 1, (int64_t)1) * nwarps : ngroups;
  unsigned long long nxt = 0;
#ifdef GFX_BFS_TIMELINE
  unsigned long long ph[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long t_last = clock64();
#endif
  for (int64_t grp = gw; grp < ngroups;) {
    const bool dyn_next = grp + nwarps >= nstatic;
    if (grab && dyn_next && lane == 0) nxt = atomicAdd(grab, 1ull);
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
      grp = (grab && dyn_next) ? nstatic + (int64_t)__shfl_sync(0xffffffffu, nxt, 0) : grp + nwarps;
      continue;
    }
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
    PULL_T(0);
#ifdef GFX_BFS_TIMELINE
    ph[5] += 1;
#endif
    cands += (unsigned long long)(lane == 0 ? total : 0);
    // phase 1: first probe of every candidate from the dense head array;
    // misses are compacted in place to the front of the list
    int nmiss = 0;
    for (int base = 0; base < total; base += 32 * kPB) {
      int32_t u[kPB], h[kPB];
      uint32_t fw[kPB];
#pragma unroll
      for (int q = 0; q < kPB; ++q) {
        const int k = base + q * 32 + lane;
        u[q] = k < total ? P.cand[k] : -1;
        h[q] = u[q] >= 0 ? ld_stream_i32(head + u[q], pol) : -1;
      }
      // with head2, head carries bit 31 = "in-degree is exactly 1" (-1 stays
      // "no in-neighbour"): such a miss is settled without a second look
      bool last[kPB];
#pragma unroll
      for (int q = 0; q < kPB; ++q) {
        last[q] = head2 != nullptr && h[q] != -1 && h[q] < 0;
        if (last[q]) h[q] &= 0x7fffffff;
      }
#pragma unroll
      for (int q = 0; q < kPB; ++q) fw[q] = h[q] >= 0 ? front.word(h[q]) : 0u;
      __syncwarp();
#pragma unroll
      for (int q = 0; q < kPB; ++q) {
        const bool hit = h[q] >= 0 && front.bit(fw[q], h[q]);
        const bool miss = h[q] >= 0 && !hit && !last[q];
        if (h[q] >= 0 && !hit && last[q]) {  // unfound, one probe, degree 1
          ++probes;
          ++in_edges;
        }
        if (hit) {
          labels.set(u[q], depth);
          preds[u[q]] = h[q];
          ++found_cnt;
          ++probes;
          if (count_in_edges) in_edges += (unsigned long long)(rrow[u[q] + 1] - rrow[u[q]]);
        }
        const unsigned hm = __ballot_sync(0xffffffffu, hit);
        if (lane == 0) P.hitmask[(base >> 5) + q] = hm;
        const unsigned mm = __ballot_sync(0xffffffffu, miss);
        if (miss) P.cand[nmiss + __popc(mm & ((1u << lane) - 1))] = u[q];
        nmiss += __popc(mm);
      }
    }
    __syncwarp();
    PULL_T(1);
#ifdef GFX_BFS_TIMELINE
    ph[6] += nmiss;
#endif
    // each lane rebuilds its word's found bits: its candidates are entries
    // [off, off + popc(cand)) of the list, whose hit bits are consecutive in
    // hitmask; deposit them onto the candidate bit positions (no shared
    // atomics -- lanes of one word would all hit the same address)
    {
      const int c = __popc(cand);
      uint32_t nb = 0u;
      if (c) {
        const int r0 = off >> 5, sh = off & 31;
        uint32_t comp = P.hitmask[r0] >> sh;
        if (sh && off + c > (r0 + 1) * 32) comp |= P.hitmask[r0 + 1] << (32 - sh);
        uint32_t x = cand;
        for (int j = 0; x; ++j) {
          const uint32_t b = x & (0u - x);
          if ((comp >> j) & 1u) nb |= b;
          x ^= b;
        }
      }
      P.newbits[lane] = nb;
    }
    __syncwarp();
    PULL_T(2);
    // phase 2a (head2 given): the second in-neighbour of every miss from the
    // dense head2 array (bit 31 = "in-degree is exactly 2"), up to
    // kPB2 misses per lane in flight; most misses settle here without their
    // row bounds, the rest are compacted in place for phase 2b
    // (dense levels only: on sparse ones misses are rare and the extra
    // pass only costs registers -- measured +2 us on the s24 level 3)
    const bool two = head2 != nullptr && !count_in_edges;
    if (two && kPB >= 8) {
      constexpr int kPB2 = 4;
      int nrest = 0;
      for (int base = 0; base < nmiss; base += 32 * kPB2) {
        int32_t uu[kPB2], h2[kPB2];
        uint32_t fw[kPB2];
#pragma unroll
        for (int q = 0; q < kPB2; ++q) {
          const int k = base + q * 32 + lane;
          uu[q] = k < nmiss ? P.cand[k] : -1;
          h2[q] = uu[q] >= 0 ? ld_stream_i32(head2 + uu[q], pol) : 0;
        }
#pragma unroll
        for (int q = 0; q < kPB2; ++q)
          fw[q] = uu[q] >= 0 ? front.word(h2[q] & 0x7fffffff) : 0u;
        __syncwarp();
#pragma unroll
        for (int q = 0; q < kPB2; ++q) {
          const int32_t s2 = h2[q] & 0x7fffffff;
          const bool hit = uu[q] >= 0 && front.bit(fw[q], s2);
          const bool rest = uu[q] >= 0 && !hit && h2[q] >= 0;
          if (hit) {
            labels.set(uu[q], depth);
            preds[uu[q]] = s2;
            atomicOr(&P.newbits[(uu[q] >> 5) - grp * 32], 1u << (uu[q] & 31));
            ++found_cnt;
            probes += 2;
          } else if (uu[q] >= 0 && !rest) {  // in-degree 2, unfound
            probes += 2;
            in_edges += 2;
          }
          const unsigned rm = __ballot_sync(0xffffffffu, rest);
          if (rest) P.cand[nrest + __popc(rm & ((1u << lane) - 1))] = uu[q];
          nrest += __popc(rm);
        }
      }
      __syncwarp();
      nmiss = nrest;
    }
    // phase 2b: misses, one per lane, scanning on from the second (third
    // after phase 2a) in-neighbour with four column loads in flight
    // (early-exit count stays exact)
    for (int base = 0; base < nmiss; base += 32) {
      const int k = base + lane;
      if (k >= nmiss) continue;
      const int32_t uu = P.cand[k];
      if (two && kPB < 8) {
        // second in-neighbour inline (see phase 2a)
        int32_t h2 = ld_stream_i32(head2 + uu, pol);
        const bool deg2 = h2 < 0;
        h2 &= 0x7fffffff;
        if (front.bit(front.word(h2), h2)) {
          labels.set(uu, depth);
          preds[uu] = h2;
          atomicOr(&P.newbits[(uu >> 5) - grp * 32], 1u << (uu & 31));
          ++found_cnt;
          probes += 2;
          continue;
        }
        if (deg2) {
          probes += 2;
          in_edges += 2;
          continue;
        }
      }
      const int64_t b = rrow[uu], e = rrow[uu + 1];
      bool found = false;
      int32_t par = -1;
      int64_t p = b + (two ? 2 : 1);
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
        labels.set(uu, depth);
        preds[uu] = par;
        atomicOr(&P.newbits[(uu >> 5) - grp * 32], 1u << (uu & 31));
        ++found_cnt;
      }
    }
    __syncwarp();
    PULL_T(3);
    {
      const uint32_t nb = w < words ? P.newbits[lane] : 0u;
      if (w < words) {
        next[w] = nb;
        if (nb) visited[w] = vis | nb;
      }
      if (qout) {
        int qt;
        const int qo = warp_excl_scan(__popc(nb), lane, &qt);
        if (qt) {
          unsigned long long qb = 0;
          if (lane == 0) qb = atomicAdd(qlen, (unsigned long long)qt);
          qb = __shfl_sync(0xffffffffu, qb, 0) + qo;
          uint32_t x = nb;
          while (x) {
            const int b = __ffs(x) - 1;
            x &= x - 1;
            qout[qb++] = (int32_t)(w * 32 + b);
          }
        }
      }
    }
    __syncwarp();
    PULL_T(4);
    grp = (grab && dyn_next) ? nstatic + (int64_t)__shfl_sync(0xffffffffu, nxt, 0) : grp + nwarps;
  }
#ifdef GFX_BFS_TIMELINE
  if (lane == 0)
    for (int k = 0; k < 7; ++k) atomicAdd(&g_pull_ph[depth & 63][k], ph[k]);
#endif
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

}  // namespace gfx
