// Device-resident partitioned near/far SSSP ("push exchange of
// (v, newdist) pairs with owner-side atomicMin; the near/far threshold is
// global and 'near empty' is decided by allreduce") -- the low-latency form
// of the host-driven engine in gfx_dsssp.cu, built like the device-resident
// partitioned BFS (gfx_pdbfs.cu): ONE cooperative launch per rank, peer
// stores into the owners' inboxes and every rank's counter table, flag
// barriers; virtual ranks (P ranks in one launch on one GPU) or real ranks
// (one process per GPU, CUDA-IPC mappings).
//
// Reference: primitives/sssp.py:41-121 (relax = atomic_min + set_pred, each
// improved vertex enqueued once per iteration), near_far.py:20-85 (split at
// the threshold; advance_bucket: threshold += delta, stale far entries
// dropped, the rest re-split).  Per iteration, in lockstep on every rank:
//   relax : the rank's near queue (local ids) is expanded; an owned target
//           is relaxed in place with one 64-bit atomicMin on
//           (dist << 32 | global pred) plus the 32-bit distance mirror, and
//           enqueued once (mark bit); a remote target keeps this rank's best
//           offer of the run in sent_key[d] (monotone filter: an offer not
//           below an earlier one is never sent) and is emitted once per
//           iteration (sent bit);
//   send  : emitted remote targets become (d, sent_key[d]) messages stored
//           into the owner's inbox region for this rank;
//   apply : after the exchange barrier owners relax the offers like local
//           relaxations;
//   split : improved owned vertices go near / far at the GLOBAL threshold;
//   sums  : (near, far, slots, touched) rows to every rank, exchange barrier,
//           global sums; an empty global near pile advances every rank's
//           bucket together.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "gfx_device.cuh"
#include "gfx_expand.cuh"
#include "gfx_internal.cuh"
#include "gfx_scan.cuh"

namespace gfx {
namespace cg = cooperative_groups;

constexpr int kPsMaxRanks = 8;

struct PsRank {
  const int64_t* row;
  const int32_t* col;
  const int32_t* w;
  unsigned long long* dp;     // local: dist << 32 | global pred
  uint32_t* dist;             // local: 32-bit distance mirror (probe array)
  int32_t* stamp;             // local: iteration that last enqueued the vertex
  unsigned long long* sent_key;  // global ids: best offer sent this run
  uint32_t* sent;             // global ids: emitted this iteration
  int32_t* nearq[2];          // local ids
  int32_t* touched;           // local ids improved this iteration (with duplicates)
  int32_t* emit;              // expansion output (global ids)
  int32_t* far[2];
  int32_t* fkey[2];
  int64_t* scan;
  int64_t* rowbase;
  int32_t* part;
  unsigned long long* status;
  Counters* C;                // 3 rotating blocks
  unsigned long long* outcnt; // messages per owner this iteration
  int32_t* out_dist;          // results (local ids)
  int32_t* out_preds;
  int64_t nl, wl, far_cap;
  // exchange block
  unsigned long long* inbox;  // P regions x inbox_cap messages (2 words each)
  unsigned long long* inbox_cnt;
  long long* ctab;            // [2][kPsMaxRanks][4]
  unsigned* flags;
};

struct PsArgs {
  const PsRank* rk;
  PsRank self;
  int P, sh, me_real;
  int64_t n, inbox_cap;
  int32_t source;
  double delta;
  gfx_iter_rec* recs;
  int64_t rec_cap;
  long long* summary;
  unsigned epoch_base;
};

struct PsCtl {
  long long nnear, nfar_loc, gnear, gfar, it, ph, slots, nrec, nadv, messages;
  int q, f;
  double th;
  unsigned long long t0;
  unsigned epoch;
  PsRank R;
};

__device__ __forceinline__ unsigned long long ps_gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <bool kVirt>
struct PsSync {
  cg::grid_group& grid;
  __device__ __forceinline__ void rank() { grid.sync(); }
  __device__ __forceinline__ void all(const PsArgs& a, PsCtl& c, int me) {
    if (kVirt || a.P == 1) {
      grid.sync();
      return;
    }
    __threadfence_system();
    grid.sync();
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      const unsigned e = ++c.epoch;
      for (int q = 0; q < a.P; ++q)
        if (q != me)
          asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(&a.rk[q].flags[me]), "r"(e)
                       : "memory");
      for (int q = 0; q < a.P; ++q) {
        if (q == me) continue;
        unsigned v;
        do {
          asm volatile("ld.acquire.sys.global.u32 %0, [%1];"
                       : "=r"(v)
                       : "l"(&a.rk[me].flags[q])
                       : "memory");
        } while ((int)(v - e) < 0);
      }
    }
    if (threadIdx.x == 0 && blockIdx.x != 0) ++c.epoch;
    grid.sync();
  }
};

// relax: owned targets in place (enqueued once per iteration), remote ones
// through the monotone offer filter (emitted once per iteration)
struct PsRelaxOp {
  static constexpr bool kWeights = true, kSrcVal = true, kEmitEdge = false;
  static constexpr int kBatch = 4;
  static constexpr int kMinBlocks = 3;
  unsigned long long* dp;
  uint32_t* dist;
  unsigned long long* sent_key;
  uint32_t* sent;
  int P, r, sh;
  uint32_t cur[kBatch];
  __device__ __forceinline__ int owner(int32_t d) const { return sh >= 0 ? (d & (P - 1)) : d % P; }
  __device__ __forceinline__ int32_t local(int32_t d) const { return sh >= 0 ? (d >> sh) : d / P; }
  __device__ int32_t src_value(int32_t l) const { return (int32_t)dist[l]; }
  __device__ void prefetch(const int32_t* d) {
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      if (d[u] < 0) cur[u] = 0u;
      else if (P == 1 || owner(d[u]) == r) cur[u] = dist[P == 1 ? d[u] : local(d[u])];
      else cur[u] = (uint32_t)(sent_key[d[u]] >> 32);
    }
  }
  __device__ bool visit(int u, int32_t d, int32_t s, int32_t w, int32_t sdist, int64_t) {
    const unsigned long long nd = (unsigned long long)(uint32_t)sdist + (uint32_t)w;
    if (nd >= cur[u]) return false;
    const unsigned long long key = (nd << 32) | (uint32_t)(s * P + r);
    if (P == 1 || owner(d) == r) {
      // every improving relaxation is emitted; the split keeps each vertex
      // once per iteration (no atomic round trip on the relax chain)
      const int32_t l = P == 1 ? d : local(d);
      atomicMin(&dp[l], key);
      atomicMin(&dist[l], (uint32_t)nd);
      return true;
    }
    atomicMin(&sent_key[d], key);
    const uint32_t bit = 1u << (d & 31);
    return !(atomicOr(&sent[d >> 5], bit) & bit);
  }
};

// block-staged near / far appends (near_far.py:40-57 split, 68-85 re-split);
// cta / ncta: this rank's CTAs (virtual ranks share the grid)
constexpr int kPsStage = 1024;
struct PsStage {
  int32_t nv[kPsStage];
  int32_t fv[kPsStage], fk[kPsStage];
  int nn, nfar;
  unsigned long long base;
};

__device__ __forceinline__ void ps_flush(PsStage& S, int32_t* near, unsigned long long* near_len,
                                         int32_t* far, int32_t* fkey,
                                         unsigned long long* far_len) {
  __syncthreads();
  if (threadIdx.x == 0) S.base = S.nn ? atomicAdd(near_len, (unsigned long long)S.nn) : 0ull;
  __syncthreads();
  for (int i = threadIdx.x; i < S.nn; i += blockDim.x) near[S.base + i] = S.nv[i];
  __syncthreads();
  if (threadIdx.x == 0) S.base = S.nfar ? atomicAdd(far_len, (unsigned long long)S.nfar) : 0ull;
  __syncthreads();
  for (int i = threadIdx.x; i < S.nfar; i += blockDim.x) {
    far[S.base + i] = S.fv[i];
    fkey[S.base + i] = S.fk[i];
  }
  __syncthreads();
  if (threadIdx.x == 0) S.nn = S.nfar = 0;
  __syncthreads();
}

// mode 0: split touched[0..n) at the threshold (clearing marks); mode 1:
// re-split the far pile (stale entries dropped); mode 2: compact the far
// pile (stale entries dropped, everything stays far)
__device__ __forceinline__ void ps_pile(PsStage& S, int mode, const int32_t* src,
                                        const int32_t* skey, int64_t n, const uint32_t* dist,
                                        int32_t* stamp, int32_t it, double th, int32_t* near,
                                        unsigned long long* near_len, int32_t* far, int32_t* fkey,
                                        unsigned long long* far_len, int64_t cta, int64_t ncta) {
  if (threadIdx.x == 0) S.nn = S.nfar = 0;
  __syncthreads();
  for (int64_t base = cta * blockDim.x; base < n; base += ncta * blockDim.x) {
    const int64_t i = base + threadIdx.x;
    if (i < n) {
      const int32_t v = src[i];
      const int32_t key = (int32_t)dist[v];
      bool keep = true;
      if (mode == 0) keep = atomicExch(&stamp[v], it) != it;  // first occurrence this iteration
      else keep = key == skey[i];                              // fresh far entries only
      if (keep) {
        if (mode != 2 && (double)key < th) {
          S.nv[atomicAdd(&S.nn, 1)] = v;
        } else {
          const int at = atomicAdd(&S.nfar, 1);
          S.fv[at] = v;
          S.fk[at] = key;
        }
      }
    }
    __syncthreads();
    if (S.nn > kPsStage - (int)blockDim.x || S.nfar > kPsStage - (int)blockDim.x)
      ps_flush(S, near, near_len, far, fkey, far_len);
  }
  ps_flush(S, near, near_len, far, fkey, far_len);
}

template <bool kVirt, bool kMulti>
__global__ void __launch_bounds__(256, 3) k_pdsssp(PsArgs a) {
  cg::grid_group grid = cg::this_grid();
  PsSync<kVirt> sync{grid};
  extern __shared__ __align__(16) unsigned char smem_raw[];
  WarpSmem& W = warp_smem(smem_raw);
  static_assert(sizeof(PsStage) <= sizeof(WarpSmem) * kWarpsPerBlock, "pile stage must fit");
  PsStage& S = *reinterpret_cast<PsStage*>(smem_raw);  // aliases the warp slices (other phases)
  __shared__ ScanSmem ss;
  __shared__ PsCtl c;
  __shared__ CtaAgg agg;
  const int P = kMulti ? a.P : 1;
  const int me = kVirt ? (int)(blockIdx.x % P) : a.me_real;
  const int64_t rcta = kVirt ? blockIdx.x / P : blockIdx.x;
  const int64_t nrcta = kVirt ? gridDim.x / P : gridDim.x;
  const int64_t gtid = rcta * blockDim.x + threadIdx.x;
  const int64_t nthr = nrcta * blockDim.x;
  const int64_t gw = gtid >> 5, nw = nthr >> 5;
  const bool rlead = rcta == 0 && threadIdx.x == 0;
  const bool leader = blockIdx.x == 0 && threadIdx.x == 0;
  if (threadIdx.x == 0) {
    if (kVirt) c.R = a.rk[me];
    c.epoch = a.epoch_base;
  }
  if (threadIdx.x < 8) agg.ctr[threadIdx.x] = 0ull;
  __syncthreads();
  const PsRank& R = kVirt ? c.R : a.self;
  const int32_t src_owner = a.sh >= 0 ? (a.source & (P - 1)) : a.source % P;
  const int32_t src_local = a.sh >= 0 ? (a.source >> a.sh) : a.source / P;
  const int lane = threadIdx.x & 31;

  // ---- init
  for (int64_t l = gtid; l < R.nl; l += nthr) {
    R.dp[l] = ~0ull;
    R.dist[l] = 0xFFFFFFFFu;
  }
  for (int64_t l = gtid; l < R.nl; l += nthr) R.stamp[l] = 0;
  if (kMulti) {
    for (int64_t i = gtid; i < a.n; i += nthr) R.sent_key[i] = ~0ull;
    for (int64_t w = gtid; w < (a.n + 31) / 32 + 1; w += nthr) R.sent[w] = 0u;
  }
  for (int64_t i = gtid; i < 3 * (int64_t)(sizeof(Counters) / 8); i += nthr)
    reinterpret_cast<unsigned long long*>(R.C)[i] = 0ull;
  for (int64_t i = gtid; i < P; i += nthr) {
    R.outcnt[i] = 0ull;
    R.inbox_cnt[i] = 0ull;
  }
  sync.all(a, c, me);
  if (rlead && me == src_owner) {
    R.dp[src_local] = 0xFFFFFFFFull;  // dist 0, pred -1
    R.dist[src_local] = 0u;
    R.nearq[0][0] = src_local;
  }
  if (threadIdx.x == 0) {
    c.nnear = me == src_owner ? 1 : 0;
    c.gnear = 1;
    c.nfar_loc = c.gfar = 0;
    c.it = c.ph = c.slots = c.nrec = c.nadv = c.messages = 0;
    c.q = c.f = 0;
    c.th = a.delta;
  }
  sync.rank();

  for (;;) {
    Counters* cur = &R.C[c.ph % 3];
    if (rcta == 0 && threadIdx.x < (int)(sizeof(Counters) / 8))
      reinterpret_cast<unsigned long long*>(&R.C[(c.ph + 1) % 3])[threadIdx.x] = 0ull;
    long long near_loc = 0, far_loc = 0, slots_loc = 0, touched_loc = 0;
    const bool advance = c.gnear == 0;
    if (advance && c.gfar == 0) break;
    if (advance) {
      // advance_bucket (near_far.py:63-85): threshold += delta, stale far
      // entries dropped, the rest re-split
      const double th = c.th + a.delta;
      ps_pile(S, 1, R.far[c.f], R.fkey[c.f], c.nfar_loc, R.dist, R.stamp, 0, th, R.nearq[c.q],
              &cur->out_len, R.far[c.f ^ 1], R.fkey[c.f ^ 1], &cur->aux1, rcta, nrcta);
      sync.rank();
      cta_read_ctrs(agg, cur);
      near_loc = (long long)agg.rd[0];
      far_loc = (long long)agg.rd[5];
      if (threadIdx.x == 0) {
        c.th = th;
        c.f ^= 1;
        c.nadv += 1;
      }
    } else {
      if (threadIdx.x == 0) {
        c.it += 1;
        c.t0 = ps_gtime();
      }
      __syncthreads();
      const int32_t* F = R.nearq[c.q];
      const int64_t nf = c.nnear;
      const int64_t stiles = (nf + kScanTileItems - 1) / kScanTileItems;
      for (int64_t t = rcta; t < stiles; t += nrcta)
        scan_tile(t, stiles, F, nf, R.row, R.scan, R.rowbase, R.part, R.status,
                  a.epoch_base + (unsigned)c.ph + 1u, cur, ss);
      sync.rank();
      cta_read_ctrs(agg, cur);
      {
        PsRelaxOp op{R.dp, R.dist, R.sent_key, R.sent, P, me, a.sh, {}};
        expand_tasks(W, op, F, nf, R.scan, R.rowbase, R.part, (int64_t)agg.rd[3],
                     (int64_t)agg.rd[2], R.col, R.w, kMulti ? R.emit : R.touched, &cur->out_len,
                     gw, nw, &agg);
      }
      for (int64_t i = gtid; i < stiles; i += nthr) R.status[i] = 0ull;
      sync.rank();
      cta_read_ctrs(agg, cur);
      slots_loc = (long long)agg.rd[2];
      unsigned long long* tlen = &cur->out_len;  // touched count (P = 1: the expansion's)
      if constexpr (kMulti) {
        // owned improved -> touched (local ids); remote -> messages to owners
        tlen = &cur->aux2;
        const int64_t nemit = (int64_t)agg.rd[0];
        PsRelaxOp op{R.dp, R.dist, R.sent_key, R.sent, P, me, a.sh, {}};
        for (int64_t base = gw * 32; base < nemit; base += nw * 32) {
          const int64_t i = base + lane;
          const bool ok = i < nemit;
          const int32_t d = ok ? R.emit[i] : 0;
          const int o = ok ? op.owner(d) : 64;
          const unsigned peers = __match_any_sync(0xffffffffu, o);
          const int lead = __ffs(peers) - 1;
          const int rank_in = __popc(peers & ((1u << lane) - 1));
          unsigned long long at = 0;
          if (ok && lane == lead)
            at = atomicAdd(o == me ? tlen : &R.outcnt[o], (unsigned long long)__popc(peers));
          at = __shfl_sync(0xffffffffu, at, lead) + rank_in;
          if (ok) {
            if (o == me) {
              R.touched[at] = op.local(d);
            } else {
              unsigned long long* msg = a.rk[o].inbox + 2 * ((int64_t)me * a.inbox_cap + at);
              msg[0] = (unsigned long long)(uint32_t)d;
              msg[1] = R.sent_key[d];
              atomicAnd(&R.sent[d >> 5], ~(1u << (d & 31)));
            }
          }
        }
        sync.rank();
        if (rlead) {
          long long sent_total = 0;
          for (int o = 0; o < P; ++o)
            if (o != me) {
              a.rk[o].inbox_cnt[me] = R.outcnt[o];
              sent_total += (long long)R.outcnt[o];
              R.outcnt[o] = 0ull;
            }
          c.messages += sent_total;
        }
        sync.all(a, c, me);  // every inbox complete
        // apply the offers (sssp.py:95-103 semantics, owner side)
        for (int q = 0; q < P; ++q) {
          if (q == me) continue;
          const int64_t cnt = (int64_t)R.inbox_cnt[q];
          const unsigned long long* box = R.inbox + 2 * (int64_t)q * a.inbox_cap;
          for (int64_t base = gtid & ~31ll; base < cnt; base += nthr) {
            const int64_t i = base + lane;
            bool em = false;
            int32_t l = 0;
            if (i < cnt) {
              const int32_t d = (int32_t)box[2 * i];
              const unsigned long long key = box[2 * i + 1];
              l = op.local(d);
              const uint32_t nd = (uint32_t)(key >> 32);
              if (nd < R.dist[l]) {
                atomicMin(&R.dp[l], key);
                atomicMin(&R.dist[l], nd);
                em = true;  // deduplicated in the split
              }
            }
            const unsigned wm = __ballot_sync(0xffffffffu, em);
            unsigned long long b = 0;
            if (lane == 0 && wm) b = atomicAdd(tlen, (unsigned long long)__popc(wm));
            b = __shfl_sync(0xffffffffu, b, 0);
            if (em) R.touched[b + __popc(wm & ((1u << lane) - 1))] = l;
          }
        }
        sync.rank();
        cta_read_ctrs(agg, cur);
      }
      touched_loc = (long long)agg.rd[kMulti ? 6 : 0];
      // split the improved vertices at the (global) threshold; far appends
      // go behind the rank's far pile
      ps_pile(S, 0, R.touched, nullptr, touched_loc, R.dist, R.stamp, (int32_t)c.it, c.th,
              R.nearq[c.q ^ 1],
              &cur->aux0, R.far[c.f] + c.nfar_loc, R.fkey[c.f] + c.nfar_loc, &cur->aux1, rcta,
              nrcta);
      sync.rank();
      cta_read_ctrs(agg, cur);
      near_loc = (long long)agg.rd[4];
      far_loc = c.nfar_loc + (long long)agg.rd[5];
      touched_loc = (long long)(agg.rd[4] + agg.rd[5]);  // improved vertices, each once
      if (threadIdx.x == 0) c.q ^= 1;
    }
    // ---- global sums (near, far, slots, touched) over the ranks
    long long g_near = near_loc, g_far = far_loc, g_slots = slots_loc, g_touched = touched_loc;
    if constexpr (kMulti) {
      const int par = (int)(c.ph & 1);
      if (rlead)
        for (int q = 0; q < P; ++q) {
          long long* row = a.rk[q].ctab + ((int64_t)par * kPsMaxRanks + me) * 4;
          row[0] = near_loc;
          row[1] = far_loc;
          row[2] = slots_loc;
          row[3] = touched_loc;
        }
      sync.all(a, c, me);
      g_near = g_far = g_slots = g_touched = 0;
      for (int q = 0; q < P; ++q) {
        const unsigned long long* row = reinterpret_cast<const unsigned long long*>(
            R.ctab + ((int64_t)par * kPsMaxRanks + q) * 4);
        g_near += (long long)ld_volatile_u64(row);
        g_far += (long long)ld_volatile_u64(row + 1);
        g_slots += (long long)ld_volatile_u64(row + 2);
        g_touched += (long long)ld_volatile_u64(row + 3);
      }
    }
    if (!advance && leader && c.nrec < a.rec_cap) {
      gfx_iter_rec rec{};
      rec.iteration = c.it;
      rec.frontier_in = c.gnear;
      rec.frontier_out = g_touched;
      rec.edges = g_slots;
      rec.work = g_slots;
      rec.bytes_alg = 20 * c.gnear + 8 * g_slots + 8 * g_touched;
      rec.n_u = g_far;
      rec.ms = (float)((ps_gtime() - c.t0) * 1e-6);
      a.recs[c.nrec] = rec;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      if (!advance) {
        c.nrec += 1;
        c.slots += g_slots;
      }
      c.nnear = near_loc;
      c.nfar_loc = far_loc;
      c.gnear = g_near;
      c.gfar = g_far;
      c.ph += 1;
    }
    __syncthreads();
    // capacity guard (global decision, so every rank runs the same
    // barriers): a far pile past half its capacity drops its stale entries
    long long far_max = c.nfar_loc;
    if constexpr (kMulti) {
      // every rank's far count is in the table row just summed
      const int par = (int)((c.ph - 1) & 1);
      far_max = 0;
      for (int q = 0; q < P; ++q)
        far_max = max(far_max, (long long)ld_volatile_u64(reinterpret_cast<const unsigned long long*>(
                                   R.ctab + ((int64_t)par * kPsMaxRanks + q) * 4 + 1)));
    }
    if (far_max > R.far_cap / 2) {
      Counters* g2 = &R.C[c.ph % 3];
      if (rcta == 0 && threadIdx.x < (int)(sizeof(Counters) / 8))
        reinterpret_cast<unsigned long long*>(&R.C[(c.ph + 1) % 3])[threadIdx.x] = 0ull;
      ps_pile(S, 2, R.far[c.f], R.fkey[c.f], c.nfar_loc, R.dist, R.stamp, 0, c.th, nullptr,
              &g2->aux2, R.far[c.f ^ 1], R.fkey[c.f ^ 1], &g2->aux1, rcta, nrcta);
      sync.rank();
      cta_read_ctrs(agg, g2);
      if (threadIdx.x == 0) {
        c.nfar_loc = (long long)agg.rd[5];
        c.f ^= 1;
        c.ph += 1;
      }
      __syncthreads();
    }
  }
  // (dist | pred) -> the int32 outputs (local ids)
  for (int64_t l = gtid; l < R.nl; l += nthr) {
    const unsigned long long x = R.dp[l];
    const uint32_t d = (uint32_t)(x >> 32);
    R.out_dist[l] = d == 0xFFFFFFFFu ? GFX_UNVISITED : (int32_t)d;
    R.out_preds[l] = (int32_t)(uint32_t)x;
  }
  if (leader) {
    a.summary[0] = c.it;
    a.summary[1] = c.slots;
    a.summary[2] = c.nadv;
    a.summary[3] = c.nrec < a.rec_cap ? c.nrec : a.rec_cap;
    a.summary[4] = c.messages;
  }
}

}  // namespace gfx

using namespace gfx;

struct gfx_pdsssp {
  gfx_ctx* ctx = nullptr;
  int P = 1, me = 0, virt = 1;
  int64_t n = 0, inbox_cap = 0;
  std::vector<std::vector<void*>> bufs;
  std::vector<PsRank> rk;
  PsRank* rk_d = nullptr;
  gfx_iter_rec* recs_d = nullptr;
  long long* summary_d = nullptr;
  int64_t rec_cap = 1 << 14;
  unsigned epoch = 0;
  int grid = 0, smem = 0;
  std::vector<void*> ipc_opened;
};

namespace {

template <class T>
int ps_alloc(std::vector<void*>& bufs, size_t count, T** out) {
  void* p = nullptr;
  GFX_CK(cudaMalloc(&p, count * sizeof(T) + 16));
  bufs.push_back(p);
  *out = static_cast<T*>(p);
  return GFX_OK;
}

int ps_setup_rank(gfx_pdsssp* e, const int64_t* lrow, const int32_t* lcol, const int32_t* lw,
                  int64_t nl, int64_t ml, std::vector<void*>& bufs, PsRank& R) {
  std::memset(&R, 0, sizeof(R));
  R.row = lrow;
  R.col = lcol;
  R.w = lw;
  R.nl = nl;
  R.wl = (nl + 31) / 32;
  R.far_cap = 2 * nl + 2;
  GFX_TRY(ps_alloc(bufs, nl + 1, &R.dp));
  GFX_TRY(ps_alloc(bufs, nl + 1, &R.dist));
  GFX_TRY(ps_alloc(bufs, nl + 1, &R.stamp));
  if (e->P > 1) {
    GFX_TRY(ps_alloc(bufs, (size_t)e->n + 1, &R.sent_key));
    GFX_TRY(ps_alloc(bufs, (size_t)(e->n + 31) / 32 + 2, &R.sent));
    GFX_TRY(ps_alloc(bufs, (size_t)(ml + e->n) + 1, &R.emit));  // owned duplicates + remote firsts
  }
  for (int k = 0; k < 2; ++k) {
    GFX_TRY(ps_alloc(bufs, nl + 1, &R.nearq[k]));
    GFX_TRY(ps_alloc(bufs, R.far_cap + 1, &R.far[k]));
    GFX_TRY(ps_alloc(bufs, R.far_cap + 1, &R.fkey[k]));
  }
  // duplicates allowed: every owned improving relaxation and every applied offer
  GFX_TRY(ps_alloc(bufs, (size_t)(ml + nl + e->P * e->inbox_cap) + 1, &R.touched));
  GFX_TRY(ps_alloc(bufs, nl + 2, &R.scan));
  GFX_TRY(ps_alloc(bufs, nl + 1, &R.rowbase));
  GFX_TRY(ps_alloc(bufs, part_capacity(ml, nl), &R.part));
  const int64_t stiles = std::max<int64_t>(1, (nl + kScanTileItems - 1) / kScanTileItems);
  GFX_TRY(ps_alloc(bufs, stiles + 1, &R.status));
  GFX_CK(cudaMemsetAsync(R.status, 0, (stiles + 1) * 8, e->ctx->stream));
  GFX_TRY(ps_alloc(bufs, 3 * sizeof(Counters) / 8, reinterpret_cast<unsigned long long**>(&R.C)));
  GFX_TRY(ps_alloc(bufs, kPsMaxRanks, &R.outcnt));
  GFX_TRY(ps_alloc(bufs, nl + 1, &R.out_dist));
  GFX_TRY(ps_alloc(bufs, nl + 1, &R.out_preds));
  GFX_TRY(ps_alloc(bufs, 2 * ((size_t)e->P * e->inbox_cap + 1), &R.inbox));
  GFX_TRY(ps_alloc(bufs, kPsMaxRanks, &R.inbox_cnt));
  GFX_TRY(ps_alloc(bufs, 2 * kPsMaxRanks * 4, &R.ctab));
  GFX_TRY(ps_alloc(bufs, kPsMaxRanks, &R.flags));
  GFX_CK(cudaMemsetAsync(R.flags, 0, kPsMaxRanks * 4, e->ctx->stream));
  GFX_CK(cudaMemsetAsync(R.ctab, 0, 2 * kPsMaxRanks * 4 * 8, e->ctx->stream));
  return GFX_OK;
}

const void* ps_kernel(const gfx_pdsssp* e) {
  if (e->P == 1) return (const void*)k_pdsssp<false, false>;
  return e->virt ? (const void*)k_pdsssp<true, true> : (const void*)k_pdsssp<false, true>;
}

int ps_finish(gfx_pdsssp* e) {
  GFX_CK(cudaMalloc(&e->rk_d, sizeof(PsRank) * e->P));
  GFX_CK(cudaMalloc(&e->recs_d, sizeof(gfx_iter_rec) * e->rec_cap));
  GFX_CK(cudaMalloc(&e->summary_d, sizeof(long long) * 8));
  const int smem = (int)sizeof(WarpSmem) * kWarpsPerBlock;
  int per_sm = 0;
  GFX_CK(cudaFuncSetAttribute(ps_kernel(e), cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  GFX_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ps_kernel(e), 256, smem));
  GFX_REQUIRE(per_sm >= 1, "k_pdsssp cannot be resident");
  e->grid = per_sm * e->ctx->sm_count;
  if (e->virt) e->grid = e->grid / e->P * e->P;
  e->smem = smem;
  GFX_CK(cudaMemcpyAsync(e->rk_d, e->rk.data(), sizeof(PsRank) * e->P, cudaMemcpyHostToDevice,
                         e->ctx->stream));
  return GFX_OK;
}

int ps_launch(gfx_pdsssp* e, int64_t source, double delta) {
  PsArgs a{};
  a.rk = e->rk_d;
  a.self = e->rk[e->virt ? 0 : e->me];
  a.P = e->P;
  a.sh = -1;
  if ((e->P & (e->P - 1)) == 0) {
    a.sh = 0;
    while ((1 << a.sh) < e->P) ++a.sh;
  }
  a.me_real = e->me;
  a.n = e->n;
  a.inbox_cap = e->inbox_cap;
  a.source = (int32_t)source;
  a.delta = delta;
  a.recs = e->recs_d;
  a.rec_cap = e->rec_cap;
  a.summary = e->summary_d;
  a.epoch_base = e->epoch;
  e->epoch += 1u << 20;  // per run: scan epochs and exchange-barrier epochs
  void* kargs[] = {&a};
  GFX_CK(cudaLaunchCooperativeKernel(ps_kernel(e), dim3(e->grid), dim3(256), kargs, e->smem,
                                     e->ctx->stream));
  count_launch();
  return GFX_OK;
}

}  // namespace

extern "C" {

int gfx_pdsssp_destroy(gfx_pdsssp* e) {
  if (!e) return GFX_OK;
  cudaSetDevice(e->ctx->device);
  cudaStreamSynchronize(e->ctx->stream);
  for (void* p : e->ipc_opened) cudaIpcCloseMemHandle(p);
  for (auto& b : e->bufs)
    for (void* p : b) cudaFree(p);
  cudaFree(e->rk_d);
  cudaFree(e->recs_d);
  cudaFree(e->summary_d);
  delete e;
  return GFX_OK;
}

int gfx_pdsssp_create_virtual(gfx_ctx* ctx, int64_t n, int P, const int64_t* const* lrow,
                              const int32_t* const* lcol, const int32_t* const* lw,
                              const int64_t* n_local, const int64_t* m_local, gfx_pdsssp** out) {
  GFX_NVTX("gfx_pdsssp_create_virtual");
  GFX_REQUIRE(ctx && lrow && lcol && lw && n_local && m_local && out,
              "gfx_pdsssp_create_virtual: null argument");
  GFX_REQUIRE(P >= 1 && P <= kPsMaxRanks, "P=%d out of range 1..%d", P, kPsMaxRanks);
  GFX_REQUIRE(n > 0 && n < (int64_t)INT32_MAX, "n=%lld out of range", (long long)n);
  for (int q = 0; q < P; ++q)
    GFX_REQUIRE(n_local[q] == (n > q ? (n - q + P - 1) / P : 0), "n_local[%d] does not match", q);
  GFX_CK(cudaSetDevice(ctx->device));
  auto* e = new gfx_pdsssp();
  e->ctx = ctx;
  e->P = P;
  e->virt = 1;
  e->n = n;
  e->inbox_cap = (n + P - 1) / P + 1;
  e->bufs.resize(P);
  e->rk.resize(P);
  for (int q = 0; q < P; ++q) {
    const int st = ps_setup_rank(e, lrow[q], lcol[q], lw[q], n_local[q], m_local[q], e->bufs[q],
                                 e->rk[q]);
    if (st != GFX_OK) {
      gfx_pdsssp_destroy(e);
      return st;
    }
  }
  const int st = ps_finish(e);
  if (st != GFX_OK) {
    gfx_pdsssp_destroy(e);
    return st;
  }
  GFX_CK(cudaStreamSynchronize(ctx->stream));
  *out = e;
  return GFX_OK;
}

int gfx_pdsssp_create_rank(gfx_ctx* ctx, int64_t n, int P, int r, const int64_t* lrow,
                           const int32_t* lcol, const int32_t* lw, int64_t n_local,
                           int64_t m_local, gfx_pdsssp** out) {
  GFX_NVTX("gfx_pdsssp_create_rank");
  GFX_REQUIRE(ctx && lrow && out, "gfx_pdsssp_create_rank: null argument");
  GFX_REQUIRE(P >= 1 && P <= kPsMaxRanks && r >= 0 && r < P, "bad partition P=%d r=%d", P, r);
  GFX_REQUIRE(n_local == (n > r ? (n - r + P - 1) / P : 0), "n_local does not match the partition");
  GFX_CK(cudaSetDevice(ctx->device));
  auto* e = new gfx_pdsssp();
  e->ctx = ctx;
  e->P = P;
  e->me = r;
  e->virt = 0;
  e->n = n;
  e->inbox_cap = (n + P - 1) / P + 1;
  e->bufs.resize(1);
  e->rk.assign(P, PsRank{});
  int st = ps_setup_rank(e, lrow, lcol, lw, n_local, m_local, e->bufs[0], e->rk[r]);
  if (st == GFX_OK) st = ps_finish(e);
  if (st != GFX_OK) {
    gfx_pdsssp_destroy(e);
    return st;
  }
  GFX_CK(cudaStreamSynchronize(ctx->stream));
  *out = e;
  return GFX_OK;
}

// 4 cudaIpcMemHandle_t (inbox, inbox counts, counter table, flags)
int gfx_pdsssp_export(gfx_pdsssp* e, void* handles) {
  GFX_REQUIRE(e && handles && !e->virt, "gfx_pdsssp_export: real-rank engine required");
  const PsRank& R = e->rk[e->me];
  void* bases[4] = {R.inbox, R.inbox_cnt, R.ctab, R.flags};
  auto* h = static_cast<cudaIpcMemHandle_t*>(handles);
  for (int k = 0; k < 4; ++k) GFX_CK(cudaIpcGetMemHandle(&h[k], bases[k]));
  return GFX_OK;
}

int gfx_pdsssp_import(gfx_pdsssp* e, const void* all_handles) {
  GFX_REQUIRE(e && all_handles && !e->virt, "gfx_pdsssp_import: real-rank engine required");
  GFX_CK(cudaSetDevice(e->ctx->device));
  const auto* h = static_cast<const cudaIpcMemHandle_t*>(all_handles);
  for (int q = 0; q < e->P; ++q) {
    if (q == e->me) continue;
    void* p[4];
    for (int k = 0; k < 4; ++k) {
      GFX_CK(cudaIpcOpenMemHandle(&p[k], h[q * 4 + k], cudaIpcMemLazyEnablePeerAccess));
      e->ipc_opened.push_back(p[k]);
    }
    PsRank& Q = e->rk[q];
    std::memset(&Q, 0, sizeof(Q));
    Q.inbox = static_cast<unsigned long long*>(p[0]);
    Q.inbox_cnt = static_cast<unsigned long long*>(p[1]);
    Q.ctab = static_cast<long long*>(p[2]);
    Q.flags = static_cast<unsigned*>(p[3]);
  }
  GFX_CK(cudaMemcpyAsync(e->rk_d, e->rk.data(), sizeof(PsRank) * e->P, cudaMemcpyHostToDevice,
                         e->ctx->stream));
  GFX_CK(cudaStreamSynchronize(e->ctx->stream));
  return GFX_OK;
}

// One SSSP (delta: near/far bucket width; <= 0 or inf: one bucket).
// dist_d[k] / preds_d[k]: rank k's (virtual) or this rank's (real, k = 0)
// int32 distances / global preds over local ids.
int gfx_pdsssp_run(gfx_pdsssp* e, int64_t source, double delta, int32_t* const* dist_d,
                   int32_t* const* preds_d, gfx_iter_rec* recs, int64_t rec_cap, gfx_stats* st) {
  GFX_NVTX("gfx_pdsssp_run");
  GFX_REQUIRE(e, "gfx_pdsssp_run: null engine");
  GFX_REQUIRE(source >= 0 && source < e->n, "source %lld out of range", (long long)source);
  if (!(delta > 0)) delta = INFINITY;
  gfx_ctx* ctx = e->ctx;
  GFX_CK(cudaSetDevice(ctx->device));
  GFX_CK(cudaEventRecord(ctx->ev0, ctx->stream));
  GFX_TRY(ps_launch(e, source, delta));
  GFX_CK(cudaEventRecord(ctx->ev1, ctx->stream));
  long long summary[8];
  GFX_CK(cudaMemcpyAsync(summary, e->summary_d, sizeof(summary), cudaMemcpyDeviceToHost,
                         ctx->stream));
  const int nr = e->virt ? e->P : 1;
  for (int k = 0; k < nr; ++k) {
    const PsRank& R = e->rk[e->virt ? k : e->me];
    if (dist_d && dist_d[k])
      GFX_CK(cudaMemcpyAsync(dist_d[k], R.out_dist, R.nl * 4, cudaMemcpyDeviceToDevice, ctx->stream));
    if (preds_d && preds_d[k])
      GFX_CK(cudaMemcpyAsync(preds_d[k], R.out_preds, R.nl * 4, cudaMemcpyDeviceToDevice,
                             ctx->stream));
  }
  GFX_CK(cudaStreamSynchronize(ctx->stream));
  float ms = 0.f;
  GFX_CK(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
  const int64_t nrec = std::min<int64_t>(summary[3], recs ? rec_cap : 0);
  if (nrec > 0)
    GFX_CK(cudaMemcpy(recs, e->recs_d, nrec * sizeof(gfx_iter_rec), cudaMemcpyDeviceToHost));
  if (st) {
    std::memset(st, 0, sizeof(*st));
    st->iterations = summary[0];
    st->work_slots = summary[1];
    st->edges_traversed = summary[1];
    st->direction_switches = summary[2];  // bucket advances
    st->reached = summary[4];             // messages exchanged
    st->device_ms = ms;
    st->num_records = nrec;
  }
  return GFX_OK;
}

int gfx_pdsssp_batch(gfx_pdsssp* e, int64_t source, int64_t count, double delta, float* ms) {
  GFX_NVTX("gfx_pdsssp_batch");
  GFX_REQUIRE(e && ms && count > 0, "gfx_pdsssp_batch: bad argument");
  GFX_REQUIRE(source >= 0 && source < e->n, "source %lld out of range", (long long)source);
  if (!(delta > 0)) delta = INFINITY;
  gfx_ctx* ctx = e->ctx;
  GFX_CK(cudaSetDevice(ctx->device));
  GFX_CK(cudaEventRecord(ctx->ev0, ctx->stream));
  for (int64_t k = 0; k < count; ++k) GFX_TRY(ps_launch(e, source, delta));
  GFX_CK(cudaEventRecord(ctx->ev1, ctx->stream));
  GFX_CK(cudaEventSynchronize(ctx->ev1));
  GFX_CK(cudaEventElapsedTime(ms, ctx->ev0, ctx->ev1));
  return GFX_OK;
}

}  // extern "C"
