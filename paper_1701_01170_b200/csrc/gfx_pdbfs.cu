// Device-resident partitioned direction-optimising BFS (the
// "low-latency path": kernels exchange through peer memory and device flags
// instead of one host-launched collective per level).
//
// Same partition and protocol as the host-driven engine (gfx_dist.cu,
// dist.py): 1D cyclic ownership owner(v) = v mod P, rank r keeps the rows of
// its owned vertices (local id l = v / P) with global column ids.  ONE
// cooperative launch per rank runs the whole BFS.  Per level, in lockstep:
//   * every CTA takes the reference direction decision (direction.py:52-70)
//     from the GLOBAL counters, so all ranks take the same one;
//   * push: the rank expands its local queue; owned targets are claimed in
//     place, remote ones are de-duplicated through a per-level bitmap over
//     global ids and written as (dst, src) pairs straight into the owner's
//     inbox region for this sender (peer stores); after the exchange barrier
//     the owner claims its inbox;
//   * pull: the rank pulls its unvisited vertices against its copy of the
//     frontier, stored as P slices (slice q = rank q's vertices in local-id
//     order), with the single-GPU pull body (gfx_pull.cuh);
//   * end of level: the rank writes its slice of the next frontier and its
//     level counters into every rank's copy (peer stores), one exchange
//     barrier, then every CTA sums the P counter rows.
// Two execution modes, one kernel body:
//   * real ranks (one process per GPU): the peer buffers are CUDA-IPC
//     mappings, the intra-rank barrier is the cooperative grid barrier and
//     the exchange barrier adds release/acquire flags over NVLink;
//   * virtual ranks (P ranks inside ONE launch on one GPU, CTA b runs rank
//     b mod P): every barrier is the grid barrier.  This runs the complete
//     multi-rank protocol -- the same code paths, buffers and exchange
//     stores -- on a single GPU; the tests check it against the one-GPU BFS
//     and the reference goldens.
// At P = 1 the exchange steps vanish and the kernel is the single-GPU level
// loop over the partitioned layout.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "gfx_device.cuh"
#include "gfx_direction.cuh"
#include "gfx_expand.cuh"
#include "gfx_internal.cuh"
#include "gfx_pull.cuh"
#include "gfx_scan.cuh"

namespace gfx {
namespace cg = cooperative_groups;

constexpr int kPdMaxRanks = 8;

// one rank's buffers; the exchange block is valid on every rank (own or
// peer-mapped), the rest only where the rank executes
struct PdRank {
  const int64_t* row;
  const int32_t* col;
  const int32_t* head;   // first / second neighbour per local row (k_dist_heads layout)
  const int32_t* head2;
  const uint32_t* nz;    // local rows with degree > 0
  uint32_t* visited;     // local ids
  int32_t* labels;       // local ids, int32 (UNVISITED / depth), written at the end
  uint8_t* lvl8;         // local ids: depth bytes while labels are deferred
  int32_t* preds;        // local ids -> global parent, -1
  int32_t* order;        // local queue, every level's frontier concatenated
  int32_t* emit;         // push output before the owner split (global ids)
  int64_t* scan;
  int64_t* rowbase;
  int32_t* part;
  unsigned long long* status;
  uint32_t* sent;        // remote targets emitted this level (global ids)
  int32_t* sent_src;
  Counters* C;           // 3 rotating blocks
  unsigned long long* outcnt;  // pairs written per owner this level
  int64_t nl, wl, nnz;
  // exchange block
  uint32_t* gfront[3];           // P slices x wmax words
  unsigned long long* inbox;     // P regions x inbox_cap pairs (region q: from rank q)
  unsigned long long* inbox_cnt; // pairs per sender region
  long long* ctab;               // [2][kPdMaxRanks][4] level counters of every rank
  unsigned* flags;               // exchange-barrier epochs written by every rank
};

struct PdArgs {
  const PdRank* rk;  // device array [P]
  PdRank self;       // the executing rank's entry (real ranks): kernel-parameter operands
  int P, sh, me_real;
  int64_t n, m, wmax, inbox_cap, nnz;
  int32_t source;
  int direction, mu_edge;
  double do_a, do_b;
  gfx_iter_rec* recs;
  int64_t rec_cap;
  long long* summary;
  unsigned epoch_base;
};

struct PdCtl {
  long long nf, nf_loc, n_u, q_off, q_end, depth, reached, edges_total, switches, nrec;
  int mode_state, queue_form, mode, fsel, direct;
  double mf, mu;
  unsigned long long t0;
  unsigned epoch;
  PdRank R;  // this CTA's rank
};

__device__ __forceinline__ unsigned long long pd_gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void st_release_sys(unsigned* p, unsigned v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __noinline__ void pd_decide(long long n, long long m, long long nf, long long n_u,
                                       int mu_edge, int direction, int mode_state,
                                       long long depth, double do_a, double do_b, double* mf,
                                       double* mu, int* mode) {
  const DirEstimate est = estimate_mf_mu(n, m, nf, n_u, mu_edge);
  *mf = est.m_f;
  *mu = est.m_u;
  if (direction == GFX_DIR_AUTO)
    *mode = decide_direction(mode_state, est, do_a, do_b);
  else if (direction == GFX_DIR_PULL)
    *mode = depth > 1 ? GFX_DIR_PULL : GFX_DIR_PUSH;
  else
    *mode = GFX_DIR_PUSH;
}

// frontier membership against the rank's copy of the sliced frontier
struct SlicedFront {
  const uint32_t* g;
  int64_t wmax;
  int P, sh;
  __device__ __forceinline__ uint32_t word(int32_t s) const {
    if (sh >= 0) return g[(int64_t)(s & (P - 1)) * wmax + ((s >> sh) >> 5)];
    return g[(int64_t)(s % P) * wmax + ((s / P) >> 5)];
  }
  __device__ __forceinline__ bool bit(uint32_t w, int32_t s) const {
    return (w >> (((sh >= 0) ? (s >> sh) : (s / P)) & 31)) & 1u;
  }
};

// deferred labels of a rank: labels[l] = depth byte if visited, else
// UNVISITED; four vertices per thread (16-byte label stores when aligned)
__device__ __forceinline__ void pd_materialize(const PdRank& R, int64_t gtid, int64_t nthr) {
  const bool vec = ((reinterpret_cast<uintptr_t>(R.labels) | reinterpret_cast<uintptr_t>(R.lvl8)) &
                    15) == 0;
  for (int64_t v = gtid * 4; v < R.nl; v += nthr * 4) {
    const uint32_t bits = (R.visited[v >> 5] >> (v & 31)) & 0xFu;
    if (vec && v + 3 < R.nl) {
      const uint32_t d4 = *reinterpret_cast<const uint32_t*>(R.lvl8 + v);
      int4 lab;
      lab.x = (bits & 1u) ? (int32_t)(d4 & 0xFF) : GFX_UNVISITED;
      lab.y = (bits & 2u) ? (int32_t)((d4 >> 8) & 0xFF) : GFX_UNVISITED;
      lab.z = (bits & 4u) ? (int32_t)((d4 >> 16) & 0xFF) : GFX_UNVISITED;
      lab.w = (bits & 8u) ? (int32_t)(d4 >> 24) : GFX_UNVISITED;
      *reinterpret_cast<int4*>(R.labels + v) = lab;
    } else {
      for (int j = 0; j < 4 && v + j < R.nl; ++j)
        R.labels[v + j] = ((bits >> j) & 1u) ? (int32_t)R.lvl8[v + j] : GFX_UNVISITED;
    }
  }
}

// push claim: owned targets claimed in place (label, pred, next-frontier
// bit) and emitted; remote targets de-duplicated through `sent` and emitted
// with their source remembered (the owner split follows the expansion)
template <int B>
struct PdClaimOpT {
  static constexpr bool kWeights = false, kSrcVal = false, kEmitEdge = false;
  static constexpr int kBatch = B;
  static constexpr int kMinBlocks = 3;
  uint32_t* visited;
  uint32_t* sent;
  int32_t* sent_src;
  int32_t* labels;
  int32_t* preds;
  uint32_t* fnext;  // this rank's slice of the next frontier (local ids)
  int32_t depth;
  int P, r, sh;
  uint32_t wv[kBatch];
  uint8_t* lvl8 = nullptr;  // deferred labels (depth bytes)
  __device__ __forceinline__ int owner(int32_t d) const { return sh >= 0 ? (d & (P - 1)) : d % P; }
  __device__ __forceinline__ int32_t local(int32_t d) const { return sh >= 0 ? (d >> sh) : d / P; }
  __device__ int32_t src_value(int32_t) const { return 0; }
  __device__ void prefetch(const int32_t* d) {
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      if (d[u] < 0) wv[u] = 0xffffffffu;
      else if (owner(d[u]) == r) wv[u] = visited[local(d[u]) >> 5];
      else wv[u] = sent[d[u] >> 5];
    }
  }
  __device__ bool visit(int u, int32_t d, int32_t s, int32_t, int32_t, int64_t) {
    const int32_t sg = s * P + r;  // frontier items are local ids
    if (owner(d) == r) {
      const int32_t l = local(d);
      const uint32_t bit = 1u << (l & 31);
      if (wv[u] & bit) return false;
      if (atomicOr(&visited[l >> 5], bit) & bit) return false;
      if (lvl8) lvl8[l] = (uint8_t)depth;
      else labels[l] = depth;
      preds[l] = sg;
      atomicOr(&fnext[l >> 5], bit);
      return true;
    }
    const uint32_t bit = 1u << (d & 31);
    if (wv[u] & bit) return false;
    if (atomicOr(&sent[d >> 5], bit) & bit) return false;
    sent_src[d] = sg;
    return true;
  }
};

template <bool kVirt>
struct PdSync {
  cg::grid_group& grid;
  // every CTA of this rank (virtual mode: of every rank)
  __device__ __forceinline__ void rank() { grid.sync(); }
  // every CTA of every rank; peer stores before it are visible after it
  __device__ __forceinline__ void all(const PdArgs& a, PdCtl& c, int me) {
    if (kVirt || a.P == 1) {
      grid.sync();
      return;
    }
    __threadfence_system();
    grid.sync();
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      const unsigned e = ++c.epoch;
      for (int q = 0; q < a.P; ++q)
        if (q != me) st_release_sys(&a.rk[q].flags[me], e);
      for (int q = 0; q < a.P; ++q)
        if (q != me)
          while ((int)(ld_acquire_sys(&a.rk[me].flags[q]) - e) < 0) {
          }
    }
    if (threadIdx.x == 0 && blockIdx.x != 0) ++c.epoch;
    grid.sync();
  }
};

// kMulti: P > 1 (the exchange code compiled in); the P = 1 instance carries
// none of it (lower register pressure in its pull and expansion loops)
template <bool kVirt, bool kMulti>
__global__ void __launch_bounds__(256, 3) k_pdbfs(PdArgs a) {
  cg::grid_group grid = cg::this_grid();
  PdSync<kVirt> sync{grid};
  extern __shared__ __align__(16) unsigned char smem_raw[];
  WarpSmem& W = *reinterpret_cast<WarpSmem*>(smem_raw + (threadIdx.x >> 5) * kWarpScratch);
  PullSmem& PS = *reinterpret_cast<PullSmem*>(smem_raw + (threadIdx.x >> 5) * kWarpScratch);
  __shared__ ScanSmem ss;
  __shared__ PdCtl c;
  __shared__ CtaAgg agg;
  const int P = kMulti ? a.P : 1;
  const int me = kVirt ? (int)(blockIdx.x % P) : a.me_real;
  const int64_t rcta = kVirt ? blockIdx.x / P : blockIdx.x;
  const int64_t nrcta = kVirt ? gridDim.x / P : gridDim.x;
  const int64_t gtid = rcta * blockDim.x + threadIdx.x;
  const int64_t nthr = nrcta * blockDim.x;
  const int64_t gw = gtid >> 5, nw = nthr >> 5;
  const bool rlead = rcta == 0 && threadIdx.x == 0;  // one thread per rank
  const bool leader = blockIdx.x == 0 && threadIdx.x == 0;
  if (threadIdx.x == 0) {
    c.R = a.rk[me];
    c.epoch = a.epoch_base;
  }
  if (threadIdx.x < 8) agg.ctr[threadIdx.x] = 0ull;
  __syncthreads();
  // virtual ranks: the CTA's rank entry in shared memory; a real rank reads
  // its own entry from the kernel parameters (constant-bank operands, no
  // registers held)
  const PdRank& R = kVirt ? c.R : a.self;
  const int32_t src_owner = a.sh >= 0 ? (a.source & (P - 1)) : a.source % P;
  const int32_t src_local = a.sh >= 0 ? (a.source >> a.sh) : a.source / P;
  const int64_t wl = R.wl, wmax = a.wmax;

  // ---- init (rank-local state; the exchange block: own copy only)
  for (int64_t l = gtid; l < R.nl; l += nthr) R.preds[l] = -1;  // labels: deferred
  for (int64_t w = gtid; w < wl; w += nthr) R.visited[w] = 0u;
  for (int64_t w = gtid; w < (a.n + 31) / 32; w += nthr) R.sent[w] = 0u;
  for (int64_t w = gtid; w < 3 * P * wmax; w += nthr) {
    const int64_t k = w / (P * wmax), o = w % (P * wmax);
    R.gfront[k][o] = 0u;
  }
  for (int64_t i = gtid; i < 3 * (int64_t)(sizeof(Counters) / 8); i += nthr)
    reinterpret_cast<unsigned long long*>(R.C)[i] = 0ull;
  for (int64_t i = gtid; i < P; i += nthr) {
    R.outcnt[i] = 0ull;
    R.inbox_cnt[i] = 0ull;
  }
  sync.all(a, c, me);  // nobody writes into a peer before every rank initialised
  if (rlead) {
    // every rank's copy of the first frontier holds the source (a pull at
    // the source's level probes it); its owner also queues it
    R.gfront[0][(int64_t)src_owner * wmax + (src_local >> 5)] = 1u << (src_local & 31);
    if (me == src_owner) {
      R.lvl8[src_local] = 0;
      R.visited[src_local >> 5] = 1u << (src_local & 31);
      R.order[0] = src_local;
    }
  }
  if (threadIdx.x == 0) {
    c.nf = 1;
    c.nf_loc = me == src_owner ? 1 : 0;
    c.n_u = a.n;
    c.q_off = 0;
    c.q_end = c.nf_loc;
    c.depth = c.reached = c.edges_total = c.switches = c.nrec = 0;
    c.mode_state = GFX_DIR_PUSH;
    c.queue_form = 1;
    c.fsel = 0;
    c.direct = 0;
  }
  sync.rank();

  for (;;) {
    if (threadIdx.x == 0) {
      c.depth += 1;
      c.n_u -= c.nf;
      int mode;
      double mf, mu;
      pd_decide(a.n, a.m, c.nf, c.n_u, a.mu_edge, a.direction, c.mode_state, c.depth, a.do_a,
                a.do_b, &mf, &mu, &mode);
      c.mf = mf;
      c.mu = mu;
      c.mode = mode;
      if (mode != c.mode_state) c.switches += 1;
      c.t0 = pd_gtime();
    }
    __syncthreads();
    if (!c.direct && c.depth == 255) {
      // depth bytes exhausted: labels so far written, labelled directly from here
      pd_materialize(R, gtid, nthr);
      sync.rank();
      if (threadIdx.x == 0) c.direct = 1;
      __syncthreads();
    }
    uint8_t* const lvl8 = c.direct ? nullptr : R.lvl8;
    const int32_t depth = (int32_t)c.depth;
    const int par = (int)(c.depth & 1);
    Counters* cur = &R.C[c.depth % 3];
    if (rcta == 0 && threadIdx.x < (int)(sizeof(Counters) / 8))
      reinterpret_cast<unsigned long long*>(&R.C[(c.depth + 1) % 3])[threadIdx.x] = 0ull;
    const uint32_t* fcur = R.gfront[c.fsel];
    uint32_t* fnext_me = R.gfront[(c.fsel + 1) % 3] + me * wmax;
    {
      // this rank's slice of the buffer the level after next writes: last
      // read one level ago (peers' slices are overwritten whole by them)
      uint32_t* fclr = R.gfront[(c.fsel + 2) % 3] + me * wmax;
      for (int64_t i = gtid; i < wl; i += nthr) fclr[i] = 0u;
    }
    long long nout_loc = 0, slots_loc = 0, probes_loc = 0, cands_loc = 0;

    if (c.mode == GFX_DIR_PUSH) {
      if (!c.queue_form) {
        // the frontier is this rank's slice of the current bitmap: queue it
        const uint32_t* myslice = fcur + me * wmax;
        const int lane = threadIdx.x & 31;
        for (int64_t grp = gw; grp * 32 < wl; grp += nw) {
          const int64_t w = grp * 32 + lane;
          uint32_t x = w < wl ? myslice[w] : 0u;
          int tot;
          const int off = warp_excl_scan(__popc(x), lane, &tot);
          if (tot == 0) continue;
          unsigned long long b = 0;
          if (lane == 0) b = atomicAdd(&cur->aux0, (unsigned long long)tot);
          b = __shfl_sync(0xffffffffu, b, 0) + off;
          while (x) {
            const int k = __ffs(x) - 1;
            x &= x - 1;
            R.order[c.q_end + b++] = (int32_t)(w * 32 + k);
          }
        }
        sync.rank();
        if (threadIdx.x == 0) {
          c.q_off = c.q_end;
          c.q_end += c.nf_loc;
          c.queue_form = 1;
        }
        __syncthreads();
      }
      const int32_t* F = R.order + c.q_off;
      const int64_t nf = c.nf_loc;
      PdClaimOpT<kVisitBatch> op{R.visited, R.sent, R.sent_src, R.labels, R.preds, fnext_me,
                                 depth, P, me, a.sh, {}, lvl8};
      // P = 1: the owned winners go straight into the queue (global = local)
      int32_t* out = P == 1 ? R.order + c.q_end : R.emit;
      // expansion by frontier size, as the single-GPU loop: <= 32 items with
      // no plan pass, <= 64K items 32 per warp (hubs after one barrier),
      // else the fused degree scan + load-balanced tiles.  Chosen on the
      // GLOBAL frontier size: every rank takes the same path, so the barrier
      // sequence is identical on every rank (virtual ranks share one grid)
      if (c.nf <= 32) {
        PdClaimOpT<4> top{R.visited, R.sent, R.sent_src, R.labels, R.preds, fnext_me, depth, P, me,
                          a.sh, {}, lvl8};
        push_tiny(W, top, F, nf, R.row, R.col, out, &cur->out_len, &cur->total, gw, nw, agg);
      } else if (c.nf <= kMidItems) {
        push_mid(W, op, F, nf, R.row, R.col, out, &cur->out_len, R.part, &cur->aux3, gw, nw, agg);
        cta_flush_ctrs(agg, cur);
        sync.rank();
        cta_read_ctrs(agg, cur);
        const int64_t nh = (int64_t)agg.rd[7];
        for (int64_t h0 = 0; h0 < nh; h0 += 32) {  // heavy items, 32 at a time
          const int lane = threadIdx.x & 31;
          int32_t v = 0;
          int64_t rb = 0, deg = 0;
          if (h0 + lane < nh) {
            v = F[R.part[h0 + lane]];
            rb = R.row[v];
            deg = R.row[v + 1] - rb;
          }
          int ocnt = 0;
          const int64_t t = expand_items32(W, op, v, rb, deg, R.col, out, &cur->out_len, ocnt,
                                           gw * 32 * kVisitBatch, nw * 32 * kVisitBatch);
          warp_flush(W, ocnt, out, &cur->out_len);
          if (gtid == 0) atomicAdd(&cur->total, (unsigned long long)t);
        }
      } else {
        const int64_t stiles = (nf + kScanTileItems - 1) / kScanTileItems;
        const unsigned ep = a.epoch_base + (unsigned)c.depth;
        for (int64_t t = rcta; t < stiles; t += nrcta)
          scan_tile(t, stiles, F, nf, R.row, R.scan, R.rowbase, R.part, R.status, ep, cur, ss);
        sync.rank();
        cta_read_ctrs(agg, cur);
        expand_tasks(W, op, F, nf, R.scan, R.rowbase, R.part, (int64_t)agg.rd[3],
                     (int64_t)agg.rd[2], R.col, nullptr, out, &cur->out_len, gw, nw, &agg);
        for (int64_t i = gtid; i < stiles; i += nthr) R.status[i] = 0ull;
      }
      sync.rank();
      cta_read_ctrs(agg, cur);
      slots_loc = (long long)agg.rd[2];
      if constexpr (!kMulti) {
        nout_loc = (long long)agg.rd[0];
      } else {
        // owner split: owned winners -> queue (local ids), remote
        // candidates -> the owner's inbox region for this rank (peer
        // stores), `sent` bits cleared for the next level
        const int64_t nemit = (long long)agg.rd[0];
        const int lane = threadIdx.x & 31;
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
            at = atomicAdd(o == me ? &cur->aux2 : &R.outcnt[o], (unsigned long long)__popc(peers));
          at = __shfl_sync(0xffffffffu, at, lead) + rank_in;
          if (ok) {
            if (o == me) {
              R.order[c.q_end + at] = op.local(d);
            } else {
              a.rk[o].inbox[(int64_t)me * a.inbox_cap + at] =
                  ((unsigned long long)(uint32_t)d << 32) | (uint32_t)R.sent_src[d];
              atomicAnd(&R.sent[d >> 5], ~(1u << (d & 31)));
            }
          }
        }
        sync.rank();
        if (rlead)
          for (int o = 0; o < P; ++o)
            if (o != me) {
              a.rk[o].inbox_cnt[me] = R.outcnt[o];
              R.outcnt[o] = 0ull;
            }
        sync.all(a, c, me);  // every inbox complete
        // claim what the other ranks sent
        for (int q = 0; q < P; ++q) {
          if (q == me) continue;
          const int64_t cnt = (int64_t)R.inbox_cnt[q];
          const unsigned long long* box = R.inbox + (int64_t)q * a.inbox_cap;
          for (int64_t base = gtid & ~31ll; base < cnt; base += nthr) {
            const int64_t i = base + lane;
            bool won = false;
            int32_t l = 0;
            if (i < cnt) {
              const unsigned long long x = box[i];
              const int32_t d = (int32_t)(x >> 32), s = (int32_t)(uint32_t)x;
              l = op.local(d);
              const uint32_t bit = 1u << (l & 31);
              if (!(atomicOr(&R.visited[l >> 5], bit) & bit)) {
                won = true;
                if (lvl8) lvl8[l] = (uint8_t)depth;
                else R.labels[l] = depth;
                R.preds[l] = s;
                atomicOr(&fnext_me[l >> 5], bit);
              }
            }
            const unsigned wm = __ballot_sync(0xffffffffu, won);
            unsigned long long b = 0;
            if (lane == 0 && wm) b = atomicAdd(&cur->aux2, (unsigned long long)__popc(wm));
            b = __shfl_sync(0xffffffffu, b, 0);
            if (won) R.order[c.q_end + b + __popc(wm & ((1u << lane) - 1))] = l;
          }
        }
        sync.rank();
        cta_read_ctrs(agg, cur);
        nout_loc = (long long)agg.rd[6];
      }
      if (threadIdx.x == 0) {
        c.q_off = c.q_end;
        c.q_end += nout_loc;
        c.queue_form = 1;
      }
    } else {
      // pull over this rank's unvisited rows against the sliced frontier
      const long long ncand = c.n_u - (a.n - a.nnz);
      const bool qsmall = ncand <= (a.n >> 6);
      Counters* actr = reinterpret_cast<Counters*>(agg.ctr);
      const SlicedFront front{fcur, wmax, P, a.sh};
      if (ncand * 8 > a.n)
        pull_groups<SlicedFront, 8>(wl, R.nz, R.visited, front, fnext_me, R.head, R.row, R.col, 0,
                                    LabelOut{R.labels, lvl8}, R.preds, depth, actr, gw, nw, PS,
                                    R.head2, &cur->aux2);
      else
        pull_groups<SlicedFront, 4>(wl, R.nz, R.visited, front, fnext_me, R.head, R.row, R.col, 0,
                                    LabelOut{R.labels, lvl8}, R.preds, depth, actr, gw, nw, PS,
                                    R.head2, nullptr, qsmall ? R.order + c.q_end : nullptr,
                                    &cur->aux3);
      cta_flush_ctrs(agg, cur);
      sync.rank();
      cta_read_ctrs(agg, cur);
      nout_loc = (long long)agg.rd[0];
      probes_loc = (long long)agg.rd[4];
      cands_loc = (long long)agg.rd[5];
      if (threadIdx.x == 0) {
        c.queue_form = qsmall ? 1 : 0;
        if (qsmall) {
          c.q_off = c.q_end;
          c.q_end += nout_loc;
        }
      }
    }
    // ---- end of level: the rank's next-frontier slice and level counters
    // to every rank, then the global sums
    long long g_nout = nout_loc, g_slots = slots_loc, g_probes = probes_loc, g_cands = cands_loc;
    if constexpr (kMulti) {
      for (int q = 0; q < P; ++q) {
        if (q == me) continue;
        uint32_t* dst = a.rk[q].gfront[(c.fsel + 1) % 3] + me * wmax;
        for (int64_t i = gtid; i < wl; i += nthr) dst[i] = fnext_me[i];
      }
      if (rlead)
        for (int q = 0; q < P; ++q) {
          long long* row = a.rk[q].ctab + ((int64_t)par * kPdMaxRanks + me) * 4;
          row[0] = nout_loc;
          row[1] = slots_loc;
          row[2] = probes_loc;
          row[3] = cands_loc;
        }
      sync.all(a, c, me);
      g_nout = g_slots = g_probes = g_cands = 0;
      for (int q = 0; q < P; ++q) {
        const long long* row = R.ctab + ((int64_t)par * kPdMaxRanks + q) * 4;
        g_nout += ld_volatile_u64(reinterpret_cast<const unsigned long long*>(row));
        g_slots += ld_volatile_u64(reinterpret_cast<const unsigned long long*>(row + 1));
        g_probes += ld_volatile_u64(reinterpret_cast<const unsigned long long*>(row + 2));
        g_cands += ld_volatile_u64(reinterpret_cast<const unsigned long long*>(row + 3));
      }
    }
    const bool push = c.mode == GFX_DIR_PUSH;
    if (leader && c.nrec < a.rec_cap) {
      gfx_iter_rec rec{};
      rec.iteration = c.depth;
      rec.frontier_in = c.nf;
      rec.frontier_out = g_nout;
      rec.n_u = c.n_u;
      rec.edges = push ? g_slots : -1;
      rec.m_f = c.mf;
      rec.m_u = c.mu;
      rec.mode_before = c.mode_state;
      rec.decision = c.mode;
      rec.ms = (float)((pd_gtime() - c.t0) * 1e-6);
      rec.candidates = push ? 0 : g_cands;
      rec.work = push ? g_slots : g_probes;
      rec.bytes_alg = push ? 20 * c.nf + 4 * g_slots + 8 * g_nout
                           : 12 * g_cands + 4 * g_probes + 8 * g_nout;
      a.recs[c.nrec] = rec;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      c.nrec += 1;
      c.reached += c.nf;
      if (push) c.edges_total += g_slots;
      c.mode_state = c.mode;
      c.nf = g_nout;
      c.nf_loc = nout_loc;
      c.fsel = (c.fsel + 1) % 3;
    }
    __syncthreads();
    if (c.nf == 0) break;
  }
  if (!c.direct) pd_materialize(R, gtid, nthr);
  if (leader) {
    a.summary[0] = c.depth;
    a.summary[1] = c.edges_total;
    a.summary[2] = c.switches;
    a.summary[3] = c.reached;
    a.summary[4] = c.nrec < a.rec_cap ? c.nrec : a.rec_cap;
  }
  if (rlead && !kVirt) a.summary[5] = c.epoch;  // the exchange-barrier epoch reached
}

// first / second neighbour per local row, bit 31 = "degree is exactly 1 / 2"
__global__ void k_pd_heads(const int64_t* __restrict__ row, const int32_t* __restrict__ col,
                           int64_t n, int32_t* __restrict__ head, int32_t* __restrict__ head2) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = row[v], d = row[v + 1] - b;
    head[v] = d > 0 ? (int32_t)((uint32_t)col[b] | (d == 1 ? 0x80000000u : 0u)) : -1;
    head2[v] = d > 1 ? (int32_t)((uint32_t)col[b + 1] | (d == 2 ? 0x80000000u : 0u)) : -1;
  }
}

}  // namespace gfx

using namespace gfx;

// one rank's device allocations (rank-local part + exchange block)
struct PdOwned {
  gfx_graph* lg = nullptr;
  std::vector<void*> bufs;
};

struct gfx_pdbfs {
  gfx_ctx* ctx = nullptr;
  int P = 1, me = 0, virt = 1;
  int64_t n = 0, m = 0, wmax = 0, inbox_cap = 0, nnz = 0;
  std::vector<PdOwned> own;    // virtual: P entries; real: 1 (this rank)
  std::vector<PdRank> rk;      // host mirror of the device rank table
  PdRank* rk_d = nullptr;
  gfx_iter_rec* recs_d = nullptr;
  long long* summary_d = nullptr;
  int64_t rec_cap = 4096;
  unsigned epoch = 0;
  int grid = 0, smem = 0;
  std::vector<void*> ipc_opened;  // peer mappings (real mode)
};

namespace {

int pd_alloc(PdOwned& o, size_t bytes, void** out) {
  void* p = nullptr;
  GFX_CK(cudaMalloc(&p, bytes ? bytes : 16));
  o.bufs.push_back(p);
  *out = p;
  return GFX_OK;
}
template <class T>
int pd_alloc_t(PdOwned& o, size_t count, T** out) {
  void* p = nullptr;
  GFX_TRY(pd_alloc(o, count * sizeof(T), &p));
  *out = static_cast<T*>(p);
  return GFX_OK;
}

// rank-local buffers + the exchange block for local rank data (row, col)
int pd_setup_rank(gfx_pdbfs* e, const int64_t* lrow, const int32_t* lcol, int64_t nl,
                  int64_t ml, PdOwned& o, PdRank& R) {
  gfx_ctx* ctx = e->ctx;
  GFX_TRY(gfx_graph_create(ctx, nl, ml, lrow, lcol, nullptr, GFX_GRAPH_UNDIRECTED, &o.lg));
  gfx_graph* g = o.lg;
  std::memset(&R, 0, sizeof(R));
  R.row = lrow;
  R.col = lcol;
  R.nl = nl;
  R.wl = (nl + 31) / 32;
  R.nnz = g->nnz_vertices;
  void* nz = nullptr;
  GFX_TRY(scratch(g, "nz_out", R.wl * 4, &nz));
  R.nz = static_cast<const uint32_t*>(nz);
  int32_t* heads;
  GFX_TRY(pd_alloc_t(o, 2 * (size_t)(nl + 1), &heads));
  if (nl > 0)
    GFX_LAUNCH(k_pd_heads, grid_for(nl, 256, ctx->sm_count * 8), 256, 0, ctx->stream, lrow, lcol,
               nl, heads, heads + nl + 1);
  R.head = heads;
  R.head2 = heads + nl + 1;
  GFX_TRY(pd_alloc_t(o, R.wl + 1, &R.visited));
  GFX_TRY(pd_alloc_t(o, nl + 1, &R.labels));
  GFX_TRY(pd_alloc_t(o, (size_t)nl + 16, &R.lvl8));
  GFX_TRY(pd_alloc_t(o, nl + 1, &R.preds));
  GFX_TRY(pd_alloc_t(o, nl + 2, &R.order));
  GFX_TRY(pd_alloc_t(o, (size_t)e->n + 1, &R.emit));
  GFX_TRY(pd_alloc_t(o, nl + 2, &R.scan));
  GFX_TRY(pd_alloc_t(o, nl + 1, &R.rowbase));
  GFX_TRY(pd_alloc_t(o, part_capacity(ml, nl), &R.part));
  const int64_t stiles = std::max<int64_t>(1, (nl + kScanTileItems - 1) / kScanTileItems);
  GFX_TRY(pd_alloc_t(o, stiles + 1, &R.status));
  GFX_CK(cudaMemsetAsync(R.status, 0, (stiles + 1) * 8, ctx->stream));
  GFX_TRY(pd_alloc_t(o, (size_t)(e->n + 31) / 32 + 1, &R.sent));
  GFX_TRY(pd_alloc_t(o, (size_t)e->n + 1, &R.sent_src));
  GFX_TRY(pd_alloc_t(o, 3 * sizeof(Counters) / 8, reinterpret_cast<unsigned long long**>(&R.C)));
  GFX_TRY(pd_alloc_t(o, kPdMaxRanks, &R.outcnt));
  // exchange block
  uint32_t* gf;
  GFX_TRY(pd_alloc_t(o, 3 * (size_t)e->P * e->wmax, &gf));
  for (int k = 0; k < 3; ++k) R.gfront[k] = gf + (size_t)k * e->P * e->wmax;
  GFX_TRY(pd_alloc_t(o, (size_t)e->P * e->inbox_cap + 1, &R.inbox));
  GFX_TRY(pd_alloc_t(o, kPdMaxRanks, &R.inbox_cnt));
  GFX_TRY(pd_alloc_t(o, 2 * kPdMaxRanks * 4, &R.ctab));
  GFX_TRY(pd_alloc_t(o, kPdMaxRanks, &R.flags));
  GFX_CK(cudaMemsetAsync(R.flags, 0, kPdMaxRanks * 4, ctx->stream));
  GFX_CK(cudaMemsetAsync(R.ctab, 0, 2 * kPdMaxRanks * 4 * 8, ctx->stream));
  return GFX_OK;
}

const void* pd_kernel(const gfx_pdbfs* e) {
  if (e->P == 1) return (const void*)k_pdbfs<false, false>;
  return e->virt ? (const void*)k_pdbfs<true, true> : (const void*)k_pdbfs<false, true>;
}

int pd_grid(gfx_pdbfs* e) {
  const int smem = kWarpScratch * kWarpsPerBlock;
  int per_sm = 0;
  const void* fn = pd_kernel(e);
  GFX_CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  GFX_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, smem));
  GFX_REQUIRE(per_sm >= 1, "k_pdbfs cannot be resident");
  int grid = per_sm * e->ctx->sm_count;
  if (e->virt) grid = grid / e->P * e->P;  // whole CTAs per virtual rank
  e->grid = grid;
  e->smem = smem;
  return GFX_OK;
}

int pd_finish_create(gfx_pdbfs* e) {
  GFX_CK(cudaMalloc(&e->rk_d, sizeof(PdRank) * e->P));
  GFX_CK(cudaMalloc(&e->recs_d, sizeof(gfx_iter_rec) * e->rec_cap));
  GFX_CK(cudaMalloc(&e->summary_d, sizeof(long long) * 8));
  GFX_TRY(pd_grid(e));
  return GFX_OK;
}

int pd_upload_table(gfx_pdbfs* e) {
  GFX_CK(cudaMemcpyAsync(e->rk_d, e->rk.data(), sizeof(PdRank) * e->P, cudaMemcpyHostToDevice,
                         e->ctx->stream));
  return GFX_OK;
}

int pd_launch(gfx_pdbfs* e, int64_t source, int direction, double do_a, double do_b,
              int mu_edge) {
  PdArgs a{};
  a.rk = e->rk_d;
  a.P = e->P;
  a.sh = -1;
  if ((e->P & (e->P - 1)) == 0) {
    a.sh = 0;
    while ((1 << a.sh) < e->P) ++a.sh;
  }
  a.me_real = e->me;
  a.self = e->rk[e->virt ? 0 : e->me];
  a.n = e->n;
  a.m = e->m;
  a.wmax = e->wmax;
  a.inbox_cap = e->inbox_cap;
  a.nnz = e->nnz;
  a.source = (int32_t)source;
  a.direction = direction;
  a.mu_edge = mu_edge;
  a.do_a = do_a;
  a.do_b = do_b;
  a.recs = e->recs_d;
  a.rec_cap = e->rec_cap;
  a.summary = e->summary_d;
  // scan epochs and exchange-barrier epochs advance monotonically across runs
  a.epoch_base = e->epoch;
  e->epoch += 4096;
  void* kargs[] = {&a};
  GFX_CK(cudaLaunchCooperativeKernel(pd_kernel(e), dim3(e->grid), dim3(256), kargs, e->smem,
                                     e->ctx->stream));
  count_launch();
  return GFX_OK;
}

}  // namespace

extern "C" {

int gfx_pdbfs_create_virtual(gfx_ctx* ctx, int64_t n, int64_t m, int P,
                             const int64_t* const* lrow, const int32_t* const* lcol,
                             const int64_t* n_local, const int64_t* m_local, gfx_pdbfs** out) {
  GFX_NVTX("gfx_pdbfs_create_virtual");
  GFX_REQUIRE(ctx && lrow && lcol && n_local && m_local && out, "gfx_pdbfs_create_virtual: null argument");
  GFX_REQUIRE(P >= 1 && P <= kPdMaxRanks, "P=%d out of range 1..%d", P, kPdMaxRanks);
  GFX_REQUIRE(n > 0 && n < (int64_t)INT32_MAX, "n=%lld out of range", (long long)n);
  for (int q = 0; q < P; ++q)
    GFX_REQUIRE(n_local[q] == (n > q ? (n - q + P - 1) / P : 0),
                "n_local[%d] does not match the partition", q);
  GFX_CK(cudaSetDevice(ctx->device));
  auto* e = new gfx_pdbfs();
  e->ctx = ctx;
  e->P = P;
  e->virt = 1;
  e->n = n;
  e->m = m;
  const int64_t nmax = (n + P - 1) / P;
  e->wmax = (nmax + 31) / 32;
  e->inbox_cap = nmax + 1;
  e->own.resize(P);
  e->rk.resize(P);
  for (int q = 0; q < P; ++q) {
    const int st = pd_setup_rank(e, lrow[q], lcol[q], n_local[q], m_local[q], e->own[q], e->rk[q]);
    if (st != GFX_OK) {
      gfx_pdbfs_destroy(e);
      return st;
    }
    e->nnz += e->rk[q].nnz;
  }
  int st = pd_finish_create(e);
  if (st == GFX_OK) st = pd_upload_table(e);
  if (st != GFX_OK) {
    gfx_pdbfs_destroy(e);
    return st;
  }
  GFX_CK(cudaStreamSynchronize(ctx->stream));
  *out = e;
  return GFX_OK;
}

// Real ranks (one process per GPU).  Rank r allocates its own buffers; its
// exchange block (frontier copies, inbox, inbox counts, counter table,
// barrier flags) is exported as CUDA-IPC handles, all-gathered by the caller
// (torch.distributed) and imported by every peer, after which peers store
// into it directly over NVLink.
constexpr int kPdHandles = 5;

int gfx_pdbfs_create_rank(gfx_ctx* ctx, int64_t n, int64_t m, int P, int r, const int64_t* lrow,
                          const int32_t* lcol, int64_t n_local, int64_t m_local,
                          gfx_pdbfs** out) {
  GFX_NVTX("gfx_pdbfs_create_rank");
  GFX_REQUIRE(ctx && lrow && out, "gfx_pdbfs_create_rank: null argument");
  GFX_REQUIRE(P >= 1 && P <= kPdMaxRanks && r >= 0 && r < P, "bad partition P=%d r=%d", P, r);
  GFX_REQUIRE(n > 0 && n < (int64_t)INT32_MAX, "n=%lld out of range", (long long)n);
  GFX_REQUIRE(n_local == (n > r ? (n - r + P - 1) / P : 0), "n_local does not match the partition");
  GFX_CK(cudaSetDevice(ctx->device));
  auto* e = new gfx_pdbfs();
  e->ctx = ctx;
  e->P = P;
  e->me = r;
  e->virt = 0;
  e->n = n;
  e->m = m;
  const int64_t nmax = (n + P - 1) / P;
  e->wmax = (nmax + 31) / 32;
  e->inbox_cap = nmax + 1;
  e->own.resize(1);
  e->rk.assign(P, PdRank{});
  int st = pd_setup_rank(e, lrow, lcol, n_local, m_local, e->own[0], e->rk[r]);
  if (st == GFX_OK) {
    e->nnz = e->rk[r].nnz;  // the global count arrives with gfx_pdbfs_import
    st = pd_finish_create(e);
  }
  if (st == GFX_OK) st = pd_upload_table(e);
  if (st != GFX_OK) {
    gfx_pdbfs_destroy(e);
    return st;
  }
  GFX_CK(cudaStreamSynchronize(ctx->stream));
  *out = e;
  return GFX_OK;
}

// vertices of this rank with degree > 0 (the caller sums them over ranks)
int gfx_pdbfs_local_nnz(gfx_pdbfs* e, int64_t* nnz) {
  GFX_REQUIRE(e && nnz, "gfx_pdbfs_local_nnz: null argument");
  *nnz = e->rk[e->virt ? 0 : e->me].nnz;
  return GFX_OK;
}

// kPdHandles cudaIpcMemHandle_t (64 bytes each) of this rank's exchange block
int gfx_pdbfs_export(gfx_pdbfs* e, void* handles) {
  GFX_REQUIRE(e && handles && !e->virt, "gfx_pdbfs_export: real-rank engine required");
  const PdRank& R = e->rk[e->me];
  void* bases[kPdHandles] = {R.gfront[0], R.inbox, R.inbox_cnt, R.ctab, R.flags};
  auto* h = static_cast<cudaIpcMemHandle_t*>(handles);
  for (int k = 0; k < kPdHandles; ++k) GFX_CK(cudaIpcGetMemHandle(&h[k], bases[k]));
  return GFX_OK;
}

// all ranks' handles (P x kPdHandles, rank-major): map every peer's
// exchange block and publish the rank table to the device
int gfx_pdbfs_import(gfx_pdbfs* e, const void* all_handles, int64_t nnz_global) {
  GFX_REQUIRE(e && all_handles && !e->virt, "gfx_pdbfs_import: real-rank engine required");
  GFX_REQUIRE(nnz_global >= e->rk[e->me].nnz && nnz_global <= e->n, "bad nnz_global %lld",
              (long long)nnz_global);
  e->nnz = nnz_global;
  GFX_CK(cudaSetDevice(e->ctx->device));
  const auto* h = static_cast<const cudaIpcMemHandle_t*>(all_handles);
  for (int q = 0; q < e->P; ++q) {
    if (q == e->me) continue;
    void* p[kPdHandles];
    for (int k = 0; k < kPdHandles; ++k) {
      GFX_CK(cudaIpcOpenMemHandle(&p[k], h[q * kPdHandles + k], cudaIpcMemLazyEnablePeerAccess));
      e->ipc_opened.push_back(p[k]);
    }
    PdRank& Q = e->rk[q];
    std::memset(&Q, 0, sizeof(Q));
    auto* gf = static_cast<uint32_t*>(p[0]);
    for (int k = 0; k < 3; ++k) Q.gfront[k] = gf + (size_t)k * e->P * e->wmax;
    Q.inbox = static_cast<unsigned long long*>(p[1]);
    Q.inbox_cnt = static_cast<unsigned long long*>(p[2]);
    Q.ctab = static_cast<long long*>(p[3]);
    Q.flags = static_cast<unsigned*>(p[4]);
  }
  GFX_TRY(pd_upload_table(e));
  GFX_CK(cudaStreamSynchronize(e->ctx->stream));
  return GFX_OK;
}

int gfx_pdbfs_destroy(gfx_pdbfs* e) {
  if (!e) return GFX_OK;
  cudaSetDevice(e->ctx->device);
  cudaStreamSynchronize(e->ctx->stream);
  for (void* p : e->ipc_opened) cudaIpcCloseMemHandle(p);
  for (auto& o : e->own) {
    for (void* p : o.bufs) cudaFree(p);
    if (o.lg) gfx_graph_destroy(o.lg);
  }
  cudaFree(e->rk_d);
  cudaFree(e->recs_d);
  cudaFree(e->summary_d);
  delete e;
  return GFX_OK;
}

// One BFS; labels / preds of rank q (local ids; preds are global ids) are
// copied to labels_d[q] / preds_d[q] when given (virtual mode: every rank's,
// real mode: q = this rank only).
int gfx_pdbfs_run(gfx_pdbfs* e, int64_t source, int direction, double do_a, double do_b,
                  int mu_edge_based, int32_t* const* labels_d, int32_t* const* preds_d,
                  gfx_iter_rec* recs, int64_t rec_cap, gfx_stats* st) {
  GFX_NVTX("gfx_pdbfs_run");
  GFX_REQUIRE(e, "gfx_pdbfs_run: null engine");
  GFX_REQUIRE(source >= 0 && source < e->n, "source %lld out of range", (long long)source);
  GFX_REQUIRE(direction == GFX_DIR_PUSH || direction == GFX_DIR_PULL || direction == GFX_DIR_AUTO,
              "unknown direction %d", direction);
  if (direction == GFX_DIR_AUTO) GFX_REQUIRE(do_a > 0 && do_b > 0, "do_a and do_b must be positive");
  gfx_ctx* ctx = e->ctx;
  GFX_CK(cudaSetDevice(ctx->device));
  GFX_CK(cudaEventRecord(ctx->ev0, ctx->stream));
  GFX_TRY(pd_launch(e, source, direction, do_a, do_b, mu_edge_based));
  GFX_CK(cudaEventRecord(ctx->ev1, ctx->stream));
  long long summary[8];
  GFX_CK(cudaMemcpyAsync(summary, e->summary_d, sizeof(summary), cudaMemcpyDeviceToHost,
                         ctx->stream));
  const int nr = e->virt ? e->P : 1;
  for (int k = 0; k < nr; ++k) {
    const int q = e->virt ? k : e->me;
    if (labels_d && labels_d[k])
      GFX_CK(cudaMemcpyAsync(labels_d[k], e->rk[q].labels, e->rk[q].nl * 4,
                             cudaMemcpyDeviceToDevice, ctx->stream));
    if (preds_d && preds_d[k])
      GFX_CK(cudaMemcpyAsync(preds_d[k], e->rk[q].preds, e->rk[q].nl * 4,
                             cudaMemcpyDeviceToDevice, ctx->stream));
  }
  GFX_CK(cudaStreamSynchronize(ctx->stream));
  float ms = 0.f;
  GFX_CK(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
  const int64_t nrec = std::min<int64_t>(summary[4], recs ? rec_cap : 0);
  if (nrec > 0)
    GFX_CK(cudaMemcpy(recs, e->recs_d, nrec * sizeof(gfx_iter_rec), cudaMemcpyDeviceToHost));
  if (st) {
    std::memset(st, 0, sizeof(*st));
    st->iterations = summary[0];
    st->edges_traversed = summary[1];
    st->direction_switches = summary[2];
    st->reached = summary[3];
    st->edges_reached = -1;
    st->device_ms = ms;
    st->num_records = nrec;
  }
  return GFX_OK;
}

// count BFS runs back to back (one cooperative launch each): device ms
int gfx_pdbfs_batch(gfx_pdbfs* e, int64_t source, int64_t count, int direction, double do_a,
                    double do_b, int mu_edge_based, float* ms) {
  GFX_NVTX("gfx_pdbfs_batch");
  GFX_REQUIRE(e && ms && count > 0, "gfx_pdbfs_batch: bad argument");
  GFX_REQUIRE(source >= 0 && source < e->n, "source %lld out of range", (long long)source);
  gfx_ctx* ctx = e->ctx;
  GFX_CK(cudaSetDevice(ctx->device));
  GFX_CK(cudaEventRecord(ctx->ev0, ctx->stream));
  for (int64_t k = 0; k < count; ++k) GFX_TRY(pd_launch(e, source, direction, do_a, do_b, mu_edge_based));
  GFX_CK(cudaEventRecord(ctx->ev1, ctx->stream));
  GFX_CK(cudaEventSynchronize(ctx->ev1));
  GFX_CK(cudaEventElapsedTime(ms, ctx->ev0, ctx->ev1));
  return GFX_OK;
}

}  // extern "C"
