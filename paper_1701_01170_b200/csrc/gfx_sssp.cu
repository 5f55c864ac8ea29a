// Single-source shortest paths with near/far bucketing on sm_100a.
//
// Reference: primitives/sssp.py:41-121 (loop, relax = atomic_min,
// set_pred + stamp, exact filter on the stamp) and near_far.py:20-85
// (two-slice pile: near = key < threshold, far keeps its enqueue key; when
// near drains, threshold += delta, stale far entries -- live key != enqueue
// key -- are dropped and the rest re-split).
//
// Device state:
//   dp     uint64[n]  (dist << 32 | pred): one 64-bit atomicMin settles the
//                     distance and a valid predecessor together, so preds are
//                     always consistent with the final distances
//   dist   uint32[n]  32-bit mirror of dp's distance: the probe array (L2-resident)
//   mark   uint32[n/32] enqueued-this-iteration bits (the reference's stamp,
//                     sssp.py:112-115): each improved vertex is enqueued once
//                     per iteration; the split kernel clears the bits it reads
//   near[2] int32[n]  near queues (double buffer)
//   touched int32[n]  vertices improved this iteration
//   far / far_key     far pile with enqueue keys, capacity 2n (compacted when
//                     it would overflow: after dropping stale entries each
//                     vertex appears at most once)
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <limits>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <string>
#include <vector>

#include "gfx_device.cuh"
#include "gfx_expand.cuh"
#include "gfx_internal.cuh"
#include "gfx_scan.cuh"
#include "gfx_sssp.cuh"

namespace gfx {

// kLate: emit every improving relaxation (duplicates allowed) and leave the
// once-per-iteration dedupe to the split pass (stamp test-and-set there):
// the relax chain then has no atomic round trip at all
template <class WT, bool kLate = false>
struct SsspRelaxOp {
  using WeightT = WT;  // weight stream element: int32 or the compact uint8 copy
  static constexpr bool kWeights = true, kSrcVal = true, kEmitEdge = false;
  static constexpr int kBatch = 4;
  static constexpr int kMinBlocks = 3;
  unsigned long long* dp;
  uint32_t* dist;  // 32-bit mirror of dp's distance (half the probe footprint)
  uint32_t* mark;  // enqueued-this-iteration bitmap
  uint32_t cur[kBatch];
  __device__ int32_t src_value(int32_t v) const { return (int32_t)dist[v]; }
  __device__ void prefetch(const int32_t* d) {
#pragma unroll
    for (int u = 0; u < kBatch; ++u) cur[u] = d[u] >= 0 ? dist[d[u]] : 0u;
  }
  // atomic_min relax (operators.py:111-124): emit d once per iteration when
  // its distance improves.  The gate is the prefetched distance; both minima
  // are fire-and-forget reductions (no round trip on the 64-bit dp word,
  // which lives in HBM), and only the L2-resident mark bit is read back, to
  // emit each improved vertex once.  A vertex that passes the gate while a
  // concurrent relaxation lowers it further is still (correctly) emitted:
  // it did improve this iteration.
  __device__ bool visit(int u, int32_t d, int32_t s, int32_t w, int32_t sdist, int64_t) {
    const unsigned long long nd = (unsigned long long)(uint32_t)sdist + (uint32_t)w;
    if (nd >= cur[u]) return false;
    const unsigned long long key = (nd << 32) | (uint32_t)s;
    atomicMin(&dp[d], key);
    atomicMin(&dist[d], (uint32_t)nd);
    if (kLate) return true;
    const uint32_t bit = 1u << (d & 31);
    return !(atomicOr(&mark[d >> 5], bit) & bit);
  }
};

// narrow the int32 weights to bytes; flag any weight outside 0..255
__global__ void k_weights_u8(const int32_t* __restrict__ w, int64_t m, uint8_t* __restrict__ w8,
                             unsigned* __restrict__ bad) {
  unsigned any = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t x = w[i];
    any |= (x < 0 || x > 255) ? 1u : 0u;
    w8[i] = (uint8_t)x;
  }
  if (__any_sync(0xffffffffu, any) && (threadIdx.x & 31) == 0) atomicOr(bad, 1u);
}

// the graph's compact weight copy, built once (nullptr when a weight
// exceeds a byte)
static int weights_u8(gfx_graph* g, const uint8_t** out) {
  *out = nullptr;
  if (g->w8_state == 2) return GFX_OK;
  void* p = nullptr;
  GFX_TRY(scratch(g, "keep_w8", (size_t)g->m + 16, &p));
  if (g->w8_state == 0) {
    gfx_ctx* ctx = g->ctx;
    unsigned* bad = reinterpret_cast<unsigned*>(g->counters) + 60;
    GFX_CK(cudaMemsetAsync(bad, 0, 4, ctx->stream));
    GFX_LAUNCH(k_weights_u8, grid_for(g->m, 256, ctx->sm_count * 8), 256, 0, ctx->stream, g->w,
               g->m, static_cast<uint8_t*>(p), bad);
    unsigned h = 0;
    GFX_CK(cudaMemcpyAsync(&h, bad, 4, cudaMemcpyDeviceToHost, ctx->stream));
    GFX_CK(cudaStreamSynchronize(ctx->stream));
    g->w8_state = h ? 2 : 1;
    if (h) return GFX_OK;
  }
  *out = static_cast<const uint8_t*>(p);
  return GFX_OK;
}

__global__ void k_sssp_seed(unsigned long long* dp, uint32_t* dist, int32_t src, int32_t* near) {
  dp[src] = 0xFFFFFFFFull;  // dist 0, pred -1
  dist[src] = 0u;
  near[0] = src;
}

// ---------------------------------------------------------------------------
// Device-resident loop: ONE cooperative launch runs the whole near/far SSSP.
// Every CTA keeps an identical copy of the loop state (near / far counts,
// threshold, queue selectors); the phases of an iteration -- fused degree
// scan, load-balanced relax expansion, near/far split -- and the bucket
// advances (stale drop + re-split) are separated by grid barriers instead of
// kernel boundaries and a host round trip per iteration.  Same kernels'
// bodies as the host-driven loop below (expand_tasks, sssp_split_phase,
// sssp_refar_phase), same results.
// ---------------------------------------------------------------------------
namespace cg = cooperative_groups;

struct PSsspArgs {
  int64_t n, words;
  const int64_t* row;
  const int32_t* col;
  const void* wgt;  // int32 weights or their compact uint8 copy
  unsigned long long* dp;
  uint32_t* dist;
  uint32_t* mark;
  int32_t* nearq[2];
  int32_t* touched;
  int32_t* stamp;  // iteration that last enqueued each vertex (split dedupe)
  int32_t* far[2];  // the soon pile (keys below the window bound)
  int32_t* fkey[2];
  int32_t* later[2];  // the later pile (keys at or above it)
  int32_t* lkey[2];
  double win;         // window width (a multiple of delta)
  int64_t* scan;
  int64_t* rowbase;
  int32_t* part;
  unsigned long long* status;
  Counters* C;  // 3 rotating blocks
  int32_t* out_dist;
  int32_t* out_preds;
  int vec;
  double delta;
  int32_t source;
  gfx_iter_rec* recs;
  int64_t rec_cap;
  long long* summary;
};

constexpr double kSsspWindow = 4.0;  // the soon pile's window, in deltas (s24 sweep 2 / 4 / 8)

struct PSCtl {
  long long nnear, nfar, nlater, lmin, it, ph, slots, bytes, nrec, nadv;
  int q, f, l;
  double th, fw;
  unsigned long long t0;
};

__device__ __forceinline__ unsigned long long sssp_gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

template <class WT>
__global__ void __launch_bounds__(256, 3) k_sssp_persistent(PSsspArgs a) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  WarpSmem& W = warp_smem(smem_raw);
  // the split / re-split phases' pile staging aliases the expansion's warp
  // slices (the phases are separated by grid barriers): 24 KB less shared
  // memory per CTA, i.e. that much more L1 for the distance probes
  static_assert(sizeof(PileStage) <= sizeof(WarpSmem) * kWarpsPerBlock, "pile stage must fit");
  static_assert(sizeof(PileStage3) <= sizeof(WarpSmem) * kWarpsPerBlock, "pile stage must fit");
  PileStage& S = *reinterpret_cast<PileStage*>(smem_raw);
  PileStage3& S3 = *reinterpret_cast<PileStage3*>(smem_raw);
  __shared__ ScanSmem ss;
  __shared__ PSCtl c;
  __shared__ CtaAgg agg;  // counters read back once per CTA (gfx_expand.cuh)
  const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  const int64_t gw = gtid >> 5, nw = nthr >> 5;
  const bool leader = blockIdx.x == 0 && threadIdx.x == 0;
  const WT* wgt = static_cast<const WT*>(a.wgt);
  // ---- init: (dist | pred) and the distance mirror at "unreached" (the
  // source's words written with its values in the same pass), marks clear
  for (int64_t v = gtid; v < a.n; v += nthr) {
    const bool src = v == a.source;
    a.dp[v] = src ? 0xFFFFFFFFull : ~0ull;  // dist 0, pred -1
    a.dist[v] = src ? 0u : 0xFFFFFFFFu;
  }
  for (int64_t i = gtid; i <= a.words; i += nthr) a.mark[i] = 0u;
  for (int64_t v = gtid; v < a.n; v += nthr) a.stamp[v] = 0;
  for (int64_t i = gtid; i < 3 * (int64_t)(sizeof(Counters) / 8); i += nthr)
    reinterpret_cast<unsigned long long*>(a.C)[i] = 0ull;
  if (leader) a.nearq[0][0] = a.source;
  if (threadIdx.x == 0) {
    c.nnear = 1;
    c.nfar = c.nlater = c.it = c.ph = c.slots = c.bytes = c.nrec = c.nadv = 0;
    c.q = c.f = c.l = 0;
    c.lmin = 0xFFFFFFFFll;  // no later entry
    c.th = a.delta;
    c.fw = a.delta + a.win;
  }
  grid.sync();
  for (;;) {
    Counters* cur = &a.C[c.ph % 3];
    if (blockIdx.x == 0 && threadIdx.x < (int)(sizeof(Counters) / 8))
      reinterpret_cast<unsigned long long*>(&a.C[(c.ph + 1) % 3])[threadIdx.x] = 0ull;
    if (c.nnear == 0) {
      if (c.nfar == 0 && c.nlater == 0) break;
      if (c.nlater + c.nfar > 3 * a.n) {
        // later-pile capacity guard: drop its stale entries (then <= n remain)
        sssp_refar_phase(S, a.later[c.l], a.lkey[c.l], c.nlater, a.dist, c.th, 0, a.nearq[c.q],
                         &cur->aux2, a.later[c.l ^ 1], a.lkey[c.l ^ 1], &cur->aux3);
        grid.sync();
        if (threadIdx.x == 0) {
          c.nlater = (long long)ld_volatile_u64(&cur->aux3);
          c.l ^= 1;
          c.ph += 1;
        }
        __syncthreads();
        continue;
      }
      // advance_bucket (near_far.py:63-85): threshold += delta, drop stale
      // far entries, re-split the rest -- the soon pile while it lasts, then
      // the later pile under the next window
      const double th = c.th + a.delta;
      // while th does not pass the smallest later key, every key below th
      // is in the soon pile, so only it is re-split (its entries at or above
      // the window bound fw join the later pile); otherwise both piles are,
      // under a new window -- the near set is exactly the one-pile loop's
      const bool from_soon = c.nfar > 0 && th <= (double)c.lmin;
      const double fw = from_soon ? c.fw : th + a.win;
      if (from_soon) {
        sssp_refar2_phase(S3, a.far[c.f], a.fkey[c.f], c.nfar, a.dist, th, fw, a.nearq[c.q],
                          &cur->out_len, a.far[c.f ^ 1], a.fkey[c.f ^ 1], &cur->aux1,
                          a.later[c.l] + c.nlater, a.lkey[c.l] + c.nlater, &cur->aux3,
                          &cur->aux2);
      } else {
        if (c.nfar > 0)
          sssp_refar2_phase(S3, a.far[c.f], a.fkey[c.f], c.nfar, a.dist, th, fw, a.nearq[c.q],
                            &cur->out_len, a.far[c.f ^ 1], a.fkey[c.f ^ 1], &cur->aux1,
                            a.later[c.l ^ 1], a.lkey[c.l ^ 1], &cur->aux3, &cur->aux2);
        sssp_refar2_phase(S3, a.later[c.l], a.lkey[c.l], c.nlater, a.dist, th, fw, a.nearq[c.q],
                          &cur->out_len, a.far[c.f ^ 1], a.fkey[c.f ^ 1], &cur->aux1,
                          a.later[c.l ^ 1], a.lkey[c.l ^ 1], &cur->aux3, &cur->aux2);
      }
      grid.sync();
      if (threadIdx.x == 0) {
        c.bytes += 8 * (from_soon ? c.nfar : c.nfar + c.nlater);
        c.th = th;
        c.fw = fw;
        c.nnear = (long long)ld_volatile_u64(&cur->out_len);
        c.nfar = (long long)ld_volatile_u64(&cur->aux1);
        const long long lmin = 0xFFFFFFFFll - (long long)ld_volatile_u64(&cur->aux2);
        if (from_soon) {
          c.nlater += (long long)ld_volatile_u64(&cur->aux3);
          c.lmin = c.lmin < lmin ? c.lmin : lmin;
        } else {
          c.nlater = (long long)ld_volatile_u64(&cur->aux3);
          c.lmin = lmin;
          c.l ^= 1;
        }
        c.f ^= 1;
        c.ph += 1;
        c.nadv += 1;
      }
      __syncthreads();
      continue;
    }
    if (threadIdx.x == 0) {
      c.it += 1;
      c.t0 = sssp_gtime();
    }
    __syncthreads();
    const int32_t* F = a.nearq[c.q];
    const int64_t nf = c.nnear;
    const int64_t stiles = (nf + kScanTileItems - 1) / kScanTileItems;
    for (int64_t t = blockIdx.x; t < stiles; t += gridDim.x)
      scan_tile(t, stiles, F, nf, a.row, a.scan, a.rowbase, a.part, a.status, (unsigned)c.ph + 1u,
                cur, ss);
    grid.sync();
    cta_read_ctrs(agg, cur);
    {
      // improving relaxations emitted with duplicates, deduplicated by the
      // split (measured: delta 4 6.78 -> 6.12 ms, delta 32 7.08 -> 6.17 at s24)
      SsspRelaxOp<WT, true> op{a.dp, a.dist, a.mark, {}};
      expand_tasks(W, op, F, nf, a.scan, a.rowbase, a.part, (int64_t)agg.rd[3],
                   (int64_t)agg.rd[2], a.col, wgt, a.touched, &cur->out_len, gw, nw, &agg);
    }
    for (int64_t i = gtid; i < stiles; i += nthr) a.status[i] = 0ull;
    grid.sync();
    cta_read_ctrs(agg, cur);
    const int64_t ntouched = (int64_t)agg.rd[0];
    sssp_split_late_phase(S, a.touched, ntouched, a.dist, a.stamp, (int32_t)c.it, c.th,
                          a.nearq[c.q ^ 1], &cur->aux0, a.far[c.f] + c.nfar, a.fkey[c.f] + c.nfar,
                          &cur->aux1);
    grid.sync();
    cta_read_ctrs(agg, cur);
    const long long slots = (long long)agg.rd[2];
    // improved vertices, each once (the touched list holds duplicates)
    const long long nimproved = (long long)(agg.rd[4] + agg.rd[5]);
    const long long bytes = 20 * nf + 8 * slots + 8 * nimproved;
    if (leader && c.nrec < a.rec_cap) {
      gfx_iter_rec r{};
      r.iteration = c.it;
      r.frontier_in = nf;
      r.frontier_out = nimproved;
      r.edges = slots;
      r.work = slots;
      r.bytes_alg = bytes;
      r.n_u = c.nfar + (long long)agg.rd[5];
      r.ms = (float)((sssp_gtime() - c.t0) * 1e-6);
      a.recs[c.nrec] = r;
    }
    if (threadIdx.x == 0) {
      c.nrec += 1;
      c.slots += slots;
      c.bytes += bytes;
      c.nnear = (long long)agg.rd[4];
      c.nfar += (long long)agg.rd[5];
      c.q ^= 1;
      c.ph += 1;
    }
    __syncthreads();
    if (c.nfar > a.n) {
      // capacity guard: drop stale far entries (each vertex then appears once)
      Counters* g2 = &a.C[c.ph % 3];
      if (blockIdx.x == 0 && threadIdx.x < (int)(sizeof(Counters) / 8))
        reinterpret_cast<unsigned long long*>(&a.C[(c.ph + 1) % 3])[threadIdx.x] = 0ull;
      sssp_refar_phase(S, a.far[c.f], a.fkey[c.f], c.nfar, a.dist, c.th, 0, a.nearq[c.q],
                       &g2->aux2, a.far[c.f ^ 1], a.fkey[c.f ^ 1], &g2->aux1);
      grid.sync();
      if (threadIdx.x == 0) {
        c.nfar = (long long)ld_volatile_u64(&g2->aux1);
        c.f ^= 1;
        c.ph += 1;
      }
      __syncthreads();
    }
  }
  sssp_unpack_phase(a.dp, a.n, a.out_dist, a.out_preds, a.vec, gtid, nthr);
  if (leader) {
    a.summary[0] = c.it;
    a.summary[1] = c.slots;
    a.summary[2] = c.bytes;
    a.summary[3] = c.nrec < a.rec_cap ? c.nrec : a.rec_cap;
    a.summary[4] = c.nadv;
  }
}

template <class WT>
static int launch_sssp_persistent(gfx_ctx* ctx, PSsspArgs& a) {
  static int per_sm = 0;
  const int smem = expand_smem_bytes();
  if (per_sm == 0) {
    GFX_CK(cudaFuncSetAttribute(k_sssp_persistent<WT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                smem));
    GFX_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sssp_persistent<WT>, 256,
                                                         smem));
    if (per_sm < 1) {
      set_error("k_sssp_persistent cannot be resident");
      return GFX_ECUDA;
    }
  }
  void* kargs[] = {&a};
  GFX_CK(cudaLaunchCooperativeKernel((const void*)k_sssp_persistent<WT>,
                                     dim3(per_sm * ctx->sm_count), dim3(256), kargs, smem,
                                     ctx->stream));
  count_launch();
  return GFX_OK;
}

int sssp_run(gfx_graph* g, int64_t source, double delta, int32_t* dist, int32_t* preds,
             gfx_iter_rec* recs, int64_t rec_cap, gfx_stats* st) {
  gfx_ctx* ctx = g->ctx;
  const int64_t n = g->n;
  unsigned long long* dp;
  uint32_t* dist32;
  uint32_t* mark;
  int32_t *nearA, *nearB, *touched, *far, *fkey, *far2, *fkey2, *part;
  int64_t *scan, *rowbase;
  GFX_TRY(scratch_t(g, "sssp_dp", n, &dp));
  // distances and the mark bitmap in one allocation: one persisting L2
  // window covers both random-probe targets
  const int64_t dist_words = (n + 63) / 64 * 64;
  GFX_TRY(scratch_t(g, "sssp_dist_mark", dist_words + g->words + 1, &dist32));
  mark = dist32 + dist_words;
  GFX_TRY(scratch_t(g, "q_order", n + 1, &nearA));
  GFX_TRY(scratch_t(g, "sssp_nearB", n + 1, &nearB));
  GFX_TRY(scratch_t(g, "sssp_touched", n + 1, &touched));
  GFX_TRY(scratch_t(g, "sssp_far", 2 * n + 64, &far));
  GFX_TRY(scratch_t(g, "sssp_fkey", 2 * n + 64, &fkey));
  GFX_TRY(scratch_t(g, "sssp_far2", 2 * n + 64, &far2));
  GFX_TRY(scratch_t(g, "sssp_fkey2", 2 * n + 64, &fkey2));
  GFX_TRY(scratch_t(g, "q_scan", n + 2, &scan));
  GFX_TRY(scratch_t(g, "q_rowbase", n + 1, &rowbase));
  GFX_TRY(scratch_t(g, "q_part", part_capacity(g->m, g->n), &part));

  const uint8_t* w8 = nullptr;
  if (!getenv("GFX_SSSP_W32")) GFX_TRY(weights_u8(g, &w8));
  Counters* C = g->counters;  // C[0]/C[1]: near sizes, C[2]: relax plan, C[3]: far
  auto* pin = static_cast<Counters*>(ctx->pinned);
  const int grid = ctx->sm_count * 8;

  // A persisting-L2 window over the distances + marks measured 11-14 %
  // SLOWER on B200 (s24: delta 4 7.51 -> 6.67 ms without it, delta 32 8.15 ->
  // 7.16): the carve-out takes L2 from everything else.  GFX_L2_PERSIST=1
  // restores it for experiments.
  const bool l2p = getenv("GFX_L2_PERSIST") != nullptr;
  if (l2p) l2_window(ctx, dist32, (dist_words + g->words + 1) * sizeof(uint32_t), true);
  // the device-resident loop (one cooperative launch, no host round trip
  // per iteration, duplicates deduplicated in the split) wins at every
  // delta measured at s24: 4 / 32 / 128 / one bucket 6.04 / 6.12 / 6.36 /
  // 6.41 ms against 8.67 / 7.17 / 7.12 / 7.10 for the host-driven kernels.
  // GFX_SSSP_LOOP=host forces the host-driven loop.
  const char* loop_env = getenv("GFX_SSSP_LOOP");
  const bool dev_loop = loop_env ? std::string(loop_env) != "host" : true;
  if (dev_loop) {
    PSsspArgs a{};
    a.n = n;
    a.words = g->words;
    a.row = g->row;
    a.col = g->col;
    a.wgt = w8 ? static_cast<const void*>(w8) : static_cast<const void*>(g->w);
    a.dp = dp;
    a.dist = dist32;
    a.mark = mark;
    a.nearq[0] = nearA;
    a.nearq[1] = nearB;
    a.touched = touched;
    // duplicates allowed: up to one entry per relaxed slot of an iteration
    GFX_TRY(scratch_t(g, "psssp_touched_dup", g->m + n + 1, &a.touched));
    GFX_TRY(scratch_t(g, "psssp_stamp", n + 1, &a.stamp));
    a.far[0] = far;
    a.far[1] = far2;
    a.fkey[0] = fkey;
    a.fkey[1] = fkey2;
    // the later pile: appended by soon-pile advances, compacted above 3n
    GFX_TRY(scratch_t(g, "psssp_later0", 4 * n + 64, &a.later[0]));
    GFX_TRY(scratch_t(g, "psssp_later1", 4 * n + 64, &a.later[1]));
    GFX_TRY(scratch_t(g, "psssp_lkey0", 4 * n + 64, &a.lkey[0]));
    GFX_TRY(scratch_t(g, "psssp_lkey1", 4 * n + 64, &a.lkey[1]));
    // window = kSsspWindow deltas (GFX_SSSP_WIN=<k> for sweeps; 0 = one far pile)
    double kwin = kSsspWindow;
    if (const char* e = getenv("GFX_SSSP_WIN")) kwin = atof(e);
    a.win = kwin > 0 ? kwin * delta : std::numeric_limits<double>::infinity();
    a.scan = scan;
    a.rowbase = rowbase;
    a.part = part;
    const int64_t stiles_max = std::max<int64_t>(1, (n + kScanTileItems - 1) / kScanTileItems);
    GFX_TRY(scratch_t(g, "psssp_status", stiles_max + 1, &a.status));
    GFX_CK(cudaMemsetAsync(a.status, 0, (stiles_max + 1) * 8, ctx->stream));
    a.C = C;
    a.out_dist = dist;
    a.out_preds = preds;
    a.vec = ((reinterpret_cast<uintptr_t>(dist) | reinterpret_cast<uintptr_t>(preds) |
              reinterpret_cast<uintptr_t>(dp)) & 15) == 0 ? 1 : 0;
    a.delta = delta;
    a.source = (int32_t)source;
    const int64_t cap = 1 << 16;
    GFX_TRY(scratch_t(g, "psssp_recs", cap, &a.recs));
    a.rec_cap = cap;
    GFX_TRY(scratch_t(g, "psssp_summary", 8, &a.summary));
    GFX_CK(cudaEventRecord(ctx->ev0, ctx->stream));
    if (w8) GFX_TRY(launch_sssp_persistent<uint8_t>(ctx, a));
    else GFX_TRY(launch_sssp_persistent<int32_t>(ctx, a));
    GFX_CK(cudaEventRecord(ctx->ev1, ctx->stream));
    long long summary[8];
    GFX_CK(cudaMemcpyAsync(summary, a.summary, 5 * sizeof(long long), cudaMemcpyDeviceToHost,
                           ctx->stream));
    GFX_CK(cudaStreamSynchronize(ctx->stream));
    if (l2p) l2_window(ctx, nullptr, 0, false);
    float ms = 0.f;
    GFX_CK(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
    const int64_t nrec = std::min<int64_t>(summary[3], recs ? rec_cap : 0);
    if (nrec > 0)
      GFX_CK(cudaMemcpy(recs, a.recs, nrec * sizeof(gfx_iter_rec), cudaMemcpyDeviceToHost));
    if (st) {
      *st = gfx_stats{};
      st->iterations = summary[0];
      st->edges_traversed = summary[1];
      st->work_slots = summary[1];
      st->bytes_alg = summary[2];
      st->device_ms = ms;
      st->num_records = nrec;
      GFX_TRY(reached_stats(g, dist, &st->reached, &st->edges_reached));
    }
    return GFX_OK;
  }
  GFX_CK(cudaEventRecord(ctx->ev0, ctx->stream));
  GFX_CK(cudaMemsetAsync(dp, 0xFF, n * sizeof(unsigned long long), ctx->stream));
  GFX_CK(cudaMemsetAsync(dist32, 0xFF, n * sizeof(uint32_t), ctx->stream));
  GFX_CK(cudaMemsetAsync(mark, 0, (g->words + 1) * sizeof(uint32_t), ctx->stream));
  GFX_CK(cudaMemsetAsync(C, 0, 4 * sizeof(Counters), ctx->stream));
  GFX_LAUNCH(k_sssp_seed, 1, 1, 0, ctx->stream, dp, dist32, (int32_t)source, nearA);
  // near count lives in C[cur].out_len
  int curq = 0;
  unsigned long long one = 1;
  GFX_CK(cudaMemcpyAsync(&C[0].out_len, &one, 8, cudaMemcpyHostToDevice, ctx->stream));

  int64_t nnear = 1, nfar = 0, it = 0, slots_total = 0, bytes_total = 0, nrec = 0;
  double threshold = delta;
  int32_t* nearq[2] = {nearA, nearB};
  while (nnear > 0 || nfar > 0) {
    if (nnear == 0) {
      // advance_bucket: threshold += delta, drop stale, re-split
      threshold += delta;
      Counters* nxt = &C[curq];
      GFX_CK(cudaMemsetAsync(nxt, 0, sizeof(Counters), ctx->stream));
      GFX_CK(cudaMemsetAsync(&C[3].aux1, 0, 8, ctx->stream));
      GFX_LAUNCH(k_sssp_refar, grid_for(nfar, 256, grid), 256, 0, ctx->stream, far, fkey, nfar,
                 dist32, threshold, 1, nearq[curq], &nxt->out_len, far2, fkey2, &C[3].aux1);
      GFX_CK(cudaMemcpyAsync(pin, C, 4 * sizeof(Counters), cudaMemcpyDeviceToHost, ctx->stream));
      GFX_CK(cudaStreamSynchronize(ctx->stream));
      bytes_total += 8 * nfar;
      nnear = (int64_t)pin[curq].out_len;
      nfar = (int64_t)pin[3].aux1;
      std::swap(far, far2);
      std::swap(fkey, fkey2);
      GFX_CK(cudaMemcpyAsync(&C[3].aux0, &pin[3].aux1, 8, cudaMemcpyHostToDevice, ctx->stream));
      continue;
    }
    ++it;
    float ms = 0.f;
    if (ctx->timing) GFX_CK(cudaEventRecord(ctx->lev0, ctx->stream));
    Counters* cur = &C[curq];
    Counters* nxt = &C[curq ^ 1];
    GFX_CK(cudaMemsetAsync(&C[2], 0, sizeof(Counters), ctx->stream));
    GFX_CK(cudaMemsetAsync(nxt, 0, sizeof(Counters), ctx->stream));
    if (w8) {
      SsspRelaxOp<uint8_t> op{dp, dist32, mark, {}};
      GFX_TRY(lb_advance(g, nearq[curq], &cur->out_len, nnear, &C[2], scan, rowbase, part, op,
                         touched, &C[2].out_len, w8));
    } else {
      SsspRelaxOp<int32_t> op{dp, dist32, mark, {}};
      GFX_TRY(lb_advance(g, nearq[curq], &cur->out_len, nnear, &C[2], scan, rowbase, part, op,
                         touched, &C[2].out_len));
    }
    GFX_LAUNCH(k_sssp_split, grid_for(n, 256, grid), 256, 0, ctx->stream, touched, &C[2].out_len,
               dist32, mark, threshold, nearq[curq ^ 1], &nxt->out_len, far, fkey, &C[3].aux0);
    GFX_CK(cudaGetLastError());
    if (ctx->timing) GFX_CK(cudaEventRecord(ctx->lev1, ctx->stream));
    GFX_CK(cudaMemcpyAsync(pin, C, 4 * sizeof(Counters), cudaMemcpyDeviceToHost, ctx->stream));
    GFX_CK(cudaStreamSynchronize(ctx->stream));
    if (ctx->timing) GFX_CK(cudaEventElapsedTime(&ms, ctx->lev0, ctx->lev1));
    const int64_t slots = (int64_t)pin[2].total;
    const int64_t ntouched = (int64_t)pin[2].out_len;
    const int64_t nnext = (int64_t)pin[curq ^ 1].out_len;
    const int64_t bytes = 20 * nnear + 8 * slots + 8 * ntouched;
    slots_total += slots;
    bytes_total += bytes;
    nfar = (int64_t)pin[3].aux0;
    if (recs && nrec < rec_cap) {
      gfx_iter_rec& r = recs[nrec++];
      r = gfx_iter_rec{};
      r.iteration = it;
      r.frontier_in = nnear;
      r.frontier_out = ntouched;
      r.edges = slots;
      r.work = slots;
      r.bytes_alg = bytes;
      r.ms = ms;
      r.n_u = nfar;
    }
    nnear = nnext;
    curq ^= 1;
    if (nfar > n) {
      // capacity guard: drop stale far entries (each vertex then appears once)
      GFX_CK(cudaMemsetAsync(&C[3].aux1, 0, 8, ctx->stream));
      GFX_LAUNCH(k_sssp_refar, grid_for(nfar, 256, grid), 256, 0, ctx->stream, far, fkey, nfar,
                 dist32, threshold, 0, nearq[curq], &C[2].aux2, far2, fkey2, &C[3].aux1);
      GFX_CK(cudaMemcpyAsync(pin, C, 4 * sizeof(Counters), cudaMemcpyDeviceToHost, ctx->stream));
      GFX_CK(cudaStreamSynchronize(ctx->stream));
      nfar = (int64_t)pin[3].aux1;
      std::swap(far, far2);
      std::swap(fkey, fkey2);
      GFX_CK(cudaMemcpyAsync(&C[3].aux0, &pin[3].aux1, 8, cudaMemcpyHostToDevice, ctx->stream));
    }
  }
  const int vec = ((reinterpret_cast<uintptr_t>(dist) | reinterpret_cast<uintptr_t>(preds) |
                    reinterpret_cast<uintptr_t>(dp)) & 15) == 0 ? 1 : 0;
  GFX_LAUNCH(k_sssp_unpack, grid_for(n, 256, grid), 256, 0, ctx->stream, dp, n, dist, preds, vec);
  if (l2p) l2_window(ctx, nullptr, 0, false);
  GFX_CK(cudaEventRecord(ctx->ev1, ctx->stream));
  GFX_CK(cudaEventSynchronize(ctx->ev1));
  float ms = 0.f;
  GFX_CK(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
  if (st) {
    *st = gfx_stats{};
    st->iterations = it;
    st->edges_traversed = slots_total;
    st->work_slots = slots_total;
    st->bytes_alg = bytes_total;
    st->device_ms = ms;
    st->num_records = nrec;
    GFX_TRY(reached_stats(g, dist, &st->reached, &st->edges_reached));
  }
  return GFX_OK;
}

}  // namespace gfx

using namespace gfx;

extern "C" int gfx_sssp(gfx_graph* g, int64_t source, double delta, int32_t* dist_d,
                        int32_t* preds_d, gfx_iter_rec* recs, int64_t rec_cap, gfx_stats* stats) {
  GFX_NVTX("gfx_sssp");
  GFX_REQUIRE(g, "gfx_sssp: null graph");
  GFX_REQUIRE(source >= 0 && source < g->n, "source %lld out of range", (long long)source);
  GFX_REQUIRE(g->w != nullptr,
              "sssp requires edge weights (assign_random_weights or a weighted file)");
  GFX_REQUIRE(dist_d && preds_d, "gfx_sssp: null output");
  GFX_CK(cudaSetDevice(g->ctx->device));
  const double d = (delta > 0 && !std::isnan(delta)) ? delta : INFINITY;
  return sssp_run(g, source, d, dist_d, preds_d, recs, rec_cap, stats);
}
