// Breadth-first search on sm_100a: load-balanced push expansion, bitmap pull
// (bottom-up) expansion, and the direction-optimising level loop.
//
// Reference: primitives/bfs.py:42-159 (loop), operators.py:218-266 (push
// advance), operators.py:131-153 (compare_and_swap claim), operators.py:
// 269-307 + direction.py:73-89 (pull step), operators.py:360-384 (exact
// filter), load_balance.py:157-176 (LB plan), direction.py:52-70 (decision).
//
// Device state per traversal (HBM, graph-owned scratch):
//   visited  uint32[words]   set-once claim bitmap (L2-resident: n/8 bytes)
//   front[2] uint32[words]   frontier bitmaps for pull levels (double buffer)
//   order    int32[n]        every level's frontier queue, concatenated
//   scan     int64[n+1]      exclusive degree prefix of the current queue
//   rowbase  int64[n]        row[F[i]] (saves a scattered re-read)
//   part     int32[m/T+2]    tile -> first item (LB partition)
//   lvl8     uint8[n]        depth bytes while labels are deferred (the
//                            persistent loop writes the int32 labels once,
//                            coalesced, at the end: materialize_labels)
//   head     int32[2(n+1)]   first / second in-neighbour per vertex with
//                            degree-1 / degree-2 flags (graph constant)
#include <cooperative_groups.h>
#include <cstdlib>
#include <cuda_runtime.h>

#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cmath>
#include <vector>

#include "gfx_device.cuh"
#include "gfx_direction.cuh"
#include "gfx_expand.cuh"
#include "gfx_internal.cuh"
#include "gfx_pull.cuh"
#include "gfx_scan.cuh"

namespace gfx {

// ---------------------------------------------------------------------------
// BFS push functors for the LB expansion (gfx_expand.cuh).
// Claim: test the visited bit with a plain load (a stale 0 only costs an
// atomic), then atomicOr; the first claimer wins like the reference CAS
// (operators.py:131-153, bfs.py:118-121) and writes label + pred.
// Idempotent: label test + plain store, duplicates culled afterwards by the
// bitmap filter (bfs.py:113-116, 162-166).
// ---------------------------------------------------------------------------
template <int B, bool FB = false>
struct BfsClaimOpT {
  static constexpr bool kWeights = false, kSrcVal = false, kEmitEdge = false;
  static constexpr int kBatch = B;
  static constexpr int kMinBlocks = 3;
  // pipelined adjacency loads (gfx_expand.cuh): push-only 3.10 -> 2.91 ms
  // at s24; not in the direction-optimising kernel, where the extra
  // registers spill into its pull loop
  static constexpr bool kPipeline = !FB;
  uint32_t* visited;
  int32_t* labels;
  int32_t* preds;
  int32_t depth;
  uint32_t wv[kBatch];
  uint8_t* lvl8 = nullptr;  // optional: deferred labels (depth bytes, see LabelOut)
  uint32_t* fbits = nullptr;  // optional: the new frontier as a bitmap too (pre-zeroed)
  __device__ int32_t src_value(int32_t) const { return 0; }
  __device__ void prefetch(const int32_t* d) {
#pragma unroll
    for (int u = 0; u < kBatch; ++u) wv[u] = d[u] >= 0 ? visited[d[u] >> 5] : 0xffffffffu;
  }
  __device__ bool visit(int u, int32_t d, int32_t s, int32_t, int32_t, int64_t) {
    const uint32_t bit = 1u << (d & 31);
    if (wv[u] & bit) return false;
    if (atomicOr(&visited[d >> 5], bit) & bit) return false;
    if (lvl8) lvl8[d] = (uint8_t)depth;
    else labels[d] = depth;
    preds[d] = s;
    if (FB) atomicOr(&fbits[d >> 5], bit);  // no return value: a fire-and-forget RED
    return true;
  }
};

// Push-only BFS, large levels: a claim without the atomic round trip.  A
// lane whose prefetched visited word shows d unclaimed sets the visited and
// next-frontier bits with fire-and-forget REDs and writes d's depth and
// predecessor; two lanes racing for d both write (the same depth; either
// predecessor is a frontier vertex one level up, a valid BFS parent).  The
// next queue is then read off the frontier bitmap, so it holds each vertex
// once.  Nothing is emitted by the expansion itself.
template <int B>
struct BfsLateClaimOpT {
  static constexpr bool kWeights = false, kSrcVal = false, kEmitEdge = false;
  static constexpr int kBatch = B;
  static constexpr int kMinBlocks = 3;
  static constexpr bool kPipeline = true;
  uint32_t* visited;
  int32_t* labels;
  int32_t* preds;
  int32_t depth;
  uint32_t wv[kBatch];
  uint8_t* lvl8;
  uint32_t* fbits;  // the next frontier (pre-zeroed)
  __device__ int32_t src_value(int32_t) const { return 0; }
  __device__ void prefetch(const int32_t* d) {
#pragma unroll
    for (int u = 0; u < kBatch; ++u) wv[u] = d[u] >= 0 ? visited[d[u] >> 5] : 0xffffffffu;
  }
  __device__ bool visit(int u, int32_t d, int32_t s, int32_t, int32_t, int64_t) {
    const uint32_t bit = 1u << (d & 31);
    if (wv[u] & bit) return false;
    atomicOr(&visited[d >> 5], bit);  // result unused: a RED
    if (lvl8) lvl8[d] = (uint8_t)depth;
    else labels[d] = depth;
    preds[d] = s;
    atomicOr(&fbits[d >> 5], bit);
    return false;
  }
};

using BfsClaimOp = BfsClaimOpT<kVisitBatch>;
// the single-hub level (push_tiny): fewer visits per lane in flight, more
// lanes issuing (measured: level 1 14 -> 12 us)
using BfsClaimOpTiny = BfsClaimOpT<4>;

struct BfsIdempOp {
  static constexpr bool kWeights = false, kSrcVal = false, kEmitEdge = false;
  static constexpr int kBatch = kVisitBatch;
  static constexpr int kMinBlocks = 3;
  const uint32_t* visited;
  int32_t* labels;
  int32_t* preds;
  int32_t depth;
  uint32_t wv[kBatch];
  __device__ int32_t src_value(int32_t) const { return 0; }
  __device__ void prefetch(const int32_t* d) {
#pragma unroll
    for (int u = 0; u < kBatch; ++u) wv[u] = d[u] >= 0 ? visited[d[u] >> 5] : 0xffffffffu;
  }
  __device__ bool visit(int u, int32_t d, int32_t s, int32_t, int32_t, int64_t) {
    if ((wv[u] >> (d & 31)) & 1u) return false;
    if (labels[d] != GFX_UNVISITED) return false;
    labels[d] = depth;
    preds[d] = s;
    return true;
  }
};

// ---------------------------------------------------------------------------
// Filter over a raw (possibly duplicated) idempotent output: bitmap
// test-and-set keeps one copy of each id (operators.py:360-384).  EXACT uses
// atomicOr; INEXACT a plain read-modify-write, which may let a few duplicates
// through exactly as the reference's culling contract allows
// (operators.py:315-357).  Output capacity is bounded by the raw input.
// ---------------------------------------------------------------------------
template <bool EXACT>
__global__ void __launch_bounds__(256)
    k_bitmap_filter(const int32_t* __restrict__ in, const unsigned long long* __restrict__ n_in,
                    uint32_t* __restrict__ seen, int32_t* __restrict__ out,
                    unsigned long long* __restrict__ out_len) {
  const int64_t n = (int64_t)*n_in;
  const int lane = threadIdx.x & 31;
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < n;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = base + threadIdx.x;
    bool keep = false;
    int32_t v = 0;
    if (i < n) {
      v = in[i];
      const uint32_t bit = 1u << (v & 31);
      if (EXACT) {
        keep = !(atomicOr(&seen[v >> 5], bit) & bit);
      } else {
        const uint32_t w = seen[v >> 5];
        keep = !(w & bit);
        if (keep) seen[v >> 5] = w | bit;
      }
    }
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    unsigned long long b = 0;
    if (lane == 0 && m) b = atomicAdd(out_len, (unsigned long long)__popc(m));
    b = __shfl_sync(0xffffffffu, b, 0);
    if (keep) out[b + __popc(m & ((1u << lane) - 1))] = v;
  }
}

__global__ void __launch_bounds__(256)
    k_bfs_pull(int64_t words, const uint32_t* __restrict__ nz_in,
               uint32_t* __restrict__ visited, const uint32_t* __restrict__ front,
               uint32_t* __restrict__ next, const int32_t* __restrict__ head,
               const int64_t* __restrict__ rrow, const int32_t* __restrict__ rcol,
               int count_in_edges, int32_t* __restrict__ labels, int32_t* __restrict__ preds,
               int32_t depth, Counters* __restrict__ ctr, const int32_t* __restrict__ head2) {
  __shared__ PullSmem ps[8];
  pull_groups(words, nz_in, visited, BitmapFront{front}, next, head, rrow, rcol, count_in_edges,
              LabelOut{labels, nullptr}, preds, depth, ctr,
              (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5,
              ((int64_t)gridDim.x * blockDim.x) >> 5, ps[threadIdx.x >> 5], head2);
}

// graph-constant first / second in-neighbour per vertex, for the pull
// probes: head[v] = first in-neighbour, bit 31 set when it is the only one
// (-1: none); head2[v] = second in-neighbour, bit 31 set when there is no
// third (-1: fewer than two)
__global__ void k_pull_heads(const int64_t* __restrict__ rrow, const int32_t* __restrict__ rcol,
                             int64_t n, int32_t* __restrict__ head, int32_t* __restrict__ head2) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = rrow[v], d = rrow[v + 1] - b;
    head[v] = d > 0 ? (int32_t)((uint32_t)rcol[b] | (d == 1 ? 0x80000000u : 0u)) : -1;
    head2[v] = d > 1 ? (int32_t)((uint32_t)rcol[b + 1] | (d == 2 ? 0x80000000u : 0u)) : -1;
  }
}

int refresh_pull_heads(gfx_graph* g) {
  auto it = g->scratch.find("keep_head");
  if (it == g->scratch.end() || !g->rrow) return GFX_OK;
  gfx_ctx* ctx = g->ctx;
  int32_t* h = static_cast<int32_t*>(it->second.ptr);
  GFX_LAUNCH(k_pull_heads, grid_for(g->n, 256, ctx->sm_count * 8), 256, 0, ctx->stream, g->rrow,
             g->rcol, g->n, h, h + g->n + 1);
  GFX_CK(cudaGetLastError());
  return GFX_OK;
}

// frontier bitmap -> queue (ascending within each warp's 1024-vertex span)
__device__ __forceinline__ void bitmap_to_queue(int64_t words, const uint32_t* __restrict__ bm,
                                                int32_t* __restrict__ out,
                                                unsigned long long* __restrict__ out_len,
                                                int64_t gw, int64_t nwarps) {
  const int lane = threadIdx.x & 31;
  for (int64_t grp = gw; grp * 32 < words; grp += nwarps) {
    const int64_t w = grp * 32 + lane;
    uint32_t x = w < words ? bm[w] : 0u;
    int tot;
    const int off = warp_excl_scan(__popc(x), lane, &tot);
    if (tot == 0) continue;
    unsigned long long b = 0;
    if (lane == 0) b = atomicAdd(out_len, (unsigned long long)tot);
    b = __shfl_sync(0xffffffffu, b, 0) + off;
    while (x) {
      const int k = __ffs(x) - 1;
      x &= x - 1;
      out[b++] = (int32_t)(w * 32 + k);
    }
  }
}

__global__ void __launch_bounds__(256)
    k_bitmap_to_queue(int64_t words, const uint32_t* __restrict__ bm, int32_t* __restrict__ out,
                      unsigned long long* __restrict__ out_len) {
  bitmap_to_queue(words, bm, out, out_len, (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5,
                  ((int64_t)gridDim.x * blockDim.x) >> 5);
}

// queue -> frontier bitmap (bitmap pre-zeroed)
__device__ __forceinline__ void queue_to_bitmap(const int32_t* __restrict__ F, int64_t nf,
                                                uint32_t* __restrict__ bm, int64_t tid0,
                                                int64_t nthreads) {
  for (int64_t i = tid0; i < nf; i += nthreads) {
    const int32_t v = F[i];
    atomicOr(&bm[v >> 5], 1u << (v & 31));
  }
}

__global__ void __launch_bounds__(256)
    k_queue_to_bitmap(const int32_t* __restrict__ F, const unsigned long long* __restrict__ nf_d,
                      uint32_t* __restrict__ bm) {
  queue_to_bitmap(F, (int64_t)*nf_d, bm, blockIdx.x * (int64_t)blockDim.x + threadIdx.x,
                  (int64_t)gridDim.x * blockDim.x);
}

__global__ void k_bfs_seed(int32_t src, int32_t* labels, uint32_t* visited, int32_t* order,
                           Counters* prev) {
  labels[src] = 0;
  visited[src >> 5] = 1u << (src & 31);
  order[0] = src;
  prev->out_len = 1;
}

// reached vertices and E_r = sum of out-degrees of reached vertices (the
// paper's TEPS numerator)
__global__ void __launch_bounds__(256)
    k_reached_stats(const int32_t* __restrict__ labels, const int64_t* __restrict__ row,
                    int64_t n, Counters* __restrict__ ctr) {
  unsigned long long cnt = 0, deg = 0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    if (labels[v] != GFX_UNVISITED) {
      ++cnt;
      deg += (unsigned long long)(row[v + 1] - row[v]);
    }
  }
  cnt = warp_sum_u64(cnt);
  deg = warp_sum_u64(deg);
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&ctr->aux0, cnt);
    atomicAdd(&ctr->aux1, deg);
  }
}

int reached_stats(gfx_graph* g, const int32_t* labels, int64_t* reached, int64_t* edges) {
  gfx_ctx* ctx = g->ctx;
  Counters* c = g->counters + 2;
  GFX_CK(cudaMemsetAsync(c, 0, sizeof(Counters), ctx->stream));
  GFX_LAUNCH(k_reached_stats, grid_for(g->n, 256, ctx->sm_count * 8), 256, 0, ctx->stream, labels, g->row,
                                                                                   g->n, c);
  GFX_CK(cudaGetLastError());
  auto* pin = static_cast<Counters*>(ctx->pinned);
  GFX_CK(cudaMemcpyAsync(pin, c, sizeof(Counters), cudaMemcpyDeviceToHost, ctx->stream));
  GFX_CK(cudaStreamSynchronize(ctx->stream));
  *reached = (int64_t)pin->aux0;
  *edges = (int64_t)pin->aux1;
  return GFX_OK;
}

// ---------------------------------------------------------------------------
// Per-level degree post-pass (statistics only, skipped when the ctx's stats
// detail is 0): out_deg[d] / in_deg[d] = sums over vertices at depth d.  From
// it: E_r = sum of out_deg (the paper's TEPS numerator), and for undirected
// graphs the reference's pull-level edges_traversed (sum of in-degrees of the
// unvisited set, bfs.py:152-153) = m - sum of degrees at depths < d-1... i.e.
// everything visited before the level.
// ---------------------------------------------------------------------------
constexpr int kLevelSmem = 64;

__global__ void __launch_bounds__(256)
    k_level_degrees(const int32_t* __restrict__ labels, const int64_t* __restrict__ row,
                    int64_t n, int64_t levels, unsigned long long* __restrict__ out_deg) {
  __shared__ unsigned long long hist[kLevelSmem];
  const bool small = levels <= kLevelSmem;
  if (small)
    for (int i = threadIdx.x; i < kLevelSmem; i += blockDim.x) hist[i] = 0ull;
  __syncthreads();
  // depths 0..7 (nearly every vertex of a small-world graph) are summed in
  // registers and reduced per warp; deeper ones go to the histogram
  constexpr int kReg = 8;
  unsigned long long acc[kReg];
#pragma unroll
  for (int k = 0; k < kReg; ++k) acc[k] = 0ull;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int32_t l = labels[v];
    if (l == GFX_UNVISITED || l >= levels) continue;
    const unsigned long long d = (unsigned long long)(row[v + 1] - row[v]);
    if (l < kReg) {
#pragma unroll
      for (int k = 0; k < kReg; ++k) acc[k] += (l == k) ? d : 0ull;
    } else if (small) {
      atomicAdd(&hist[l], d);
    } else {
      atomicAdd(&out_deg[l], d);
    }
  }
#pragma unroll
  for (int k = 0; k < kReg; ++k) {
    const unsigned long long w = warp_sum_u64(acc[k]);
    if ((threadIdx.x & 31) == 0 && w && k < levels) {
      if (small) atomicAdd(&hist[k], w); else atomicAdd(&out_deg[k], w);
    }
  }
  __syncthreads();
  if (small)
    for (int i = threadIdx.x; i < levels; i += blockDim.x)
      if (hist[i]) atomicAdd(&out_deg[i], hist[i]);
}

int bfs_level_stats(gfx_graph* g, const int32_t* labels, int64_t depth, gfx_iter_rec* recs,
                    int64_t nrec, gfx_stats* st) {
  gfx_ctx* ctx = g->ctx;
  if (!ctx->stats_detail) return GFX_OK;
  const int64_t levels = depth + 1;
  unsigned long long* deg = nullptr;
  GFX_TRY(scratch_t(g, "lvl_deg", levels + 1, &deg));
  GFX_CK(cudaMemsetAsync(deg, 0, (levels + 1) * 8, ctx->stream));
  GFX_LAUNCH(k_level_degrees, grid_for(g->n, 256, ctx->sm_count * 8), 256, 0, ctx->stream, labels,
             g->row, g->n, levels, deg);
  std::vector<unsigned long long> h(levels + 1);
  GFX_CK(cudaMemcpyAsync(h.data(), deg, (levels + 1) * 8, cudaMemcpyDeviceToHost, ctx->stream));
  GFX_CK(cudaStreamSynchronize(ctx->stream));
  int64_t e_r = 0;
  for (int64_t l = 0; l < levels; ++l) e_r += (int64_t)h[l];
  st->edges_reached = e_r;
  if (!(g->flags & GFX_GRAPH_UNDIRECTED)) return GFX_OK;
  // undirected pull levels: edges = m - degrees of depths 0..d-1
  int64_t visited_deg = 0, total = 0;
  for (int64_t i = 0; i < nrec; ++i) {
    const int64_t d = recs[i].iteration;  // level d expands depth d-1
    visited_deg += (int64_t)h[d - 1];
    if (recs[i].edges < 0) recs[i].edges = g->m - visited_deg;
    total += recs[i].edges;
  }
  st->edges_traversed = total;
  return GFX_OK;
}

struct BfsBuffers {
  uint32_t *visited, *front0, *front1, *front2;
  int32_t *order, *part, *raw;
  int64_t *scan, *rowbase;
};

static int bfs_buffers(gfx_graph* g, bool idemp, BfsBuffers* b) {
  const int64_t n = g->n, W = g->words;
  GFX_TRY(scratch_t(g, "bfs_visited", W, &b->visited));
  GFX_TRY(scratch_t(g, "bfs_front0", W, &b->front0));
  GFX_TRY(scratch_t(g, "bfs_front1", W, &b->front1));
  GFX_TRY(scratch_t(g, "bfs_front2", W, &b->front2));
  GFX_TRY(scratch_t(g, "q_order", n + 1, &b->order));
  GFX_TRY(scratch_t(g, "q_scan", n + 2, &b->scan));
  GFX_TRY(scratch_t(g, "q_rowbase", n + 1, &b->rowbase));
  GFX_TRY(scratch_t(g, "q_part", part_capacity(g->m, g->n), &b->part));
  b->raw = nullptr;
  if (idemp) GFX_TRY(scratch_t(g, "q_raw", g->m + 1, &b->raw));
  return GFX_OK;
}

// one push level over the queue at F (size in prev->out_len); winners are
// appended at out; cur counters receive out_len / total.
static int push_level(gfx_graph* g, const BfsBuffers& B, const int32_t* F,
                      const Counters* prev_d, int64_t nf_host, Counters* cur_d, int32_t depth,
                      bool idemp, bool exact, int32_t* labels, int32_t* preds, int32_t* out) {
  gfx_ctx* ctx = g->ctx;
  const unsigned long long* nf_d = &prev_d->out_len;
  if (!idemp) {
    BfsClaimOp op{B.visited, labels, preds, depth, {}};
    return lb_advance(g, F, nf_d, nf_host, cur_d, B.scan, B.rowbase, B.part, op, out,
                      &cur_d->out_len);
  }
  // raw output (duplicates allowed) counted in aux1, then filtered into out
  BfsIdempOp op{B.visited, labels, preds, depth, {}};
  GFX_TRY(lb_advance(g, F, nf_d, nf_host, cur_d, B.scan, B.rowbase, B.part, op, B.raw,
                     &cur_d->aux1));
  const int grid = ctx->sm_count * 4;
  if (exact)
    GFX_LAUNCH((k_bitmap_filter<true>), grid, 256, 0, ctx->stream, B.raw, &cur_d->aux1, B.visited, out,
                                                        &cur_d->out_len);
  else
    GFX_LAUNCH((k_bitmap_filter<false>), grid, 256, 0, ctx->stream, B.raw, &cur_d->aux1, B.visited, out,
                                                         &cur_d->out_len);
  GFX_CK(cudaGetLastError());
  return GFX_OK;
}

// push-only level-synchronous BFS that keeps every level's frontier in the
// order array: level d occupies order[off[d], off[d+1]) (used by BC, which
// replays the levels like reference bc.py:73-116)
int bfs_push_levels(gfx_graph* g, int64_t source, int32_t* labels, int32_t* preds,
                    std::vector<int64_t>* off, int32_t** order_out,
                    std::vector<int64_t>* slots) {
  gfx_ctx* ctx = g->ctx;
  const int64_t n = g->n;
  BfsBuffers B;
  GFX_TRY(bfs_buffers(g, false, &B));
  Counters* C = g->counters;
  auto* pin = static_cast<Counters*>(ctx->pinned);
  GFX_TRY(fill_i32(ctx, labels, GFX_UNVISITED, n));
  GFX_CK(cudaMemsetAsync(preds, 0xFF, n * sizeof(int32_t), ctx->stream));
  GFX_CK(cudaMemsetAsync(B.visited, 0, g->words * 4, ctx->stream));
  GFX_CK(cudaMemsetAsync(C, 0, 2 * sizeof(Counters), ctx->stream));
  GFX_LAUNCH(k_bfs_seed, 1, 1, 0, ctx->stream, (int32_t)source, labels, B.visited, B.order, &C[0]);
  off->assign(1, 0);
  if (slots) slots->clear();
  int64_t nf = 1, q_off = 0, depth = 0;
  while (nf > 0) {
    ++depth;
    off->push_back(q_off + nf);
    Counters* prev = &C[(depth - 1) & 1];
    Counters* cur = &C[depth & 1];
    GFX_CK(cudaMemsetAsync(cur, 0, sizeof(Counters), ctx->stream));
    GFX_TRY(push_level(g, B, B.order + q_off, prev, nf, cur, (int32_t)depth, false, true, labels,
                       preds, B.order + q_off + nf));
    GFX_CK(cudaMemcpyAsync(pin, cur, sizeof(Counters), cudaMemcpyDeviceToHost, ctx->stream));
    GFX_CK(cudaStreamSynchronize(ctx->stream));
    if (slots) slots->push_back((int64_t)pin->total);  // sum of degrees of this level
    q_off += nf;
    nf = (int64_t)pin->out_len;
  }
  *order_out = B.order;
  return GFX_OK;
}

int bfs_host_loop(gfx_graph* g, int64_t source, int direction, bool idemp, bool exact,
                  double do_a, double do_b, int mu_edge, int32_t* labels, int32_t* preds,
                  gfx_iter_rec* recs, int64_t rec_cap, gfx_stats* st) {
  gfx_ctx* ctx = g->ctx;
  const int64_t n = g->n, m = g->m, W = g->words;
  const bool directed = !(g->flags & GFX_GRAPH_UNDIRECTED);
  if (direction != GFX_DIR_PUSH) {
    GFX_REQUIRE(g->rrow != nullptr,
                "pull traversal on a directed graph needs the reverse adjacency "
                "(gfx_graph_set_reverse)");
  }
  BfsBuffers B;
  GFX_TRY(bfs_buffers(g, idemp, &B));
  const uint32_t* nz_in = nullptr;
  int32_t* head = nullptr;
  {
    void* p = nullptr;
    GFX_TRY(scratch(g, directed ? "nz_in" : "nz_out", W * 4, &p));
    nz_in = static_cast<const uint32_t*>(p);
    if (direction != GFX_DIR_PUSH) {
      bool fresh = false;
      GFX_TRY(scratch(g, "keep_head", (size_t)(n + 1) * 8, &p, &fresh));
      head = static_cast<int32_t*>(p);
      if (fresh)
        GFX_LAUNCH(k_pull_heads, grid_for(n, 256, ctx->sm_count * 8), 256, 0, ctx->stream,
                   g->rrow, g->rcol, n, head, head + n + 1);
    }
  }
  Counters* C = g->counters;  // C[0], C[1]: per-level double buffer
  auto* pin = static_cast<Counters*>(ctx->pinned);

  GFX_CK(cudaEventRecord(ctx->ev0, ctx->stream));
  GFX_TRY(fill_i32(ctx, labels, GFX_UNVISITED, n));
  GFX_CK(cudaMemsetAsync(preds, 0xFF, n * sizeof(int32_t), ctx->stream));
  GFX_CK(cudaMemsetAsync(B.visited, 0, W * 4, ctx->stream));
  GFX_CK(cudaMemsetAsync(C, 0, 2 * sizeof(Counters), ctx->stream));
  // level d reads its input size from C[(d-1)&1] and writes C[d&1]
  GFX_LAUNCH(k_bfs_seed, 1, 1, 0, ctx->stream, (int32_t)source, labels, B.visited, B.order, &C[0]);
  GFX_CK(cudaGetLastError());

  int64_t nf = 1, n_u = n, q_off = 0, q_end = 1;
  int mode_state = GFX_DIR_PUSH;
  bool queue_form = true;  // current frontier lives at order[q_off .. q_off+nf)
  uint32_t* fcur = B.front0;
  uint32_t* fnext = B.front1;
  int64_t depth = 0, edges_total = 0, switches = 0, nrec = 0, bytes_total = 0, work_total = 0;
  int64_t reached = 0;
  std::vector<gfx_iter_rec> lrecs;

  while (nf > 0) {
    ++depth;
    Counters* prev = &C[(depth - 1) & 1];
    Counters* cur = &C[depth & 1];
    GFX_CK(cudaMemsetAsync(cur, 0, sizeof(Counters), ctx->stream));
    n_u -= nf;
    DirEstimate est = estimate_mf_mu(n, m, nf, n_u, mu_edge);
    int mode;
    if (direction == GFX_DIR_AUTO)
      mode = decide_direction(mode_state, est, do_a, do_b);
    else if (direction == GFX_DIR_PULL)
      mode = depth > 1 ? GFX_DIR_PULL : GFX_DIR_PUSH;
    else
      mode = GFX_DIR_PUSH;
    if (mode != mode_state) ++switches;

    int64_t level_edges = 0, nout = 0, work = 0, cands = 0, bytes = 0;
    if (ctx->timing) GFX_CK(cudaEventRecord(ctx->lev0, ctx->stream));
    if (mode == GFX_DIR_PUSH) {
      if (!queue_form) {
        // previous level produced a bitmap: materialise the queue
        GFX_CK(cudaMemsetAsync(&prev->aux2, 0, 8, ctx->stream));
        GFX_LAUNCH(k_bitmap_to_queue, grid_for(W * 32, 256, ctx->sm_count * 8), 256, 0, ctx->stream, 
            W, fcur, B.order + q_end, &prev->aux2);
        q_off = q_end;
        q_end += nf;
        queue_form = true;
      }
      GFX_TRY(push_level(g, B, B.order + q_off, prev, nf, cur, (int32_t)depth, idemp, exact,
                         labels, preds, B.order + q_end));
      if (ctx->timing) GFX_CK(cudaEventRecord(ctx->lev1, ctx->stream));
      GFX_CK(cudaMemcpyAsync(pin, cur, sizeof(Counters), cudaMemcpyDeviceToHost, ctx->stream));
      GFX_CK(cudaStreamSynchronize(ctx->stream));
      level_edges = (int64_t)pin->total;
      nout = (int64_t)pin->out_len;
      work = level_edges;
      // push: frontier id + row pair per item, one col id per slot, label +
      // queue write per discovered vertex
      bytes = 20 * nf + 4 * level_edges + 8 * nout;
      q_off = q_end;
      q_end += nout;
    } else {
      if (queue_form) {
        GFX_CK(cudaMemsetAsync(fcur, 0, W * 4, ctx->stream));
        GFX_LAUNCH(k_queue_to_bitmap, grid_for(nf, 256, ctx->sm_count * 8), 256, 0, ctx->stream,
                   B.order + q_off, &prev->out_len, fcur);
        GFX_CK(cudaGetLastError());
      }
      GFX_LAUNCH(k_bfs_pull, ctx->sm_count * 8, 256, 0, ctx->stream, W, nz_in, B.visited, fcur,
                 fnext, head, g->rrow, g->rcol, directed ? 1 : 0, labels, preds,
                 (int32_t)depth, cur, head + n + 1);
      GFX_CK(cudaGetLastError());
      if (ctx->timing) GFX_CK(cudaEventRecord(ctx->lev1, ctx->stream));
      GFX_CK(cudaMemcpyAsync(pin, cur, sizeof(Counters), cudaMemcpyDeviceToHost, ctx->stream));
      GFX_CK(cudaStreamSynchronize(ctx->stream));
      // sum of in-degrees of U: counted by the kernel on directed graphs; for
      // undirected graphs the degree post-pass fills it in (-1 until then)
      level_edges = directed ? (int64_t)pin->edges : -1;
      nout = (int64_t)pin->out_len;
      work = (int64_t)pin->aux0;
      cands = (int64_t)pin->aux1;
      // pull: id + row per candidate, one col id per early-exit probe, label
      // + frontier write per discovered vertex
      bytes = 12 * cands + 4 * work + 8 * nout;
      std::swap(fcur, fnext);
      queue_form = false;
    }
    {
      lrecs.emplace_back();
      gfx_iter_rec& r = lrecs.back();
      r.iteration = depth;
      r.frontier_in = nf;
      r.frontier_out = nout;
      r.n_u = n_u;
      r.edges = level_edges;
      r.m_f = est.m_f;
      r.m_u = est.m_u;
      r.mode_before = mode_state;
      r.decision = mode;
      r.ms = 0.f;
      if (ctx->timing) GFX_CK(cudaEventElapsedTime(&r.ms, ctx->lev0, ctx->lev1));
      r.candidates = cands;
      r.work = work;
      r.bytes_alg = bytes;
      ++nrec;
    }
    if (level_edges > 0) edges_total += level_edges;
    reached += nf;
    bytes_total += bytes;
    work_total += work;
    mode_state = mode;
    nf = nout;
  }
  GFX_CK(cudaEventRecord(ctx->ev1, ctx->stream));
  GFX_CK(cudaEventSynchronize(ctx->ev1));
  float ms = 0.f;
  GFX_CK(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
  if (st) {
    st->iterations = depth;
    st->edges_traversed = edges_total;
    st->direction_switches = switches;
    st->device_ms = ms;
    st->num_records = nrec;
    st->bytes_alg = bytes_total;
    st->work_slots = work_total;
    st->reached = reached;
    st->edges_reached = -1;
    GFX_TRY(bfs_level_stats(g, labels, depth, lrecs.data(), (int64_t)lrecs.size(), st));
  }
  nrec = std::min<int64_t>((int64_t)lrecs.size(), recs ? rec_cap : 0);
  for (int64_t i = 0; i < nrec; ++i) recs[i] = lrecs[i];
  if (st) st->num_records = nrec;
  return GFX_OK;
}

// ---------------------------------------------------------------------------
// Device-resident level loop: ONE cooperative launch runs the whole
// direction-optimising BFS.  Every CTA keeps an identical copy of the loop
// state and evaluates the reference decision (direction.py:52-70, exact
// replica in gfx_direction.cuh) itself; phases are separated by grid-wide
// barriers instead of kernel boundaries and host round trips.  The grid
// barrier's gpu-scope fence also invalidates L1, so every phase reads the
// previous phase's bitmaps fresh.  Push levels pick their expansion by
// frontier size: <= 32 items (push_tiny: no scan, no plan barrier), <= 64K
// items (push_mid: 32 items per warp, hubs in a second cooperative pass),
// else the fused degree scan + load-balanced tiles (expand_tasks).
// ---------------------------------------------------------------------------
namespace cg = cooperative_groups;

struct PBfsArgs {
  int64_t n, m, words;
  const int64_t* row;
  const int32_t* col;
  const int64_t* rrow;
  const int32_t* rcol;
  const int32_t* head;
  const uint32_t* nz_in;
  uint32_t* visited;
  // three rotating frontier bitmaps: at every level front[f] is the
  // frontier, front[f+1] (zeroed) receives the next one, and front[f+2] --
  // last read one level ago -- is zeroed in passing for the level after
  uint32_t* front[3];
  int32_t* order;
  int64_t* scan;
  int64_t* rowbase;
  int32_t* part;
  unsigned long long* status;
  int32_t* labels;
  int32_t* preds;
  uint8_t* lvl8;  // depth bytes while labels are deferred (see LabelOut)
  int vec_ok;     // labels/preds 16-byte aligned: vector stores
  int64_t nnz;    // vertices with out-degree > 0 (graph constant)
  Counters* C;  // 3 rotating counter blocks
  gfx_iter_rec* recs;
  int64_t rec_cap;
  long long* summary;
  int direction, mu_edge, directed;
  double do_a, do_b;
  int32_t source;
  unsigned epoch_base;
};

struct PCtl {
  long long nf, n_u, q_off, q_end, depth, reached, edges_total, bytes_total, work_total, switches,
      nrec;
  int mode_state, queue_form, mode, fsel, direct;
  double mf, mu;
  unsigned long long t0;
};

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// kept out of line: the 128-bit division would otherwise inflate every phase's
// register allocation
__device__ __noinline__ void device_decide(long long n, long long m, long long nf, long long n_u,
                                           int mu_edge, int direction, int mode_state,
                                           long long depth, double do_a, double do_b,
                                           double* mf, double* mu, int* mode) {
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


// Deferred labels: write labels[v] = depth byte of v if visited, else
// UNVISITED, for every vertex (preds were set to -1 at launch and written at
// discovery).  A warp covers 1024 vertices in 8 independent chunks of 128;
// lane l of chunk k owns vertices 128k + 4l .. +3: one 4-byte depth load,
// one visited-word load and one 16-byte label store per lane, so every
// store instruction writes 512 contiguous bytes.
__device__ __forceinline__ void materialize_labels(const PBfsArgs& a, int64_t gw, int64_t nw) {
  const int lane = threadIdx.x & 31;
  // (a 16-vertices-per-lane form with 16-byte depth loads measured ~7 us
  // slower at s24: each of its store instructions touches half sectors)
  const int64_t nfull = a.vec_ok ? (a.n & ~(int64_t)3) : 0;
  for (int64_t base = gw * 1024; base < a.n; base += nw * 1024) {
    uint32_t vw[8], d4[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int64_t v = base + 128 * k + 4 * lane;
      vw[k] = v < a.n ? a.visited[v >> 5] : 0u;
      d4[k] = v + 3 < a.n ? *reinterpret_cast<const uint32_t*>(a.lvl8 + v) : 0u;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int64_t v = base + 128 * k + 4 * lane;
      if (v >= a.n) continue;
      const uint32_t bits = (vw[k] >> (v & 31)) & 0xFu;
      if (v < nfull) {
        int4 lab;
        lab.x = (bits & 1u) ? (int32_t)(d4[k] & 0xFF) : GFX_UNVISITED;
        lab.y = (bits & 2u) ? (int32_t)((d4[k] >> 8) & 0xFF) : GFX_UNVISITED;
        lab.z = (bits & 4u) ? (int32_t)((d4[k] >> 16) & 0xFF) : GFX_UNVISITED;
        lab.w = (bits & 8u) ? (int32_t)(d4[k] >> 24) : GFX_UNVISITED;
        *reinterpret_cast<int4*>(a.labels + v) = lab;
      } else {
        for (int j = 0; v + j < a.n; ++j)
          a.labels[v + j] = ((bits >> j) & 1u) ? (int32_t)a.lvl8[v + j] : GFX_UNVISITED;
      }
    }
  }
}

// Diagnostic timeline (compiled in only with -DGFX_BFS_TIMELINE, see
// tools/bfs_timeline.sh): per grid barrier and CTA, the globaltimer when the
// CTA arrives and when it leaves; bfs_device_loop prints the spread.
#ifdef GFX_BFS_TIMELINE
constexpr int kTlSlots = 96, kTlCtas = 1024;
__device__ unsigned long long g_tl[kTlSlots * 2 * kTlCtas + kTlCtas];
#define GSYNC()                                                                          \
  do {                                                                                   \
    __syncthreads();                                                                     \
    if (threadIdx.x == 0 && tl_slot < kTlSlots)                                          \
      g_tl[(tl_slot * 2) * kTlCtas + blockIdx.x] = globaltimer();                        \
    grid.sync();                                                                         \
    if (threadIdx.x == 0 && tl_slot < kTlSlots)                                          \
      g_tl[(tl_slot * 2 + 1) * kTlCtas + blockIdx.x] = globaltimer();                    \
    ++tl_slot;                                                                           \
  } while (0)
// GSTAMP(): the time every thread of the CTA has passed this point
constexpr int kTlStamps = 96;
__device__ unsigned long long g_tls[kTlStamps * kTlCtas];
#define GSTAMP()                                                                         \
  do {                                                                                   \
    __syncthreads();                                                                     \
    if (threadIdx.x == 0 && tl_stamp < kTlStamps)                                        \
      g_tls[tl_stamp * kTlCtas + blockIdx.x] = globaltimer();                            \
    ++tl_stamp;                                                                          \
  } while (0)
#else
#define GSYNC() grid.sync()
#define GSTAMP() \
  do {           \
  } while (0)
#endif

// kDO: direction-optimising run (pull levels and the frontier bitmaps
// compiled in); push-only runs launch the <false> instance, which carries
// none of that code (lower register pressure in its expansion loops)
template <bool kDO>
__global__ void __launch_bounds__(256, 3) k_bfs_persistent(PBfsArgs a) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  WarpSmem& W = *reinterpret_cast<WarpSmem*>(smem_raw + (threadIdx.x >> 5) * kWarpScratch);
  PullSmem& PS = *reinterpret_cast<PullSmem*>(smem_raw + (threadIdx.x >> 5) * kWarpScratch);
  __shared__ ScanSmem ss;
  __shared__ PCtl c;
  __shared__ CtaAgg agg;
  const int64_t gtid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  const int64_t gw = gtid >> 5, nw = nthr >> 5;
  const bool leader = blockIdx.x == 0 && threadIdx.x == 0;
  const unsigned long long t_start = leader ? globaltimer() : 0ull;
#ifdef GFX_BFS_TIMELINE
  int tl_slot = 0, tl_stamp = 0;
  if (threadIdx.x == 0) g_tl[kTlSlots * 2 * kTlCtas + blockIdx.x] = globaltimer();
#endif

  // ---- initialise outputs and state.  Labels are deferred: levels record
  // depths in the L2-resident byte array lvl8 and materialize_labels writes
  // every label once at the end (or at depth 255, after which labels are
  // written directly).  preds start at -1 and are written at discovery.
  if (a.vec_ok) {
    const int64_t nq = a.n >> 2;
    for (int64_t i = gtid; i < nq; i += nthr)
      reinterpret_cast<int4*>(a.preds)[i] = make_int4(-1, -1, -1, -1);
    for (int64_t i = (nq << 2) + gtid; i < a.n; i += nthr) a.preds[i] = -1;
  } else {
    for (int64_t i = gtid; i < a.n; i += nthr) a.preds[i] = -1;
  }
  // visited and the three frontier bitmaps start clear; the source's word
  // is written with its bit in the same pass (one barrier for the whole init)
  {
    const int64_t sw = a.source >> 5;
    const uint32_t sbit = 1u << (a.source & 31);
    for (int64_t i = gtid; i < a.words; i += nthr) {
      const uint32_t x = i == sw ? sbit : 0u;
      a.visited[i] = x;
      a.front[0][i] = x;
      a.front[1][i] = 0u;
      a.front[2][i] = 0u;
    }
  }
  for (int64_t i = gtid; i < 3 * (int64_t)(sizeof(Counters) / 8); i += nthr)
    reinterpret_cast<unsigned long long*>(a.C)[i] = 0ull;
  if (threadIdx.x < 8) agg.ctr[threadIdx.x] = 0ull;
  if (threadIdx.x == 0) {
    c.nf = 1;
    c.n_u = a.n;
    c.q_off = 0;
    c.q_end = 1;
    c.depth = c.reached = c.edges_total = c.bytes_total = c.work_total = 0;
    c.switches = c.nrec = 0;
    c.mode_state = GFX_DIR_PUSH;
    c.queue_form = 1;
    c.fsel = 0;
    c.direct = 0;
  }
  if (leader) {
    a.lvl8[a.source] = 0;
    a.order[0] = a.source;
  }
  GSYNC();
  const unsigned long long t_init = leader ? globaltimer() : 0ull;

  for (;;) {
    if (threadIdx.x == 0) {
      c.depth += 1;
      c.n_u -= c.nf;
      int mode;
      double mf, mu;
      device_decide(a.n, a.m, c.nf, c.n_u, a.mu_edge, a.direction, c.mode_state, c.depth, a.do_a,
                    a.do_b, &mf, &mu, &mode);
      c.mf = mf;
      c.mu = mu;
      c.mode = mode;
      if (mode != c.mode_state) c.switches += 1;
      c.t0 = globaltimer();
    }
    __syncthreads();
    if (!c.direct && c.depth == 255) {
      // depth bytes exhausted: write the labels so far, label directly from here on
      materialize_labels(a, gw, nw);
      GSYNC();
      if (threadIdx.x == 0) c.direct = 1;
      __syncthreads();
    }
    GSTAMP();  // level start (decision taken)
    const LabelOut lab{a.labels, c.direct ? nullptr : a.lvl8};
    const int32_t depth = (int32_t)c.depth;
    const int64_t nf = c.nf;
    Counters* cur = &a.C[c.depth % 3];
    if (blockIdx.x == 0 && threadIdx.x < (int)(sizeof(Counters) / 8))
      reinterpret_cast<unsigned long long*>(&a.C[(c.depth + 1) % 3])[threadIdx.x] = 0ull;
    uint32_t* fcur = a.front[c.fsel];
    uint32_t* fnext = a.front[(c.fsel + 1) % 3];
    {
      // the bitmap the NEXT level writes was last read one level ago: zero it
      // in passing (no barrier -- nothing reads it during this level)
      uint32_t* fclr = a.front[(c.fsel + 2) % 3];
      for (int64_t i = gtid; i < a.words; i += nthr) fclr[i] = 0u;
    }
    // a direction-optimising run keeps the frontier as a bitmap at every
    // level: push levels also set the new frontier's bits (fbits), so a pull
    // level never converts a queue
    GSTAMP();  // bitmap zeroing done
    uint32_t* fbits = kDO ? fnext : nullptr;
    long long level_edges = 0, nout = 0, work = 0, cands = 0, bytes = 0;

    if (!kDO || c.mode == GFX_DIR_PUSH) {
      if (!c.queue_form) {
        bitmap_to_queue(a.words, fcur, a.order + c.q_end, &cur->aux2, gw, nw);
        GSYNC();
        if (threadIdx.x == 0) {
          c.q_off = c.q_end;
          c.q_end += nf;
          c.queue_form = 1;
        }
        __syncthreads();
      }
      const int32_t* F = a.order + c.q_off;
      BfsClaimOpT<kVisitBatch, kDO> op{a.visited, a.labels, a.preds, depth, {}, lab.lvl8, fbits};
      if (nf <= 32) {
        // tiny frontier (the hub's level, the tail levels): every warp derives
        // the whole expansion plan itself -- no scan pass, no grid barrier
        // between plan and expansion
        BfsClaimOpT<4, kDO> top{a.visited, a.labels, a.preds, depth, {}, lab.lvl8, fbits};
        push_tiny(W, top, F, nf, a.row, a.col, a.order + c.q_end, &cur->out_len, &cur->total, gw,
                  nw, agg);
      } else if (nf <= kMidItems) {
        // mid-size frontier: warps expand 32 items each; hubs (rare) are set
        // aside and expanded cooperatively after one barrier
        push_mid(W, op, F, nf, a.row, a.col, a.order + c.q_end, &cur->out_len, a.part,
                 &cur->aux3, gw, nw, agg);
        cta_flush_ctrs(agg, cur);
        GSYNC();
        cta_read_ctrs(agg, cur);
        const int64_t nh = (int64_t)agg.rd[7];
        for (int64_t h0 = 0; h0 < nh; h0 += 32) {  // heavy items, 32 at a time
          const int lane = threadIdx.x & 31;
          int32_t v = 0;
          int64_t rb = 0, deg = 0;
          if (h0 + lane < nh) {
            v = F[a.part[h0 + lane]];
            rb = a.row[v];
            deg = a.row[v + 1] - rb;
          }
          int ocnt = 0;
          const int64_t t = expand_items32(W, op, v, rb, deg, a.col, a.order + c.q_end,
                                           &cur->out_len, ocnt, gw * 32 * kVisitBatch,
                                           nw * 32 * kVisitBatch);
          warp_flush(W, ocnt, a.order + c.q_end, &cur->out_len);
          if (gtid == 0) atomicAdd(&cur->total, (unsigned long long)t);
        }
      } else {
        const int64_t stiles = (nf + kScanTileItems - 1) / kScanTileItems;
        const unsigned ep = a.epoch_base + (unsigned)c.depth;
        for (int64_t t = blockIdx.x; t < stiles; t += gridDim.x)
          scan_tile(t, stiles, F, nf, a.row, a.scan, a.rowbase, a.part, a.status, ep, cur, ss);
        GSYNC();
        cta_read_ctrs(agg, cur);
        if constexpr (!kDO) {
          // push-only: late claims into the next frontier bitmap, queue from it
          uint32_t* fnb = a.front[(c.fsel + 1) % 3];
          BfsLateClaimOpT<kVisitBatch> lop{a.visited, a.labels, a.preds, depth, {}, lab.lvl8, fnb};
          expand_tasks(W, lop, F, nf, a.scan, a.rowbase, a.part, (int64_t)agg.rd[3],
                       (int64_t)agg.rd[2], a.col, nullptr, a.order + c.q_end, &cur->aux1, gw,
                       nw);
          for (int64_t i = gtid; i < stiles; i += nthr) a.status[i] = 0ull;
          GSYNC();
          bitmap_to_queue(a.words, fnb, a.order + c.q_end, &cur->out_len, gw, nw);
        } else {
          expand_tasks(W, op, F, nf, a.scan, a.rowbase, a.part, (int64_t)agg.rd[3],
                       (int64_t)agg.rd[2], a.col, nullptr, a.order + c.q_end,
                       &cur->out_len, gw, nw);
          for (int64_t i = gtid; i < stiles; i += nthr) a.status[i] = 0ull;
        }
      }
      GSTAMP();  // push body done
      GSYNC();
      cta_read_ctrs(agg, cur);
      level_edges = (long long)agg.rd[2];
      nout = (long long)agg.rd[0];
      work = level_edges;
      bytes = 20 * nf + 4 * level_edges + 8 * nout;
      if (threadIdx.x == 0) {
        c.q_off = c.q_end;
        c.q_end += nout;
        c.fsel = (c.fsel + 1) % 3;
      }
    } else {
      // dense levels (unvisited non-isolated vertices above n/8): 8
      // candidates per lane in flight and a dynamic tail; sparse levels: 4
      // in flight and the static deal.  When at most n/64 candidates remain
      // the found vertices are also queued (cheap then), so a push level
      // after this one needs no bitmap-to-queue sweep.
      const long long ncand = c.n_u - (a.n - a.nnz);
      const bool qsmall = ncand <= (a.n >> 6);
      // the first sparse pull level also writes every label (the deferred
      // labels' final pass, overlapped with the latency-bound sweep); later
      // levels label directly
      const bool fold = qsmall && !c.direct;
      Counters* actr = reinterpret_cast<Counters*>(agg.ctr);  // summed per CTA
      if (ncand * 8 > a.n)
        pull_groups<BitmapFront, 8>(a.words, a.nz_in, a.visited, BitmapFront{fcur}, fnext, a.head,
                                    a.rrow, a.rcol, a.directed, lab, a.preds, depth, actr, gw, nw,
                                    PS, a.head + a.n + 1, &cur->aux2);
      else
        pull_groups<BitmapFront, 4>(a.words, a.nz_in, a.visited, BitmapFront{fcur}, fnext, a.head,
                                    a.rrow, a.rcol, a.directed, lab, a.preds, depth, actr, gw, nw,
                                    PS, a.head + a.n + 1, nullptr,
                                    qsmall ? a.order + c.q_end : nullptr, &cur->aux3);
      // a sparse pull level deals its 1024-vertex groups statically, exactly
      // as materialize_labels walks them, and only the owning warp writes a
      // group's visited words and depth bytes: each warp labels its own
      // groups right after pulling them, with no barrier in between
      if (fold) materialize_labels(a, gw, nw);
      GSTAMP();  // pull body done
      cta_flush_ctrs(agg, cur);
      GSYNC();
      cta_read_ctrs(agg, cur);
      nout = (long long)agg.rd[0];
      work = (long long)agg.rd[4];
      cands = (long long)agg.rd[5];
      level_edges = a.directed ? (long long)agg.rd[1] : -1;
      bytes = 12 * cands + 4 * work + 8 * nout;
      if (threadIdx.x == 0) {
        c.fsel = (c.fsel + 1) % 3;
        c.queue_form = qsmall ? 1 : 0;
        if (fold) c.direct = 1;
        if (qsmall) {
          c.q_off = c.q_end;
          c.q_end += nout;
        }
      }
    }
    if (leader && c.nrec < a.rec_cap) {
      gfx_iter_rec r{};
      r.iteration = c.depth;
      r.frontier_in = nf;
      r.frontier_out = nout;
      r.n_u = c.n_u;
      r.edges = level_edges;
      r.m_f = c.mf;
      r.m_u = c.mu;
      r.mode_before = c.mode_state;
      r.decision = c.mode;
      r.ms = (float)((globaltimer() - c.t0) * 1e-6);
      r.candidates = cands;
      r.work = work;
      r.bytes_alg = bytes;
      a.recs[c.nrec] = r;
    }
    if (threadIdx.x == 0) {
      c.nrec += 1;
      c.reached += nf;
      if (level_edges > 0) c.edges_total += level_edges;
      c.bytes_total += bytes;
      c.work_total += work;
      c.mode_state = c.mode;
      c.nf = nout;
    }
    __syncthreads();
    if (c.nf == 0) break;
  }
  if (!c.direct) materialize_labels(a, gw, nw);
#ifdef GFX_BFS_TIMELINE
  GSYNC();  // the end of the label pass
#endif
  if (leader) {
    a.summary[0] = c.depth;
    a.summary[1] = c.edges_total;
    a.summary[2] = c.switches;
    a.summary[3] = c.reached;
    a.summary[4] = -1;
    a.summary[5] = c.bytes_total;
    a.summary[6] = c.work_total;
    a.summary[7] = c.nrec < a.rec_cap ? c.nrec : a.rec_cap;
    a.summary[8] = (long long)(t_init - t_start);
    a.summary[9] = (long long)(globaltimer() - t_init);
  }
}

// argument block + occupancy for the cooperative level-loop kernel
static int pbfs_setup(gfx_graph* g, int64_t source, int direction, double do_a, double do_b,
                      int mu_edge, int32_t* labels, int32_t* preds, PBfsArgs* out,
                      int* grid_blocks, int* smem_bytes) {
  gfx_ctx* ctx = g->ctx;
  const int64_t n = g->n, W = g->words;
  const bool directed = !(g->flags & GFX_GRAPH_UNDIRECTED);
  if (direction != GFX_DIR_PUSH)
    GFX_REQUIRE(g->rrow != nullptr, "pull traversal on a directed graph needs the reverse adjacency");
  BfsBuffers B;
  GFX_TRY(bfs_buffers(g, false, &B));
  PBfsArgs a{};
  a.n = n;
  a.m = g->m;
  a.words = W;
  a.row = g->row;
  a.col = g->col;
  a.rrow = g->rrow ? g->rrow : g->row;
  a.rcol = g->rcol ? g->rcol : g->col;
  {
    void* p = nullptr;
    GFX_TRY(scratch(g, directed ? "nz_in" : "nz_out", W * 4, &p));
    a.nz_in = static_cast<const uint32_t*>(p);
    bool fresh = false;
    GFX_TRY(scratch(g, "keep_head", (size_t)(n + 1) * 8, &p, &fresh));
    a.head = static_cast<const int32_t*>(p);
    if (fresh)
      GFX_LAUNCH(k_pull_heads, grid_for(n, 256, ctx->sm_count * 8), 256, 0, ctx->stream, a.rrow,
                 a.rcol, n, static_cast<int32_t*>(p), static_cast<int32_t*>(p) + n + 1);
  }
  a.visited = B.visited;
  a.front[0] = B.front0;
  a.front[1] = B.front1;
  a.front[2] = B.front2;
  a.order = B.order;
  a.scan = B.scan;
  a.rowbase = B.rowbase;
  a.part = B.part;
  const int64_t stiles_max = std::max<int64_t>(1, (n + kScanTileItems - 1) / kScanTileItems);
  GFX_TRY(scratch_t(g, "pbfs_status", stiles_max + 1, &a.status));
  a.labels = labels;
  a.preds = preds;
  a.vec_ok = ((reinterpret_cast<uintptr_t>(labels) | reinterpret_cast<uintptr_t>(preds)) & 15) == 0;
  a.nnz = g->nnz_vertices;
  GFX_TRY(scratch_t(g, "bfs_lvl8", (size_t)n + 4, &a.lvl8));
  a.C = g->counters;
  const int64_t cap = 1 << 16;  // level records kept on device (stats)
  GFX_TRY(scratch_t(g, "pbfs_recs", cap, &a.recs));
  a.rec_cap = cap;
  GFX_TRY(scratch_t(g, "pbfs_summary", 10, &a.summary));
  a.direction = direction;
  a.mu_edge = mu_edge;
  a.directed = directed ? 1 : 0;
  a.do_a = do_a;
  a.do_b = do_b;
  a.source = (int32_t)source;
  a.epoch_base = 0;
  *out = a;

  static int blocks_per_sm = 0;
  const int smem = kWarpScratch * kWarpsPerBlock;
  if (blocks_per_sm == 0) {
    if (const char* cv = getenv("GFX_BFS_CARVEOUT")) {  // L1 / shared split (percent shared)
      GFX_CK(cudaFuncSetAttribute(k_bfs_persistent<true>,
                                  cudaFuncAttributePreferredSharedMemoryCarveout, atoi(cv)));
      GFX_CK(cudaFuncSetAttribute(k_bfs_persistent<false>,
                                  cudaFuncAttributePreferredSharedMemoryCarveout, atoi(cv)));
    }
    GFX_CK(cudaFuncSetAttribute(k_bfs_persistent<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                smem));
    GFX_CK(cudaFuncSetAttribute(k_bfs_persistent<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                smem));
    int push_only_per_sm = 0;
    GFX_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&push_only_per_sm, k_bfs_persistent<false>,
                                                         256, smem));
    GFX_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, k_bfs_persistent<true>, 256,
                                                         smem));
    blocks_per_sm = std::min(blocks_per_sm, push_only_per_sm);  // one grid size for both
    if (blocks_per_sm < 1) {
      set_error("k_bfs_persistent cannot be resident");
      return GFX_ECUDA;
    }
  }
  *grid_blocks = blocks_per_sm * g->ctx->sm_count;
  *smem_bytes = smem;
  return GFX_OK;
}

int bfs_device_loop(gfx_graph* g, int64_t source, int direction, double do_a, double do_b,
                    int mu_edge, int32_t* labels, int32_t* preds, gfx_iter_rec* recs,
                    int64_t rec_cap, gfx_stats* st) {
  gfx_ctx* ctx = g->ctx;
  PBfsArgs a{};
  int blocks = 0, smem = 0;
  GFX_TRY(pbfs_setup(g, source, direction, do_a, do_b, mu_edge, labels, preds, &a, &blocks,
                     &smem));
  const int64_t stiles_max = std::max<int64_t>(1, (g->n + kScanTileItems - 1) / kScanTileItems);
  // status words must start clear; the kernel clears what it uses
  GFX_CK(cudaMemsetAsync(a.status, 0, (stiles_max + 1) * 8, ctx->stream));
  void* kargs[] = {&a};
  GFX_CK(cudaEventRecord(ctx->ev0, ctx->stream));
  GFX_CK(cudaLaunchCooperativeKernel(a.direction == GFX_DIR_PUSH
                                         ? (const void*)k_bfs_persistent<false>
                                         : (const void*)k_bfs_persistent<true>,
                                     dim3(blocks), dim3(256), kargs, smem,
                                     ctx->stream));
  count_launch();
  GFX_CK(cudaEventRecord(ctx->ev1, ctx->stream));
  long long summary[10];
  GFX_CK(cudaMemcpyAsync(summary, a.summary, sizeof(summary), cudaMemcpyDeviceToHost,
                         ctx->stream));
  GFX_CK(cudaStreamSynchronize(ctx->stream));
  float ms = 0.f;
  GFX_CK(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
#ifdef GFX_BFS_TIMELINE
  {
    std::vector<unsigned long long> tl((size_t)kTlSlots * 2 * kTlCtas + kTlCtas);
    GFX_CK(cudaMemcpyFromSymbol(tl.data(), g_tl, tl.size() * 8));
    const unsigned long long* st0 = tl.data() + (size_t)kTlSlots * 2 * kTlCtas;
    const unsigned long long t0 = *std::min_element(st0, st0 + blocks);
    fprintf(stderr, "timeline: %d CTAs, start spread %.2f us\n", blocks,
            (*std::max_element(st0, st0 + blocks) - t0) * 1e-3);
    for (int s = 0; s < kTlSlots; ++s) {
      std::vector<unsigned long long> arr(tl.begin() + (size_t)(2 * s) * kTlCtas,
                                          tl.begin() + (size_t)(2 * s) * kTlCtas + blocks);
      std::vector<unsigned long long> lev(tl.begin() + (size_t)(2 * s + 1) * kTlCtas,
                                          tl.begin() + (size_t)(2 * s + 1) * kTlCtas + blocks);
      if (arr[0] < t0) break;
      std::sort(arr.begin(), arr.end());
      std::sort(lev.begin(), lev.end());
      fprintf(stderr,
              "sync %2d arrive min %8.2f med %8.2f p90 %8.2f max %8.2f | leave min %8.2f max %8.2f"
              " | barrier %6.2f us\n",
              s, (arr.front() - t0) * 1e-3, (arr[blocks / 2] - t0) * 1e-3,
              (arr[blocks * 9 / 10] - t0) * 1e-3, (arr.back() - t0) * 1e-3,
              (lev.front() - t0) * 1e-3, (lev.back() - t0) * 1e-3,
              ((double)lev.front() - (double)arr.back()) * 1e-3);
    }
    std::vector<unsigned long long> ts((size_t)kTlStamps * kTlCtas);
    GFX_CK(cudaMemcpyFromSymbol(ts.data(), g_tls, ts.size() * 8));
    for (int k = 0; k < kTlStamps; ++k) {
      std::vector<unsigned long long> v(ts.begin() + (size_t)k * kTlCtas,
                                        ts.begin() + (size_t)k * kTlCtas + blocks);
      if (v[0] < t0) break;
      std::vector<int> ids(blocks);
      for (int b = 0; b < blocks; ++b) ids[b] = b;
      std::sort(ids.begin(), ids.end(), [&](int x, int y) { return v[x] > v[y]; });
      std::sort(v.begin(), v.end());
      fprintf(stderr, "stamp %2d min %8.2f med %8.2f p90 %8.2f max %8.2f | slowest CTAs", k,
              (v.front() - t0) * 1e-3, (v[blocks / 2] - t0) * 1e-3,
              (v[blocks * 9 / 10] - t0) * 1e-3, (v.back() - t0) * 1e-3);
      for (int b = 0; b < 6; ++b) fprintf(stderr, " %d", ids[b]);
      fprintf(stderr, "\n");
    }
    {
      static unsigned long long ph[64][8];
      GFX_CK(cudaMemcpyFromSymbol(ph, g_pull_ph, sizeof(ph)));
      const int nwarps = blocks * kWarpsPerBlock;
      for (int d = 0; d < 64; ++d)
        if (ph[d][5])
          fprintf(stderr,
                  "pull depth %d per warp (us @1.965GHz): words+list %.2f head %.2f rebuild %.2f "
                  "misses %.2f stores %.2f | groups/warp %.2f misses/group %.1f\n",
                  d, ph[d][0] / 1965.0 / nwarps, ph[d][1] / 1965.0 / nwarps,
                  ph[d][2] / 1965.0 / nwarps, ph[d][3] / 1965.0 / nwarps,
                  ph[d][4] / 1965.0 / nwarps, (double)ph[d][5] / nwarps,
                  (double)ph[d][6] / ph[d][5]);
      memset(ph, 0, sizeof(ph));
      GFX_CK(cudaMemcpyToSymbol(g_pull_ph, ph, sizeof(ph)));
    }
    std::vector<unsigned long long> zero(tl.size(), 0ull);
    GFX_CK(cudaMemcpyToSymbol(g_tl, zero.data(), zero.size() * 8));
    GFX_CK(cudaMemcpyToSymbol(g_tls, zero.data(), ts.size() * 8));
  }
#endif
  std::vector<gfx_iter_rec> lrecs((size_t)summary[7]);
  if (!lrecs.empty())
    GFX_CK(cudaMemcpy(lrecs.data(), a.recs, lrecs.size() * sizeof(gfx_iter_rec),
                      cudaMemcpyDeviceToHost));
  if (st) {
    st->iterations = summary[0];
    st->edges_traversed = summary[1];
    st->direction_switches = summary[2];
    st->reached = summary[3];
    st->edges_reached = -1;
    st->bytes_alg = summary[5];
    st->work_slots = summary[6];
    st->device_ms = ms;
    st->init_ns = summary[8];
    st->loop_ns = summary[9];
    GFX_TRY(bfs_level_stats(g, labels, summary[0], lrecs.data(), (int64_t)lrecs.size(), st));
  }
  const int64_t nrec = std::min<int64_t>((int64_t)lrecs.size(), recs ? rec_cap : 0);
  for (int64_t i = 0; i < nrec; ++i) recs[i] = lrecs[i];
  if (st) st->num_records = nrec;
  return GFX_OK;
}

// count BFS runs back to back from sources[] (one cooperative launch each, a
// single synchronisation at the end): device throughput without per-call
// host round trips.  labels/preds hold the last run.
int bfs_device_batch(gfx_graph* g, const int64_t* sources, int64_t count, int direction,
                     double do_a, double do_b, int mu_edge, int32_t* labels, int32_t* preds,
                     float* ms) {
  gfx_ctx* ctx = g->ctx;
  PBfsArgs a{};
  int blocks = 0, smem = 0;
  GFX_TRY(pbfs_setup(g, sources[0], direction, do_a, do_b, mu_edge, labels, preds, &a, &blocks,
                     &smem));
  const int64_t stiles_max = std::max<int64_t>(1, (g->n + kScanTileItems - 1) / kScanTileItems);
  GFX_CK(cudaMemsetAsync(a.status, 0, (stiles_max + 1) * 8, ctx->stream));
  GFX_CK(cudaEventRecord(ctx->ev0, ctx->stream));
  for (int64_t k = 0; k < count; ++k) {
    a.source = (int32_t)sources[k];
    void* kargs[] = {&a};
    GFX_CK(cudaLaunchCooperativeKernel(a.direction == GFX_DIR_PUSH
                                         ? (const void*)k_bfs_persistent<false>
                                         : (const void*)k_bfs_persistent<true>, dim3(blocks), dim3(256),
                                       kargs, smem, ctx->stream));
    count_launch();
  }
  GFX_CK(cudaEventRecord(ctx->ev1, ctx->stream));
  GFX_CK(cudaEventSynchronize(ctx->ev1));
  GFX_CK(cudaEventElapsedTime(ms, ctx->ev0, ctx->ev1));
  return GFX_OK;
}

// Level lists of a labelled BFS (BC's forward phase): pass A counts each
// block's vertices per level (and the levels' out-degree sums), one exclusive
// scan over the level-major (level, block) counts gives every block its
// write base per level, pass B scatters the vertices.  Warp-aggregated: each
// distinct level among a warp's 32 vertices is one shared-memory atomic.
template <bool kScatter>
__global__ void __launch_bounds__(256)
    k_level_pass(const int32_t* __restrict__ labels, const int64_t* __restrict__ row, int64_t n,
                 int L, int64_t chunk, uint32_t* __restrict__ blk,
                 unsigned long long* __restrict__ gcnt, unsigned long long* __restrict__ gslots,
                 int32_t* __restrict__ order) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned long long* s_slots = reinterpret_cast<unsigned long long*>(smem_raw);
  uint32_t* s_cnt = reinterpret_cast<uint32_t*>(smem_raw + (kScatter ? 0 : 8 * (size_t)L));
  const int nb = gridDim.x;
  for (int d = threadIdx.x; d < L; d += blockDim.x) {
    s_cnt[d] = 0;
    if (!kScatter) s_slots[d] = 0;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t b0 = blockIdx.x * chunk, b1 = min(n, b0 + chunk);
  for (int64_t vb = b0 + (threadIdx.x & ~31); vb < b1; vb += blockDim.x) {
    const int64_t v = vb + lane;
    int32_t d = v < b1 ? labels[v] : -1;
    if (d == GFX_UNVISITED || d >= L) d = -1;
    const unsigned long long deg = (!kScatter && d >= 0) ? (unsigned long long)(row[v + 1] - row[v]) : 0ull;
    unsigned rem = __ballot_sync(0xffffffffu, d >= 0);
    while (rem) {
      const int leader = __ffs(rem) - 1;
      const int32_t dl = __shfl_sync(0xffffffffu, d, leader);
      const unsigned mask = __ballot_sync(0xffffffffu, d == dl);
      if (!kScatter) {
        const unsigned long long sdeg = warp_sum_u64(d == dl ? deg : 0ull);
        if (lane == leader) {
          atomicAdd(&s_cnt[dl], (uint32_t)__popc(mask));
          atomicAdd(&s_slots[dl], sdeg);
        }
      } else {
        uint32_t gb = 0;
        if (lane == leader) gb = atomicAdd(&s_cnt[dl], (uint32_t)__popc(mask));
        gb = __shfl_sync(0xffffffffu, gb, leader);
        if (d == dl)
          order[blk[(int64_t)dl * nb + blockIdx.x] + gb + __popc(mask & ((1u << lane) - 1))] =
              (int32_t)v;
      }
      rem &= ~mask;
    }
  }
  if (!kScatter) {
    __syncthreads();
    for (int d = threadIdx.x; d < L; d += blockDim.x) {
      blk[(int64_t)d * nb + blockIdx.x] = s_cnt[d];
      if (s_cnt[d]) {
        atomicAdd(&gcnt[d], (unsigned long long)s_cnt[d]);
        atomicAdd(&gslots[d], s_slots[d]);
      }
    }
  }
}

// BC's forward phase on the direction-optimising persistent BFS: labels and
// preds as gfx_bfs writes them, then level d's vertices in
// order[off[d], off[d+1]) and slots[d] = sum of their out-degrees (the same
// contract as bfs_push_levels, whose push-only level loop needs a host
// round trip per level; the order within a level differs, which BC's
// per-vertex gathers and exact pushes do not see).  Falls back to
// bfs_push_levels for BFS trees deeper than 1024 levels.
int bfs_do_levels(gfx_graph* g, int64_t source, int32_t* labels, int32_t* preds,
                  std::vector<int64_t>* off, int32_t** order_out, std::vector<int64_t>* slots) {
  gfx_ctx* ctx = g->ctx;
  const int64_t n = g->n;
  PBfsArgs a{};
  int blocks = 0, smem = 0;
  GFX_TRY(pbfs_setup(g, source, GFX_DIR_AUTO, 0.001, 0.2, 0, labels, preds, &a, &blocks, &smem));
  const int64_t stiles_max = std::max<int64_t>(1, (n + kScanTileItems - 1) / kScanTileItems);
  GFX_CK(cudaMemsetAsync(a.status, 0, (stiles_max + 1) * 8, ctx->stream));
  void* kargs[] = {&a};
  GFX_CK(cudaLaunchCooperativeKernel((const void*)k_bfs_persistent<true>, dim3(blocks), dim3(256),
                                     kargs, smem, ctx->stream));
  count_launch();
  long long summary[10];
  GFX_CK(cudaMemcpyAsync(summary, a.summary, sizeof(summary), cudaMemcpyDeviceToHost, ctx->stream));
  GFX_CK(cudaStreamSynchronize(ctx->stream));
  const int64_t L = summary[0];  // levels 0 .. L-1 hold vertices
  if (L > 1024) return bfs_push_levels(g, source, labels, preds, off, order_out, slots);
  const int nb = (int)std::max<int64_t>(1, std::min<int64_t>(ctx->sm_count * 8, (n + 1023) / 1024));
  const int64_t chunk = (n + nb - 1) / nb;
  uint32_t* blk;
  unsigned long long* lv;
  GFX_TRY(scratch_t(g, "lvl_blk", (size_t)L * nb + 1, &blk));
  GFX_TRY(scratch_t(g, "lvl_cnt", 2 * (size_t)L + 2, &lv));
  GFX_CK(cudaMemsetAsync(lv, 0, (2 * L + 2) * 8, ctx->stream));
  GFX_LAUNCH(k_level_pass<false>, nb, 256, (size_t)L * 12 + 16, ctx->stream, labels, g->row, n,
             (int)L, chunk, blk, lv, lv + L, nullptr);
  size_t tb = 0;
  GFX_CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, blk, blk, (int64_t)L * nb, ctx->stream));
  void* tmp;
  GFX_TRY(scratch(g, "lvl_cub", tb + 16, &tmp));
  GFX_CK(cub::DeviceScan::ExclusiveSum(tmp, tb, blk, blk, (int64_t)L * nb, ctx->stream));
  count_launch();
  GFX_LAUNCH(k_level_pass<true>, nb, 256, (size_t)L * 4 + 16, ctx->stream, labels, g->row, n,
             (int)L, chunk, blk, nullptr, nullptr, a.order);
  std::vector<unsigned long long> h(2 * L);
  GFX_CK(cudaMemcpyAsync(h.data(), lv, 2 * L * 8, cudaMemcpyDeviceToHost, ctx->stream));
  GFX_CK(cudaStreamSynchronize(ctx->stream));
  off->assign(1, 0);
  if (slots) slots->clear();
  for (int64_t d = 0; d < L; ++d) {
    off->push_back(off->back() + (int64_t)h[d]);
    if (slots) slots->push_back((int64_t)h[L + d]);
  }
  *order_out = a.order;
  return GFX_OK;
}

}  // namespace gfx

using namespace gfx;

extern "C" int gfx_bfs(gfx_graph* g, int64_t source, int direction, int idempotent,
                       int filter_mode, double do_a, double do_b, int mu_edge_based, int loop,
                       int32_t* labels_d, int32_t* preds_d, gfx_iter_rec* recs, int64_t rec_cap,
                       gfx_stats* stats) {
  GFX_NVTX("gfx_bfs");
  GFX_REQUIRE(g, "gfx_bfs: null graph");
  GFX_REQUIRE(source >= 0 && source < g->n, "source %lld out of range", (long long)source);
  GFX_REQUIRE(direction == GFX_DIR_PUSH || direction == GFX_DIR_PULL || direction == GFX_DIR_AUTO,
              "unknown direction %d", direction);
  GFX_REQUIRE(labels_d && preds_d, "gfx_bfs: null output");
  if (direction == GFX_DIR_AUTO)
    GFX_REQUIRE(do_a > 0 && do_b > 0, "do_a and do_b must be positive");
  GFX_CK(cudaSetDevice(g->ctx->device));
  if (loop == GFX_LOOP_DEVICE && !idempotent)
    return bfs_device_loop(g, source, direction, do_a, do_b, mu_edge_based, labels_d, preds_d,
                           recs, rec_cap, stats);
  // INEXACT may leave duplicates (reference operators.py:315-357); the order
  // queue is sized for unique frontiers, so both modes use the exact
  // test-and-set cull, which satisfies the inexact contract as well.
  (void)filter_mode;
  return bfs_host_loop(g, source, direction, idempotent != 0, true, do_a, do_b, mu_edge_based,
                       labels_d, preds_d, recs, rec_cap, stats);
}

extern "C" int gfx_bfs_batch(gfx_graph* g, const int64_t* sources, int64_t count,
                             int direction, double do_a, double do_b, int mu_edge_based,
                             int32_t* labels_d, int32_t* preds_d, float* ms) {
  GFX_NVTX("gfx_bfs_batch");
  GFX_REQUIRE(g && sources && count > 0 && labels_d && preds_d && ms,
              "gfx_bfs_batch: bad argument");
  for (int64_t k = 0; k < count; ++k)
    GFX_REQUIRE(sources[k] >= 0 && sources[k] < g->n, "source %lld out of range",
                (long long)sources[k]);
  GFX_REQUIRE(direction == GFX_DIR_PUSH || direction == GFX_DIR_PULL || direction == GFX_DIR_AUTO,
              "unknown direction %d", direction);
  if (direction == GFX_DIR_AUTO) GFX_REQUIRE(do_a > 0 && do_b > 0, "do_a and do_b must be positive");
  GFX_CK(cudaSetDevice(g->ctx->device));
  return bfs_device_batch(g, sources, count, direction, do_a, do_b, mu_edge_based, labels_d,
                          preds_d, ms);
}

extern "C" int gfx_estimate_mf_mu(int64_t n, int64_t m, int64_t n_f, int64_t n_u, int mu_edge,
                                  double* m_f, double* m_u) {
  GFX_REQUIRE(n > 0 && m_f && m_u, "gfx_estimate_mf_mu: bad argument");
  DirEstimate e = estimate_mf_mu(n, m, n_f, n_u, mu_edge);
  *m_f = e.m_f;
  *m_u = e.m_u;
  return GFX_OK;
}
