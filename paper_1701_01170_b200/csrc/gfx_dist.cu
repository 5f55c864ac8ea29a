// Partitioned (multi-GPU) direction-optimising BFS: per-rank device engine.
//
// 1D cyclic vertex partition, owner(v) = v mod P, so the R-MAT
// hubs (low ids, generators.py:48-51 does not permute) spread over all ranks.
// Rank r stores the rows of its owned vertices (local id l = v / P) with
// GLOBAL column ids, its own labels / preds / visited bits, and per level
// either
//   push: expands its local frontier; owned destinations are claimed locally,
//         remote ones are de-duplicated per level through a bitmap over
//         global ids and emitted as (dst, src) pairs bucketed by owner; the
//         host exchanges them (NCCL all_to_all) and the owner claims them;
//   pull: the host all-gathers every rank's local frontier bitmap; the rank
//         then pulls its unvisited vertices against that gathered view.
// The direction decision needs the global n_f (allreduce on the host) and is
// the same reference formula as on one GPU (direction.py:52-70), so the
// trace equals the single-GPU trace.  The host owns the buffers that cross
// the network (send / recv pairs, local and gathered frontier bitmaps) as
// torch tensors and passes their device pointers in.
#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>

#include <vector>

#include "gfx_device.cuh"
#include "gfx_expand.cuh"
#include "gfx_internal.cuh"
#include "gfx_pull.cuh"

struct gfx_dbfs {
  gfx_ctx* ctx = nullptr;
  gfx_graph* lg = nullptr;  // local CSR (rows = owned vertices, cols = global ids)
  int P = 1, r = 0;
  int64_t n = 0, m = 0, nl = 0, ml = 0, wl = 0, wmax = 0;
  int32_t* labels = nullptr;
  int32_t* preds = nullptr;
  // host-owned exchange buffers
  unsigned long long* send = nullptr;
  unsigned long long* recv = nullptr;
  uint32_t* front_local = nullptr;  // wmax words: local frontier bitmap (pull levels)
  uint32_t* gathered = nullptr;     // P * wmax words
  int64_t send_cap = 0, recv_cap = 0;
  // engine state
  int64_t nf = 0, q_off = 0, q_end = 0, local_new = 0;
  bool queue_form = true;
  std::vector<long long> bucket_off;
};

namespace gfx {

__global__ void k_part_degrees(const int64_t* __restrict__ row, int64_t n, int P, int r,
                               int64_t nl, int64_t* __restrict__ deg) {
  for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < nl;
       l += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = l * P + r;
    deg[l] = row[v + 1] - row[v];
  }
}

// warp per owned row: copy its adjacency (global ids) into the local CSR
__global__ void k_part_copy(const int64_t* __restrict__ row, const int32_t* __restrict__ col,
                            int P, int r, int64_t nl, const int64_t* __restrict__ lrow,
                            int32_t* __restrict__ lcol) {
  const int lane = threadIdx.x & 31;
  for (int64_t l = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; l < nl;
       l += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t v = l * P + r;
    const int64_t b = row[v], e = row[v + 1], o = lrow[l];
    for (int64_t p = b + lane; p < e; p += 32) lcol[o + (p - b)] = col[p];
  }
}

// push functor: owned destinations are claimed, remote ones emitted once per
// level (the `sent` bitmap over global ids) with their source remembered
struct DistClaimOp {
  static constexpr bool kWeights = false, kSrcVal = false, kEmitEdge = false;
  static constexpr int kBatch = kVisitBatch;
  static constexpr int kMinBlocks = 3;
  uint32_t* visited;   // local bits
  uint32_t* sent;      // global bits
  int32_t* sent_src;   // global ids -> source of the emitted pair
  int32_t* labels;
  int32_t* preds;
  int32_t depth;
  int P, r;
  uint32_t wv[kBatch];
  __device__ int32_t src_value(int32_t) const { return 0; }
  __device__ void prefetch(const int32_t* d) {
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      if (d[u] < 0) {
        wv[u] = 0xffffffffu;
      } else if (d[u] % P == r) {
        const int32_t l = d[u] / P;
        wv[u] = visited[l >> 5];
      } else {
        wv[u] = sent[d[u] >> 5];
      }
    }
  }
  __device__ bool visit(int u, int32_t d, int32_t s, int32_t, int32_t, int64_t) {
    const int32_t sg = s * P + r;  // frontier items are local ids
    if (d % P == r) {
      const int32_t l = d / P;
      const uint32_t bit = 1u << (l & 31);
      if (wv[u] & bit) return false;
      if (atomicOr(&visited[l >> 5], bit) & bit) return false;
      labels[l] = depth;
      preds[l] = sg;
      return true;
    }
    const uint32_t bit = 1u << (d & 31);
    if (wv[u] & bit) return false;
    if (atomicOr(&sent[d >> 5], bit) & bit) return false;
    sent_src[d] = sg;
    return true;
  }
};

// split the expansion output: owned winners -> next queue (local ids),
// remote candidates -> send buckets (pairs dst<<32 | src), clearing their
// `sent` bits for the next level.  pass 0 counts per owner, pass 1 scatters.
template <int PASS>
__global__ void __launch_bounds__(256)
    k_dist_bucket(const int32_t* __restrict__ emit, const unsigned long long* __restrict__ n_d,
                  int P, int r, unsigned long long* __restrict__ counts,
                  unsigned long long* __restrict__ cursors, const int32_t* __restrict__ sent_src,
                  uint32_t* __restrict__ sent, unsigned long long* __restrict__ send,
                  int32_t* __restrict__ next_q, unsigned long long* __restrict__ next_len) {
  __shared__ unsigned long long hist[64];
  const int64_t n = (int64_t)*n_d;
  if (PASS == 0) {
    for (int i = threadIdx.x; i < P; i += blockDim.x) hist[i] = 0;
    __syncthreads();
  }
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t d = emit[i];
    const int o = d % P;
    if (PASS == 0) {
      atomicAdd(&hist[o], 1ull);
    } else if (o == r) {
      next_q[atomicAdd(next_len, 1ull)] = d / P;
    } else {
      const unsigned long long at = atomicAdd(&cursors[o], 1ull);
      send[at] = ((unsigned long long)(uint32_t)d << 32) | (uint32_t)sent_src[d];
      atomicAnd(&sent[d >> 5], ~(1u << (d & 31)));
    }
  }
  if (PASS == 0) {
    __syncthreads();
    for (int i = threadIdx.x; i < P; i += blockDim.x)
      if (hist[i]) atomicAdd(&counts[i], hist[i]);
  }
}

// owner side: claim received (dst, src) pairs
__global__ void __launch_bounds__(256)
    k_dist_claim(const unsigned long long* __restrict__ recv, int64_t nrecv, int P,
                 uint32_t* __restrict__ visited, int32_t* __restrict__ labels,
                 int32_t* __restrict__ preds, int32_t depth, int32_t* __restrict__ next_q,
                 unsigned long long* __restrict__ next_len) {
  const int lane = threadIdx.x & 31;
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < nrecv;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = base + threadIdx.x;
    bool won = false;
    int32_t l = 0;
    if (i < nrecv) {
      const unsigned long long x = recv[i];
      const int32_t d = (int32_t)(x >> 32), s = (int32_t)(uint32_t)x;
      l = d / P;
      const uint32_t bit = 1u << (l & 31);
      if (!(atomicOr(&visited[l >> 5], bit) & bit)) {
        won = true;
        labels[l] = depth;
        preds[l] = s;
      }
    }
    const unsigned wm = __ballot_sync(0xffffffffu, won);
    unsigned long long b = 0;
    if (lane == 0 && wm) b = atomicAdd(next_len, (unsigned long long)__popc(wm));
    b = __shfl_sync(0xffffffffu, b, 0);
    if (won) next_q[b + __popc(wm & ((1u << lane) - 1))] = l;
  }
}

// frontier membership against the all-gathered per-rank local bitmaps
struct GatheredFront {
  const uint32_t* g;
  int64_t wmax;
  int P;
  __device__ __forceinline__ uint32_t word(int32_t s) const {
    return g[(int64_t)(s % P) * wmax + ((s / P) >> 5)];
  }
  __device__ __forceinline__ bool bit(uint32_t w, int32_t s) const {
    return (w >> ((s / P) & 31)) & 1u;
  }
};

__global__ void __launch_bounds__(256)
    k_dist_pull(int64_t words, const uint32_t* __restrict__ nz, uint32_t* __restrict__ visited,
                GatheredFront front, uint32_t* __restrict__ next, const int32_t* __restrict__ head,
                const int64_t* __restrict__ lrow, const int32_t* __restrict__ lcol,
                int32_t* __restrict__ labels, int32_t* __restrict__ preds, int32_t depth,
                Counters* __restrict__ ctr) {
  __shared__ PullSmem ps[8];
  pull_groups(words, nz, visited, front, next, head, lrow, lcol, 0, LabelOut{labels, nullptr}, preds, depth, ctr,
              (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5,
              ((int64_t)gridDim.x * blockDim.x) >> 5, ps[threadIdx.x >> 5]);
}

__global__ void k_dist_seed(int64_t l, int32_t* labels, uint32_t* visited, int32_t* order) {
  labels[l] = 0;
  visited[l >> 5] |= 1u << (l & 31);
  order[0] = (int32_t)l;
}

__global__ void k_first_neighbour(const int64_t* __restrict__ row, const int32_t* __restrict__ col,
                                  int64_t n, int32_t* __restrict__ head) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = row[v];
    head[v] = row[v + 1] > b ? col[b] : -1;
  }
}

// bitmap<->queue conversions over LOCAL ids (same as the single-GPU ones)
__global__ void __launch_bounds__(256)
    k_dist_bm2q(int64_t words, const uint32_t* __restrict__ bm, int32_t* __restrict__ out,
                unsigned long long* __restrict__ out_len) {
  const int lane = threadIdx.x & 31;
  for (int64_t grp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; grp * 32 < words;
       grp += ((int64_t)gridDim.x * blockDim.x) >> 5) {
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

__global__ void k_dist_q2bm(const int32_t* __restrict__ F, int64_t nf, uint32_t* __restrict__ bm) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nf;
       i += (int64_t)gridDim.x * blockDim.x)
    atomicOr(&bm[F[i] >> 5], 1u << (F[i] & 31));
}

}  // namespace gfx

using namespace gfx;

static int db_scratch_i32(gfx_dbfs* db, const char* name, size_t count, int32_t** out) {
  return scratch_t(db->lg, name, count, out);
}

extern "C" {

int gfx_dist_partition_sizes(gfx_graph* g, int P, int r, int64_t* n_local, int64_t* m_local) {
  GFX_REQUIRE(g && n_local && m_local, "gfx_dist_partition_sizes: null argument");
  GFX_REQUIRE(P >= 1 && P <= 64 && r >= 0 && r < P, "bad partition P=%d r=%d", P, r);
  gfx_ctx* ctx = g->ctx;
  GFX_CK(cudaSetDevice(ctx->device));
  const int64_t nl = g->n > r ? (g->n - r + P - 1) / P : 0;
  int64_t* deg = nullptr;
  GFX_TRY(scratch_t(g, "part_deg", nl + 1, &deg));
  GFX_LAUNCH(k_part_degrees, grid_for(nl, 256, ctx->sm_count * 8), 256, 0, ctx->stream, g->row,
             g->n, P, r, nl, deg);
  GFX_CK(cudaMemsetAsync(deg + nl, 0, 8, ctx->stream));
  int64_t* off = nullptr;
  GFX_TRY(scratch_t(g, "part_off", nl + 1, &off));
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, deg, off, nl + 1, ctx->stream);
  void* tmp = nullptr;
  GFX_TRY(scratch(g, "part_tmp", tb, &tmp));
  cub::DeviceScan::ExclusiveSum(tmp, tb, deg, off, nl + 1, ctx->stream);
  int64_t ml = 0;
  GFX_CK(cudaMemcpyAsync(&ml, off + nl, 8, cudaMemcpyDeviceToHost, ctx->stream));
  GFX_CK(cudaStreamSynchronize(ctx->stream));
  *n_local = nl;
  *m_local = ml;
  return GFX_OK;
}

int gfx_dist_partition(gfx_graph* g, int P, int r, int64_t* lrow_d, int32_t* lcol_d) {
  GFX_REQUIRE(g && lrow_d, "gfx_dist_partition: null argument");
  int64_t nl = 0, ml = 0;
  GFX_TRY(gfx_dist_partition_sizes(g, P, r, &nl, &ml));
  gfx_ctx* ctx = g->ctx;
  const int64_t* off = static_cast<const int64_t*>(g->scratch["part_off"].ptr);
  GFX_CK(cudaMemcpyAsync(lrow_d, off, (nl + 1) * 8, cudaMemcpyDeviceToDevice, ctx->stream));
  if (ml > 0)
    GFX_LAUNCH(k_part_copy, grid_for(nl * 32, 256, ctx->sm_count * 16), 256, 0, ctx->stream,
               g->row, g->col, P, r, nl, lrow_d, lcol_d);
  GFX_CK(cudaGetLastError());
  GFX_CK(cudaStreamSynchronize(ctx->stream));
  return GFX_OK;
}

int gfx_dbfs_create(gfx_ctx* ctx, int64_t n, int64_t m, int P, int r, const int64_t* lrow_d,
                    const int32_t* lcol_d, int64_t n_local, int64_t m_local, gfx_dbfs** out) {
  GFX_REQUIRE(ctx && out && lrow_d, "gfx_dbfs_create: null argument");
  GFX_REQUIRE(P >= 1 && P <= 64 && r >= 0 && r < P, "bad partition P=%d r=%d", P, r);
  GFX_REQUIRE(n_local == (n > r ? (n - r + P - 1) / P : 0), "n_local does not match the partition");
  gfx_graph* lg = nullptr;
  GFX_TRY(gfx_graph_create(ctx, n_local, m_local, lrow_d, lcol_d, nullptr, GFX_GRAPH_UNDIRECTED,
                           &lg));
  auto* db = new gfx_dbfs();
  db->ctx = ctx;
  db->lg = lg;
  db->P = P;
  db->r = r;
  db->n = n;
  db->m = m;
  db->nl = n_local;
  db->ml = m_local;
  db->wl = (n_local + 31) / 32;
  const int64_t nmax = (n + P - 1) / P;
  db->wmax = (nmax + 31) / 32;
  *out = db;
  return GFX_OK;
}

int gfx_dbfs_destroy(gfx_dbfs* db) {
  if (!db) return GFX_OK;
  gfx_graph_destroy(db->lg);
  delete db;
  return GFX_OK;
}

int gfx_dbfs_words(gfx_dbfs* db, int64_t* words_local, int64_t* words_max) {
  GFX_REQUIRE(db && words_local && words_max, "gfx_dbfs_words: null argument");
  *words_local = db->wl;
  *words_max = db->wmax;
  return GFX_OK;
}

int gfx_dbfs_bind(gfx_dbfs* db, int32_t* labels_d, int32_t* preds_d, void* send_d,
                  int64_t send_cap, void* recv_d, int64_t recv_cap, uint32_t* front_local_d,
                  uint32_t* gathered_d) {
  GFX_REQUIRE(db && labels_d && preds_d && send_d && recv_d && front_local_d && gathered_d,
              "gfx_dbfs_bind: null argument");
  db->labels = labels_d;
  db->preds = preds_d;
  db->send = static_cast<unsigned long long*>(send_d);
  db->recv = static_cast<unsigned long long*>(recv_d);
  db->send_cap = send_cap;
  db->recv_cap = recv_cap;
  db->front_local = front_local_d;
  db->gathered = gathered_d;
  return GFX_OK;
}

int gfx_dbfs_reset(gfx_dbfs* db, int64_t source, int64_t* nf_local) {
  GFX_REQUIRE(db && nf_local && db->labels, "gfx_dbfs_reset: unbound engine");
  GFX_REQUIRE(source >= 0 && source < db->n, "source %lld out of range", (long long)source);
  gfx_graph* g = db->lg;
  gfx_ctx* ctx = db->ctx;
  GFX_CK(cudaSetDevice(ctx->device));
  uint32_t *visited, *sent;
  int32_t *order, *head, *sent_src;
  GFX_TRY(scratch_t(g, "d_visited", db->wl + 1, &visited));
  GFX_TRY(scratch_t(g, "d_sent", (db->n + 31) / 32 + 1, &sent));
  GFX_TRY(db_scratch_i32(db, "d_sent_src", db->n + 1, &sent_src));
  GFX_TRY(db_scratch_i32(db, "q_order", db->nl + 1, &order));
  {
    bool fresh = false;
    void* p = nullptr;
    GFX_TRY(scratch(g, "keep_dhead", (size_t)(db->nl + 1) * 4, &p, &fresh));
    head = static_cast<int32_t*>(p);
    if (fresh && db->nl > 0)
      GFX_LAUNCH(k_first_neighbour, grid_for(db->nl, 256, ctx->sm_count * 8), 256, 0, ctx->stream,
                 g->row, g->col, db->nl, head);
  }
  GFX_TRY(fill_i32(ctx, db->labels, GFX_UNVISITED, db->nl));
  GFX_CK(cudaMemsetAsync(db->preds, 0xFF, db->nl * 4, ctx->stream));
  GFX_CK(cudaMemsetAsync(visited, 0, (db->wl + 1) * 4, ctx->stream));
  GFX_CK(cudaMemsetAsync(sent, 0, ((db->n + 31) / 32 + 1) * 4, ctx->stream));
  db->q_off = 0;
  db->q_end = 0;
  db->nf = 0;
  db->queue_form = true;
  if (source % db->P == db->r) {
    GFX_LAUNCH(k_dist_seed, 1, 1, 0, ctx->stream, source / db->P, db->labels, visited, order);
    db->nf = 1;
    db->q_end = 1;
  }
  GFX_CK(cudaStreamSynchronize(ctx->stream));
  *nf_local = db->nf;
  return GFX_OK;
}

// push: expand the local frontier; returns per-destination-rank pair counts
// (host array of P) and the number of owned vertices claimed locally
int gfx_dbfs_push_expand(gfx_dbfs* db, int32_t depth, int64_t* send_counts, int64_t* local_new,
                         int64_t* edges) {
  GFX_REQUIRE(db && send_counts && local_new && edges, "gfx_dbfs_push_expand: null argument");
  gfx_graph* g = db->lg;
  gfx_ctx* ctx = db->ctx;
  GFX_CK(cudaSetDevice(ctx->device));
  uint32_t* visited = static_cast<uint32_t*>(g->scratch["d_visited"].ptr);
  uint32_t* sent = static_cast<uint32_t*>(g->scratch["d_sent"].ptr);
  int32_t* sent_src = static_cast<int32_t*>(g->scratch["d_sent_src"].ptr);
  int32_t* order = static_cast<int32_t*>(g->scratch["q_order"].ptr);
  int32_t *emit, *part;
  int64_t *scan, *rowbase;
  GFX_TRY(db_scratch_i32(db, "d_emit", db->n + 1, &emit));
  GFX_TRY(scratch_t(g, "q_scan", db->nl + 2, &scan));
  GFX_TRY(scratch_t(g, "q_rowbase", db->nl + 1, &rowbase));
  GFX_TRY(scratch_t(g, "q_part", part_capacity(db->ml, db->nl), &part));
  Counters* C = g->counters;
  auto* pin = static_cast<Counters*>(ctx->pinned);
  GFX_CK(cudaMemsetAsync(C, 0, 3 * sizeof(Counters), ctx->stream));
  if (!db->queue_form) {
    GFX_LAUNCH(k_dist_bm2q, grid_for(db->wl * 32, 256, ctx->sm_count * 8), 256, 0, ctx->stream,
               db->wl, db->front_local, order + db->q_end, &C[2].aux0);
    db->q_off = db->q_end;
    db->q_end += db->nf;
    db->queue_form = true;
  }
  const unsigned long long nf = (unsigned long long)db->nf;
  GFX_CK(cudaMemcpyAsync(&C[0].out_len, &nf, 8, cudaMemcpyHostToDevice, ctx->stream));
  DistClaimOp op{visited, sent, sent_src, db->labels, db->preds, depth, db->P, db->r, {}};
  GFX_TRY(lb_advance(g, order + db->q_off, &C[0].out_len, db->nf, &C[1], scan, rowbase, part, op,
                     emit, &C[1].out_len));
  // pass 0: per-owner counts
  unsigned long long* cnt64 = nullptr;
  GFX_TRY(scratch_t(g, "d_counts", 2 * 64, &cnt64));
  GFX_CK(cudaMemsetAsync(cnt64, 0, 2 * 64 * 8, ctx->stream));
  const int grid = ctx->sm_count * 4;
  GFX_LAUNCH((k_dist_bucket<0>), grid, 256, 0, ctx->stream, emit, &C[1].out_len, db->P, db->r,
             cnt64, nullptr, sent_src, sent, db->send, nullptr, nullptr);
  std::vector<unsigned long long> hc(db->P);
  GFX_CK(cudaMemcpyAsync(hc.data(), cnt64, db->P * 8, cudaMemcpyDeviceToHost, ctx->stream));
  GFX_CK(cudaMemcpyAsync(pin, C, 2 * sizeof(Counters), cudaMemcpyDeviceToHost, ctx->stream));
  GFX_CK(cudaStreamSynchronize(ctx->stream));
  const int64_t total_slots = (int64_t)pin[1].total;
  // cursors = exclusive scan over remote owners (own bucket excluded)
  std::vector<unsigned long long> cur(db->P, 0);
  unsigned long long acc = 0;
  for (int o = 0; o < db->P; ++o) {
    cur[o] = acc;
    send_counts[o] = (o == db->r) ? 0 : (int64_t)hc[o];
    if (o != db->r) acc += hc[o];
  }
  GFX_REQUIRE((int64_t)acc <= db->send_cap, "send buffer too small (%llu > %lld)",
              (unsigned long long)acc, (long long)db->send_cap);
  GFX_CK(cudaMemcpyAsync(cnt64 + 64, cur.data(), db->P * 8, cudaMemcpyHostToDevice, ctx->stream));
  GFX_CK(cudaMemsetAsync(&C[2].out_len, 0, 8, ctx->stream));
  GFX_LAUNCH((k_dist_bucket<1>), grid, 256, 0, ctx->stream, emit, &C[1].out_len, db->P, db->r,
             nullptr, cnt64 + 64, sent_src, sent, db->send, order + db->q_end, &C[2].out_len);
  GFX_CK(cudaGetLastError());
  GFX_CK(cudaStreamSynchronize(ctx->stream));
  db->local_new = (int64_t)hc[db->r];
  *local_new = db->local_new;
  *edges = total_slots;
  return GFX_OK;
}

int gfx_dbfs_push_claim(gfx_dbfs* db, int64_t nrecv, int32_t depth, int64_t* nf_local) {
  GFX_REQUIRE(db && nf_local, "gfx_dbfs_push_claim: null argument");
  GFX_REQUIRE(nrecv >= 0 && nrecv <= db->recv_cap, "received %lld pairs, capacity %lld",
              (long long)nrecv, (long long)db->recv_cap);
  gfx_graph* g = db->lg;
  gfx_ctx* ctx = db->ctx;
  GFX_CK(cudaSetDevice(ctx->device));
  uint32_t* visited = static_cast<uint32_t*>(g->scratch["d_visited"].ptr);
  int32_t* order = static_cast<int32_t*>(g->scratch["q_order"].ptr);
  Counters* C = g->counters;
  auto* pin = static_cast<Counters*>(ctx->pinned);
  const unsigned long long ln = (unsigned long long)db->local_new;
  GFX_CK(cudaMemcpyAsync(&C[2].out_len, &ln, 8, cudaMemcpyHostToDevice, ctx->stream));
  if (nrecv > 0)
    GFX_LAUNCH(k_dist_claim, grid_for(nrecv, 256, ctx->sm_count * 8), 256, 0, ctx->stream,
               db->recv, nrecv, db->P, visited, db->labels, db->preds, depth, order + db->q_end,
               &C[2].out_len);
  GFX_CK(cudaMemcpyAsync(pin, &C[2], sizeof(Counters), cudaMemcpyDeviceToHost, ctx->stream));
  GFX_CK(cudaStreamSynchronize(ctx->stream));
  db->nf = (int64_t)pin->out_len;
  db->q_off = db->q_end;
  db->q_end += db->nf;
  db->queue_form = true;
  *nf_local = db->nf;
  return GFX_OK;
}

// pull, step 1: local frontier as a bitmap in the host-bound front_local
int gfx_dbfs_pull_prepare(gfx_dbfs* db) {
  GFX_REQUIRE(db, "gfx_dbfs_pull_prepare: null engine");
  gfx_graph* g = db->lg;
  gfx_ctx* ctx = db->ctx;
  GFX_CK(cudaSetDevice(ctx->device));
  if (db->queue_form) {
    int32_t* order = static_cast<int32_t*>(g->scratch["q_order"].ptr);
    GFX_CK(cudaMemsetAsync(db->front_local, 0, db->wmax * 4, ctx->stream));
    if (db->nf > 0)
      GFX_LAUNCH(k_dist_q2bm, grid_for(db->nf, 256, ctx->sm_count * 8), 256, 0, ctx->stream,
                 order + db->q_off, db->nf, db->front_local);
    db->queue_form = false;
  }
  GFX_CK(cudaStreamSynchronize(ctx->stream));
  return GFX_OK;
}

// pull, step 2 (after the host all-gathered front_local into gathered)
int gfx_dbfs_pull(gfx_dbfs* db, int32_t depth, int64_t* nf_local, int64_t* probes,
                  int64_t* candidates) {
  GFX_REQUIRE(db && nf_local && probes && candidates, "gfx_dbfs_pull: null argument");
  gfx_graph* g = db->lg;
  gfx_ctx* ctx = db->ctx;
  GFX_CK(cudaSetDevice(ctx->device));
  uint32_t* visited = static_cast<uint32_t*>(g->scratch["d_visited"].ptr);
  int32_t* head = static_cast<int32_t*>(g->scratch["keep_dhead"].ptr);
  void* nzp = nullptr;
  GFX_TRY(scratch(g, "nz_out", db->wl * 4, &nzp));
  uint32_t* next = nullptr;
  GFX_TRY(scratch_t(g, "d_next", db->wmax + 1, &next));
  Counters* C = g->counters;
  auto* pin = static_cast<Counters*>(ctx->pinned);
  GFX_CK(cudaMemsetAsync(C, 0, sizeof(Counters), ctx->stream));
  GatheredFront front{db->gathered, db->wmax, db->P};
  GFX_LAUNCH(k_dist_pull, ctx->sm_count * 8, 256, 0, ctx->stream, db->wl,
             static_cast<const uint32_t*>(nzp), visited, front, next, head, g->row, g->col,
             db->labels, db->preds, depth, C);
  // the new frontier becomes the local bitmap
  GFX_CK(cudaMemsetAsync(db->front_local, 0, db->wmax * 4, ctx->stream));
  GFX_CK(cudaMemcpyAsync(db->front_local, next, db->wl * 4, cudaMemcpyDeviceToDevice,
                         ctx->stream));
  GFX_CK(cudaMemcpyAsync(pin, C, sizeof(Counters), cudaMemcpyDeviceToHost, ctx->stream));
  GFX_CK(cudaStreamSynchronize(ctx->stream));
  db->nf = (int64_t)pin->out_len;
  db->queue_form = false;
  *nf_local = db->nf;
  *probes = (int64_t)pin->aux0;
  *candidates = (int64_t)pin->aux1;
  return GFX_OK;
}

}  // extern "C"
