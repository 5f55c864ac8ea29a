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
#include <dlfcn.h>

#include <cmath>
#include <cstring>

#include <vector>

#include "gfx_device.cuh"
#include "gfx_direction.cuh"
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
  int64_t* send_counts = nullptr;   // P: pairs per destination rank
  int64_t* stats = nullptr;         // 4: new frontier, slots, probes, candidates
  int64_t send_cap = 0, recv_cap = 0;
  // engine state (host mirror; nf arrives through gfx_dbfs_commit)
  int64_t nf = 0, q_off = 0, q_end = 0;
  bool queue_form = true;
  bool pending_push = false;  // the level in flight appends to the queue
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
  int sh;  // log2(P) when P is a power of two, else -1
  uint32_t wv[kBatch];
  __device__ __forceinline__ int owner(int32_t d) const { return sh >= 0 ? (d & (P - 1)) : d % P; }
  __device__ __forceinline__ int32_t local(int32_t d) const { return sh >= 0 ? (d >> sh) : d / P; }
  __device__ int32_t src_value(int32_t) const { return 0; }
  __device__ void prefetch(const int32_t* d) {
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      if (d[u] < 0) {
        wv[u] = 0xffffffffu;
      } else if (owner(d[u]) == r) {
        const int32_t l = local(d[u]);
        wv[u] = visited[l >> 5];
      } else {
        wv[u] = sent[d[u] >> 5];
      }
    }
  }
  __device__ bool visit(int u, int32_t d, int32_t s, int32_t, int32_t, int64_t) {
    const int32_t sg = s * P + r;  // frontier items are local ids
    if (owner(d) == r) {
      const int32_t l = local(d);
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
  const int lane = threadIdx.x & 31;
  const int64_t n = (int64_t)*n_d;
  if (PASS == 0) {
    for (int i = threadIdx.x; i < P; i += blockDim.x) hist[i] = 0;
    __syncthreads();
  }
  // warp-uniform trip count so the match / shuffle below see full warps
  for (int64_t base = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) & ~31ll; base < n;
       base += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = base + lane;
    const bool ok = i < n;
    const int32_t d = ok ? emit[i] : 0;
    const int o = ok ? d % P : 64;  // 64: idle lanes form their own group
    const unsigned peers = __match_any_sync(0xffffffffu, o);
    const int leader = __ffs(peers) - 1;
    const int rank_in = __popc(peers & ((1u << lane) - 1));
    if (PASS == 0) {
      if (ok && lane == leader) atomicAdd(&hist[o], (unsigned long long)__popc(peers));
    } else {
      unsigned long long at = 0;
      if (ok && lane == leader)
        at = atomicAdd(o == r ? next_len : &cursors[o], (unsigned long long)__popc(peers));
      at = __shfl_sync(0xffffffffu, at, leader) + rank_in;
      if (ok) {
        if (o == r) {
          next_q[at] = d / P;
        } else {
          send[at] = ((unsigned long long)(uint32_t)d << 32) | (uint32_t)sent_src[d];
          atomicAnd(&sent[d >> 5], ~(1u << (d & 31)));
        }
      }
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
// (P a power of two -- 1, 2, 4, 8 GPUs -- replaces the divisions by shifts)
struct GatheredFront {
  const uint32_t* g;
  int64_t wmax;
  int P;
  int sh;  // log2(P) when P is a power of two, else -1
  __device__ __forceinline__ uint32_t word(int32_t s) const {
    if (sh >= 0) return g[(int64_t)(s & (P - 1)) * wmax + ((s >> sh) >> 5)];
    return g[(int64_t)(s % P) * wmax + ((s / P) >> 5)];
  }
  __device__ __forceinline__ bool bit(uint32_t w, int32_t s) const {
    return (w >> (((sh >= 0) ? (s >> sh) : (s / P)) & 31)) & 1u;
  }
};

static int pow2_shift(int P) {
  if (P <= 0 || (P & (P - 1))) return -1;
  int sh = 0;
  while ((1 << sh) < P) ++sh;
  return sh;
}

__global__ void __launch_bounds__(256)
    k_dist_pull(int64_t words, const uint32_t* __restrict__ nz, uint32_t* __restrict__ visited,
                GatheredFront front, uint32_t* __restrict__ next, const int32_t* __restrict__ head,
                const int64_t* __restrict__ lrow, const int32_t* __restrict__ lcol,
                int32_t* __restrict__ labels, int32_t* __restrict__ preds, int32_t depth,
                Counters* __restrict__ ctr, const int32_t* __restrict__ head2) {
  __shared__ PullSmem ps[8];
  pull_groups(words, nz, visited, front, next, head, lrow, lcol, 0, LabelOut{labels, nullptr},
              preds, depth, ctr, (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5,
              ((int64_t)gridDim.x * blockDim.x) >> 5, ps[threadIdx.x >> 5], head2);
}

__global__ void k_dist_seed(int64_t l, int32_t* labels, uint32_t* visited, int32_t* order) {
  labels[l] = 0;
  visited[l >> 5] |= 1u << (l & 31);
  order[0] = (int32_t)l;
}

// first two neighbours of every owned row, bit 31 flagging "degree is
// exactly 1 / 2" (the single-GPU pull's head / head2 arrays)
__global__ void k_dist_heads(const int64_t* __restrict__ row, const int32_t* __restrict__ col,
                             int64_t n, int32_t* __restrict__ head, int32_t* __restrict__ head2) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = row[v], d = row[v + 1] - b;
    head[v] = d > 0 ? (int32_t)((uint32_t)col[b] | (d == 1 ? 0x80000000u : 0u)) : -1;
    head2[v] = d > 1 ? (int32_t)((uint32_t)col[b + 1] | (d == 2 ? 0x80000000u : 0u)) : -1;
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

// remote-owner cursors (exclusive scan, own bucket excluded) and the
// host-visible per-destination counts; clears the owned-append counter
__global__ void k_dist_cursors(int P, int r, const unsigned long long* __restrict__ hist,
                               unsigned long long* __restrict__ cursors,
                               int64_t* __restrict__ send_counts,
                               unsigned long long* __restrict__ next_len) {
  if (threadIdx.x != 0) return;
  unsigned long long acc = 0;
  for (int o = 0; o < P; ++o) {
    cursors[o] = acc;
    const unsigned long long c = o == r ? 0ull : hist[o];
    send_counts[o] = (int64_t)c;
    acc += c;
  }
  *next_len = 0;
}

// zero the three level counters and seed the frontier length
__global__ void k_dist_level_init(Counters* C, unsigned long long nf) {
  unsigned long long* w = reinterpret_cast<unsigned long long*>(C);
  for (int i = threadIdx.x; i < 3 * (int)(sizeof(Counters) / 8); i += blockDim.x) w[i] = 0;
  __syncthreads();
  if (threadIdx.x == 0) C[0].out_len = nf;
}

// level counters -> the host-bound stats array, twice: st[0..3] stay this
// rank's, st[4..7] are the copy the host allreduces in place
__global__ void k_dist_stats(const Counters* __restrict__ C, int which, int64_t* __restrict__ st) {
  if (threadIdx.x != 0) return;
  int64_t v[4];
  if (which == 0) {  // push: new frontier = owned claims + received claims; slots
    v[0] = (int64_t)C[2].out_len;
    v[1] = (int64_t)C[1].total;
    v[2] = 0;
    v[3] = 0;
  } else {  // pull
    v[0] = (int64_t)C[0].out_len;
    v[1] = 0;
    v[2] = (int64_t)C[0].aux0;
    v[3] = (int64_t)C[0].aux1;
  }
  for (int k = 0; k < 4; ++k) st[k] = st[4 + k] = v[k];
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
                  uint32_t* gathered_d, int64_t* send_counts_d, int64_t* stats_d) {
  GFX_REQUIRE(db && labels_d && preds_d && send_d && recv_d && front_local_d && gathered_d &&
                  send_counts_d && stats_d,
              "gfx_dbfs_bind: null argument");
  GFX_REQUIRE(send_cap >= db->n && recv_cap >= db->n,
              "exchange buffers need n pairs (send %lld, recv %lld, n %lld)", (long long)send_cap,
              (long long)recv_cap, (long long)db->n);
  db->labels = labels_d;
  db->preds = preds_d;
  db->send = static_cast<unsigned long long*>(send_d);
  db->recv = static_cast<unsigned long long*>(recv_d);
  db->send_cap = send_cap;
  db->recv_cap = recv_cap;
  db->front_local = front_local_d;
  db->gathered = gathered_d;
  db->send_counts = send_counts_d;
  db->stats = stats_d;
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
    GFX_TRY(scratch(g, "keep_dhead", (size_t)(db->nl + 1) * 8, &p, &fresh));
    head = static_cast<int32_t*>(p);
    if (fresh && db->nl > 0)
      GFX_LAUNCH(k_dist_heads, grid_for(db->nl, 256, ctx->sm_count * 8), 256, 0, ctx->stream,
                 g->row, g->col, db->nl, head, head + db->nl + 1);
  }
  GFX_TRY(fill_i32(ctx, db->labels, GFX_UNVISITED, db->nl));
  GFX_CK(cudaMemsetAsync(db->preds, 0xFF, db->nl * 4, ctx->stream));
  GFX_CK(cudaMemsetAsync(visited, 0, (db->wl + 1) * 4, ctx->stream));
  GFX_CK(cudaMemsetAsync(sent, 0, ((db->n + 31) / 32 + 1) * 4, ctx->stream));
  db->q_off = 0;
  db->q_end = 0;
  db->nf = 0;
  db->queue_form = true;
  db->pending_push = false;
  if (source % db->P == db->r) {
    GFX_LAUNCH(k_dist_seed, 1, 1, 0, ctx->stream, source / db->P, db->labels, visited, order);
    db->nf = 1;
    db->q_end = 1;
  }
  GFX_CK(cudaGetLastError());
  *nf_local = db->nf;
  return GFX_OK;
}

// push: expand the local frontier, claim owned targets, bucket remote pairs
int gfx_dbfs_push_expand(gfx_dbfs* db, int32_t depth) {
  GFX_REQUIRE(db && db->stats, "gfx_dbfs_push_expand: unbound engine");
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
  unsigned long long* cnt64 = nullptr;
  GFX_TRY(scratch_t(g, "d_counts", 2 * 64, &cnt64));
  Counters* C = g->counters;
  GFX_LAUNCH(k_dist_level_init, 1, 32, 0, ctx->stream, C, (unsigned long long)db->nf);
  if (!db->queue_form) {
    GFX_LAUNCH(k_dist_bm2q, grid_for(db->wl * 32, 256, ctx->sm_count * 8), 256, 0, ctx->stream,
               db->wl, db->front_local, order + db->q_end, &C[2].aux0);
    db->q_off = db->q_end;
    db->q_end += db->nf;
    db->queue_form = true;
  }
  DistClaimOp op{visited, sent, sent_src, db->labels, db->preds, depth, db->P, db->r,
                 pow2_shift(db->P), {}};
  GFX_TRY(lb_advance(g, order + db->q_off, &C[0].out_len, db->nf, &C[1], scan, rowbase, part, op,
                     emit, &C[1].out_len));
  // pass 0: per-owner counts; cursors on the device; pass 1: scatter
  GFX_CK(cudaMemsetAsync(cnt64, 0, 64 * 8, ctx->stream));
  const int grid = ctx->sm_count * 4;
  GFX_LAUNCH((k_dist_bucket<0>), grid, 256, 0, ctx->stream, emit, &C[1].out_len, db->P, db->r,
             cnt64, nullptr, sent_src, sent, db->send, nullptr, nullptr);
  GFX_LAUNCH(k_dist_cursors, 1, 32, 0, ctx->stream, db->P, db->r, cnt64, cnt64 + 64,
             db->send_counts, &C[2].out_len);
  GFX_LAUNCH((k_dist_bucket<1>), grid, 256, 0, ctx->stream, emit, &C[1].out_len, db->P, db->r,
             nullptr, cnt64 + 64, sent_src, sent, db->send, order + db->q_end, &C[2].out_len);
  GFX_CK(cudaGetLastError());
  db->pending_push = true;
  return GFX_OK;
}

int gfx_dbfs_push_claim(gfx_dbfs* db, int64_t nrecv, int32_t depth) {
  GFX_REQUIRE(db && db->stats, "gfx_dbfs_push_claim: unbound engine");
  GFX_REQUIRE(nrecv >= 0 && nrecv <= db->recv_cap, "received %lld pairs, capacity %lld",
              (long long)nrecv, (long long)db->recv_cap);
  gfx_graph* g = db->lg;
  gfx_ctx* ctx = db->ctx;
  GFX_CK(cudaSetDevice(ctx->device));
  uint32_t* visited = static_cast<uint32_t*>(g->scratch["d_visited"].ptr);
  int32_t* order = static_cast<int32_t*>(g->scratch["q_order"].ptr);
  Counters* C = g->counters;
  if (nrecv > 0)
    GFX_LAUNCH(k_dist_claim, grid_for(nrecv, 256, ctx->sm_count * 8), 256, 0, ctx->stream,
               db->recv, nrecv, db->P, visited, db->labels, db->preds, depth, order + db->q_end,
               &C[2].out_len);
  GFX_LAUNCH(k_dist_stats, 1, 32, 0, ctx->stream, C, 0, db->stats);
  GFX_CK(cudaGetLastError());
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
  GFX_CK(cudaGetLastError());
  return GFX_OK;
}

// pull, step 2 (after the host all-gathered front_local into gathered)
int gfx_dbfs_pull(gfx_dbfs* db, int32_t depth) {
  GFX_REQUIRE(db && db->stats, "gfx_dbfs_pull: unbound engine");
  gfx_graph* g = db->lg;
  gfx_ctx* ctx = db->ctx;
  GFX_CK(cudaSetDevice(ctx->device));
  uint32_t* visited = static_cast<uint32_t*>(g->scratch["d_visited"].ptr);
  int32_t* head = static_cast<int32_t*>(g->scratch["keep_dhead"].ptr);
  void* nzp = nullptr;
  GFX_TRY(scratch(g, "nz_out", db->wl * 4, &nzp));
  Counters* C = g->counters;
  GFX_LAUNCH(k_dist_level_init, 1, 32, 0, ctx->stream, C, 0ull);
  // the new frontier is written straight into the local bitmap (the pull
  // reads only the gathered copy); words past wl stay zero
  GFX_CK(cudaMemsetAsync(db->front_local, 0, db->wmax * 4, ctx->stream));
  GatheredFront front{db->gathered, db->wmax, db->P, pow2_shift(db->P)};
  GFX_LAUNCH(k_dist_pull, ctx->sm_count * 8, 256, 0, ctx->stream, db->wl,
             static_cast<const uint32_t*>(nzp), visited, front, db->front_local, head, g->row,
             g->col, db->labels, db->preds, depth, C, head + db->nl + 1);
  GFX_LAUNCH(k_dist_stats, 1, 32, 0, ctx->stream, C, 1, db->stats);
  GFX_CK(cudaGetLastError());
  db->pending_push = false;
  return GFX_OK;
}

int gfx_dbfs_commit(gfx_dbfs* db, int64_t nf_local) {
  GFX_REQUIRE(db, "gfx_dbfs_commit: null engine");
  GFX_REQUIRE(nf_local >= 0 && nf_local <= db->nl, "frontier %lld out of range",
              (long long)nf_local);
  db->nf = nf_local;
  if (db->pending_push) {
    GFX_REQUIRE(db->q_end + nf_local <= db->nl + 1, "queue overflow");
    db->q_off = db->q_end;
    db->q_end += nf_local;
    db->queue_form = true;
  } else {
    db->queue_form = false;
  }
  db->pending_push = false;
  return GFX_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Native level loop: the same per-level protocol as
// dist.py:bfs_partitioned, driven from C++ with NCCL called directly on the
// context stream -- one host synchronisation per pull level (the allreduced
// level counters), two per push level (pair counts, then counters).  NCCL is
// the library torch already loaded in this process (resolved with dlopen /
// dlsym, so libgfx carries no link-time NCCL dependency and cannot pick up a
// second, different NCCL).
// ---------------------------------------------------------------------------
namespace {

struct NcclUid {
  char internal[128];
};
using nres_t = int;
constexpr int kNcclInt32 = 2, kNcclInt64 = 4, kNcclUint64 = 5, kNcclSum = 0;

struct NcclApi {
  void* lib = nullptr;
  nres_t (*GetUniqueId)(NcclUid*) = nullptr;
  nres_t (*CommInitRank)(void**, int, NcclUid, int) = nullptr;
  nres_t (*CommDestroy)(void*) = nullptr;
  nres_t (*AllReduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  nres_t (*AllGather)(const void*, void*, size_t, int, void*, cudaStream_t) = nullptr;
  nres_t (*Send)(const void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  nres_t (*Recv)(void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  nres_t (*GroupStart)() = nullptr;
  nres_t (*GroupEnd)() = nullptr;
  const char* (*ErrorString)(nres_t) = nullptr;
};
NcclApi g_nccl;

template <class F>
bool nccl_sym(F& f, const char* name) {
  f = reinterpret_cast<F>(dlsym(g_nccl.lib, name));
  return f != nullptr;
}

}  // namespace

struct gfx_nccl {
  void* comm = nullptr;
  int nranks = 1, rank = 0;
};

#define GFX_NCCL(call)                                                                        \
  do {                                                                                         \
    const nres_t rc_ = (call);                                                                 \
    GFX_REQUIRE(rc_ == 0, "NCCL error %d (%s) at %s:%d", rc_,                                  \
                g_nccl.ErrorString ? g_nccl.ErrorString(rc_) : "?", __FILE__, __LINE__);      \
  } while (0)

extern "C" {

int gfx_nccl_load(const char* path) {
  if (g_nccl.lib) return GFX_OK;
  void* h = nullptr;
  if (path && *path) h = dlopen(path, RTLD_NOW | RTLD_NOLOAD);
  if (!h && path && *path) h = dlopen(path, RTLD_NOW);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  GFX_REQUIRE(h, "gfx_nccl_load: NCCL is not loaded in this process (%s)",
              path ? path : "no path given");
  g_nccl.lib = h;
  bool ok = nccl_sym(g_nccl.GetUniqueId, "ncclGetUniqueId") &&
            nccl_sym(g_nccl.CommInitRank, "ncclCommInitRank") &&
            nccl_sym(g_nccl.CommDestroy, "ncclCommDestroy") &&
            nccl_sym(g_nccl.AllReduce, "ncclAllReduce") &&
            nccl_sym(g_nccl.AllGather, "ncclAllGather") && nccl_sym(g_nccl.Send, "ncclSend") &&
            nccl_sym(g_nccl.Recv, "ncclRecv") && nccl_sym(g_nccl.GroupStart, "ncclGroupStart") &&
            nccl_sym(g_nccl.GroupEnd, "ncclGroupEnd") &&
            nccl_sym(g_nccl.ErrorString, "ncclGetErrorString");
  if (!ok) {
    g_nccl = NcclApi{};
    GFX_REQUIRE(false, "gfx_nccl_load: NCCL symbols missing");
  }
  return GFX_OK;
}

int gfx_nccl_unique_id(uint8_t* id_out) {
  GFX_REQUIRE(id_out, "gfx_nccl_unique_id: null argument");
  GFX_REQUIRE(g_nccl.lib, "gfx_nccl_unique_id: call gfx_nccl_load first");
  NcclUid uid;
  GFX_NCCL(g_nccl.GetUniqueId(&uid));
  std::memcpy(id_out, uid.internal, sizeof(uid.internal));
  return GFX_OK;
}

int gfx_nccl_comm_create(gfx_ctx* ctx, int nranks, int rank, const uint8_t* id, gfx_nccl** out) {
  GFX_REQUIRE(ctx && id && out, "gfx_nccl_comm_create: null argument");
  GFX_REQUIRE(g_nccl.lib, "gfx_nccl_comm_create: call gfx_nccl_load first");
  GFX_REQUIRE(nranks >= 1 && nranks <= 64 && rank >= 0 && rank < nranks, "bad rank %d of %d",
              rank, nranks);
  GFX_CK(cudaSetDevice(ctx->device));
  NcclUid uid;
  std::memcpy(uid.internal, id, sizeof(uid.internal));
  auto* c = new gfx_nccl();
  c->nranks = nranks;
  c->rank = rank;
  const nres_t rc = g_nccl.CommInitRank(&c->comm, nranks, uid, rank);
  if (rc != 0) {
    delete c;
    GFX_NCCL(rc);
  }
  *out = c;
  return GFX_OK;
}

int gfx_nccl_comm_destroy(gfx_nccl* c) {
  if (!c) return GFX_OK;
  if (c->comm && g_nccl.CommDestroy) g_nccl.CommDestroy(c->comm);
  delete c;
  return GFX_OK;
}

}  // extern "C"

namespace {

// NCCL implementation of the collective table (user = NcclCtx)
struct NcclCtx {
  gfx_dbfs* db;
  void* comm;
};

int nccl_counts(void* user) {
  auto* c = static_cast<NcclCtx*>(user);
  gfx_dbfs* db = c->db;
  const int P = db->P;
  cudaStream_t st = db->ctx->stream;
  GFX_NCCL(g_nccl.GroupStart());
  for (int o = 0; o < P; ++o) {
    GFX_NCCL(g_nccl.Send(db->send_counts + o, 1, kNcclInt64, o, c->comm, st));
    GFX_NCCL(g_nccl.Recv(db->send_counts + P + o, 1, kNcclInt64, o, c->comm, st));
  }
  GFX_NCCL(g_nccl.GroupEnd());
  return GFX_OK;
}

int nccl_pairs(void* user, const int64_t* sc, const int64_t* rc) {
  auto* c = static_cast<NcclCtx*>(user);
  gfx_dbfs* db = c->db;
  cudaStream_t st = db->ctx->stream;
  int64_t so = 0, ro = 0;
  GFX_NCCL(g_nccl.GroupStart());
  for (int o = 0; o < db->P; ++o) {
    if (o != db->r) {
      if (sc[o]) GFX_NCCL(g_nccl.Send(db->send + so, sc[o], kNcclUint64, o, c->comm, st));
      if (rc[o]) GFX_NCCL(g_nccl.Recv(db->recv + ro, rc[o], kNcclUint64, o, c->comm, st));
    }
    so += sc[o];
    ro += rc[o];
  }
  GFX_NCCL(g_nccl.GroupEnd());
  return GFX_OK;
}

int nccl_gather(void* user) {
  auto* c = static_cast<NcclCtx*>(user);
  gfx_dbfs* db = c->db;
  GFX_NCCL(g_nccl.AllGather(db->front_local, db->gathered, (size_t)db->wmax, kNcclInt32, c->comm,
                            db->ctx->stream));
  return GFX_OK;
}

int nccl_reduce(void* user) {
  auto* c = static_cast<NcclCtx*>(user);
  gfx_dbfs* db = c->db;
  GFX_NCCL(g_nccl.AllReduce(db->stats + 4, db->stats + 4, 4, kNcclInt64, kNcclSum, c->comm,
                            db->ctx->stream));
  return GFX_OK;
}

}  // namespace

extern "C" {

int gfx_dbfs_run_comm(gfx_dbfs* db, const gfx_dbfs_comm* comm, int64_t source, int direction,
                      double do_a, double do_b, int mu_edge_based, gfx_iter_rec* recs,
                      int64_t rec_cap, gfx_stats* stats) {
  GFX_NVTX("gfx_dbfs_run_comm");
  GFX_REQUIRE(db && stats && db->stats, "gfx_dbfs_run: unbound engine");
  GFX_REQUIRE(direction == GFX_DIR_PUSH || direction == GFX_DIR_PULL || direction == GFX_DIR_AUTO,
              "bad direction %d", direction);
  GFX_REQUIRE(do_a > 0 && do_b > 0, "do_a and do_b must be positive");
  const int P = db->P;
  GFX_REQUIRE(P == 1 || (comm && comm->exchange_counts && comm->exchange_pairs &&
                         comm->allgather_frontier && comm->allreduce_stats),
              "gfx_dbfs_run: P = %d needs a collective table", P);
  gfx_ctx* ctx = db->ctx;
  cudaStream_t st = ctx->stream;
  auto* pin = static_cast<int64_t*>(ctx->pinned);  // 4 KB: 2P counts or 8 stats
  std::memset(stats, 0, sizeof(*stats));
  cudaEvent_t e0, e1;
  GFX_CK(cudaEventCreate(&e0));
  GFX_CK(cudaEventCreate(&e1));
  GFX_CK(cudaEventRecord(e0, st));
  int64_t nf_local = 0;
  GFX_TRY(gfx_dbfs_reset(db, source, &nf_local));
  int64_t nf = 1, n_u = db->n, depth = 0, nrec = 0;
  int mode = GFX_DIR_PUSH;
  std::vector<int64_t> sc(P), rc(P);
  while (nf > 0) {
    ++depth;
    n_u -= nf;
    const DirEstimate est = estimate_mf_mu(db->n, db->m, nf, n_u, mu_edge_based);
    int dec;
    if (direction == GFX_DIR_AUTO)
      dec = decide_direction(mode == GFX_DIR_PULL ? 1 : 0, est, do_a, do_b) ? GFX_DIR_PULL
                                                                            : GFX_DIR_PUSH;
    else if (direction == GFX_DIR_PULL)
      dec = depth > 1 ? GFX_DIR_PULL : GFX_DIR_PUSH;
    else
      dec = GFX_DIR_PUSH;
    int64_t edges = 0, work = 0;
    if (dec == GFX_DIR_PUSH) {
      GFX_TRY(gfx_dbfs_push_expand(db, (int32_t)depth));
      int64_t nrecv = 0;
      if (comm) {
        GFX_REQUIRE(comm->exchange_counts(comm->user) == 0, "exchange_counts failed");
        GFX_CK(cudaMemcpyAsync(pin, db->send_counts, 2 * P * 8, cudaMemcpyDeviceToHost, st));
        GFX_CK(cudaStreamSynchronize(st));
        for (int o = 0; o < P; ++o) {
          sc[o] = pin[o];
          rc[o] = pin[P + o];
          nrecv += rc[o];
        }
        GFX_REQUIRE(nrecv <= db->recv_cap, "received %lld pairs, capacity %lld",
                    (long long)nrecv, (long long)db->recv_cap);
        GFX_REQUIRE(comm->exchange_pairs(comm->user, sc.data(), rc.data()) == 0,
                    "exchange_pairs failed");
      }
      GFX_TRY(gfx_dbfs_push_claim(db, nrecv, (int32_t)depth));
    } else {
      GFX_TRY(gfx_dbfs_pull_prepare(db));
      if (comm)
        GFX_REQUIRE(comm->allgather_frontier(comm->user) == 0, "allgather_frontier failed");
      else
        GFX_CK(cudaMemcpyAsync(db->gathered, db->front_local, db->wmax * 4,
                               cudaMemcpyDeviceToDevice, st));
      GFX_TRY(gfx_dbfs_pull(db, (int32_t)depth));
    }
    if (comm) GFX_REQUIRE(comm->allreduce_stats(comm->user) == 0, "allreduce_stats failed");
    GFX_CK(cudaMemcpyAsync(pin, db->stats, 8 * 8, cudaMemcpyDeviceToHost, st));
    GFX_CK(cudaStreamSynchronize(st));
    const int64_t local_out = pin[0], nout = pin[4];
    if (dec == GFX_DIR_PUSH) {
      edges = pin[5];
      work = 20 * nf + 4 * edges;
      stats->edges_traversed += edges;
    } else {
      work = 12 * pin[7] + 4 * pin[6];
    }
    GFX_TRY(gfx_dbfs_commit(db, local_out));
    if (recs && nrec < rec_cap) {
      gfx_iter_rec& x = recs[nrec++];
      std::memset(&x, 0, sizeof(x));
      x.iteration = depth;
      x.frontier_in = nf;
      x.frontier_out = nout;
      x.n_u = n_u;
      x.edges = edges;
      x.m_f = est.m_f;
      x.m_u = est.m_u;
      x.mode_before = mode;
      x.decision = dec;
      x.candidates = dec == GFX_DIR_PULL ? pin[7] : 0;
      x.work = dec == GFX_DIR_PULL ? pin[6] : edges;
      x.bytes_alg = work + 8 * nout;
    }
    if (dec != mode) stats->direction_switches += 1;
    stats->bytes_alg += work + 8 * nout;
    mode = dec;
    nf = nout;
  }
  GFX_CK(cudaEventRecord(e1, st));
  GFX_CK(cudaEventSynchronize(e1));
  float ms = 0.f;
  GFX_CK(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  stats->iterations = depth;
  stats->device_ms = ms;
  stats->num_records = nrec;
  return GFX_OK;
}

int gfx_dbfs_run(gfx_dbfs* db, gfx_nccl* comm, int64_t source, int direction, double do_a,
                 double do_b, int mu_edge_based, gfx_iter_rec* recs, int64_t rec_cap,
                 gfx_stats* stats) {
  GFX_REQUIRE(db, "gfx_dbfs_run: null engine");
  // P = 1 without a communicator: the collectives are identities and are
  // skipped; with one (a 1-rank NCCL communicator) they run through NCCL
  if (db->P == 1 && !comm)
    return gfx_dbfs_run_comm(db, nullptr, source, direction, do_a, do_b, mu_edge_based, recs,
                             rec_cap, stats);
  GFX_REQUIRE(comm && comm->comm && comm->nranks == db->P && comm->rank == db->r,
              "gfx_dbfs_run: P = %d needs a communicator of P ranks with this rank", db->P);
  NcclCtx c{db, comm->comm};
  gfx_dbfs_comm ops{&c, nccl_counts, nccl_pairs, nccl_gather, nccl_reduce};
  return gfx_dbfs_run_comm(db, &ops, source, direction, do_a, do_b, mu_edge_based, recs, rec_cap,
                           stats);
}

}  // extern "C"
