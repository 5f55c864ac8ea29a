// Partitioned (multi-GPU) near/far SSSP: per-rank device engine.
//
// SURVEY 8(e) "SSSP: push exchange of (v, newdist) pairs with owner-side
// atomicMin; the near/far threshold is global and 'near empty' is decided by
// allreduce".  Reference algorithm: primitives/sssp.py:41-121 (relax =
// atomic_min + set_pred, each improved vertex enqueued once per iteration)
// and near_far.py:20-85 (split at the threshold, advance_bucket drops stale
// far entries and re-splits).
//
// Same 1D cyclic partition as the partitioned BFS (gfx_dist.cu): rank r owns
// v = l*P + r and keeps their rows with GLOBAL column ids and the weights.
// Per iteration, on every rank in lockstep:
//   relax : the local near queue is expanded (load-balanced warp tiles);
//           owned targets are relaxed in place -- one 64-bit atomicMin on
//           (dist << 32 | pred) -- and enqueued once (mark bit); a remote
//           target keeps its best offer this run in sent_key[d] (64-bit
//           atomicMin, monotone: an offer not below an earlier one is never
//           sent again) and is emitted once per iteration (sent bit);
//   bucket: emitted ids split into the touched list (owned) and per-owner
//           send buckets of (d, dist << 32 | pred) messages -- two 8-byte
//           words each -- with block-aggregated reservations;
//   (host exchanges counts, then messages: NCCL all_to_all)
//   apply : owners relax the received offers exactly like local ones;
//   split : touched -> near / far at the GLOBAL threshold (k_sssp_split);
//   stats : (near, far, slots, touched) for the host's allreduce; when the
//           global near count is 0 every rank advances the bucket
//           (threshold += delta, k_sssp_refar) in lockstep.
#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>

#include <cmath>
#include <utility>

#include "gfx_device.cuh"
#include "gfx_expand.cuh"
#include "gfx_internal.cuh"
#include "gfx_sssp.cuh"

struct gfx_dsssp {
  gfx_ctx* ctx = nullptr;
  gfx_graph* lg = nullptr;  // local CSR: owned rows, global column ids, weights
  int P = 1, r = 0, sh = -1;
  int64_t n = 0, nl = 0, ml = 0, wl = 0;
  unsigned long long* dp = nullptr;  // nl: dist << 32 | pred (global pred)
  uint32_t* dist = nullptr;          // nl: 32-bit mirror (probe array)
  uint32_t* mark = nullptr;          // wl + 1 words: enqueued this iteration
  unsigned long long* sent_key = nullptr;  // n: best offer sent per remote target this run
  uint32_t* sent = nullptr;          // n/32 + 1: emitted this iteration
  int32_t* nearq[2] = {nullptr, nullptr};
  int32_t *emit = nullptr, *touched = nullptr;
  int32_t *far = nullptr, *fkey = nullptr, *far2 = nullptr, *fkey2 = nullptr;
  int64_t *scan = nullptr, *rowbase = nullptr;
  int32_t* part = nullptr;
  gfx::Counters* C = nullptr;  // 0/1: near sizes, 2: expansion plan + emitted, 3: far, 4: touched
  unsigned long long* cursors = nullptr;  // 2 * 64: bucket cursors / counts
  // host-owned exchange buffers
  unsigned long long* send = nullptr;
  unsigned long long* recv = nullptr;
  int64_t send_cap = 0, recv_cap = 0;
  int64_t* send_counts = nullptr;  // P words per destination
  int64_t* stats = nullptr;        // 8: near, far, slots, touched | copy to allreduce
  int cur = 0;
};

namespace gfx {

__global__ void k_part_weights(const int64_t* __restrict__ row, const int32_t* __restrict__ w,
                               int P, int r, int64_t nl, const int64_t* __restrict__ lrow,
                               int32_t* __restrict__ lw) {
  const int lane = threadIdx.x & 31;
  for (int64_t l = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; l < nl;
       l += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t v = l * P + r;
    const int64_t b = row[v], e = row[v + 1], o = lrow[l];
    for (int64_t p = b + lane; p < e; p += 32) lw[o + (p - b)] = w[p];
  }
}

struct DistRelaxOp {
  static constexpr bool kWeights = true, kSrcVal = true, kEmitEdge = false;
  static constexpr int kBatch = 4;
  static constexpr int kMinBlocks = 3;
  unsigned long long* dp;
  uint32_t* dist;
  uint32_t* mark;
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
      else if (owner(d[u]) == r) cur[u] = dist[local(d[u])];
      else cur[u] = (uint32_t)(sent_key[d[u]] >> 32);
    }
  }
  __device__ bool visit(int u, int32_t d, int32_t s, int32_t w, int32_t sdist, int64_t) {
    const unsigned long long nd = (unsigned long long)(uint32_t)sdist + (uint32_t)w;
    if (nd >= cur[u]) return false;
    const unsigned long long key = (nd << 32) | (uint32_t)(s * P + r);
    if (owner(d) == r) {
      const int32_t l = local(d);
      atomicMin(&dp[l], key);
      atomicMin(&dist[l], (uint32_t)nd);
      const uint32_t bit = 1u << (l & 31);
      return !(atomicOr(&mark[l >> 5], bit) & bit);
    }
    atomicMin(&sent_key[d], key);
    const uint32_t bit = 1u << (d & 31);
    return !(atomicOr(&sent[d >> 5], bit) & bit);
  }
};

__device__ __forceinline__ int owner_of(int32_t d, int P, int sh) {
  return sh >= 0 ? (d & (P - 1)) : d % P;
}

// pass 0: count messages per owner (block histogram, one global atomic per
// owner and block).  pass 1: reserve per (block, owner) ranges behind the
// cursors, scatter (d, key) messages, append owned ids to `touched`, clear
// the sent bits.
template <int PASS>
__global__ void __launch_bounds__(256)
    k_dsssp_bucket(const int32_t* __restrict__ emit, const unsigned long long* __restrict__ n_d,
                   int P, int r, int sh, unsigned long long* __restrict__ counts,
                   unsigned long long* __restrict__ cursors,
                   const unsigned long long* __restrict__ sent_key, uint32_t* __restrict__ sent,
                   unsigned long long* __restrict__ send, int32_t* __restrict__ touched,
                   unsigned long long* __restrict__ touched_len) {
  __shared__ unsigned int hist[65];
  __shared__ unsigned long long base[65];
  const int64_t n = (int64_t)*n_d;
  for (int64_t b0 = blockIdx.x * (int64_t)blockDim.x; b0 < n;
       b0 += (int64_t)gridDim.x * blockDim.x) {
    for (int q = threadIdx.x; q <= P; q += blockDim.x) hist[q] = 0;
    __syncthreads();
    const int64_t i = b0 + threadIdx.x;
    int32_t d = -1;
    int slot = -1, pos = 0;
    if (i < n) {
      d = emit[i];
      const int q = owner_of(d, P, sh);
      slot = q == r ? P : q;  // slot P: owned (touched)
      pos = (int)atomicAdd(&hist[slot], 1u);
    }
    __syncthreads();
    if (PASS == 0) {
      for (int q = threadIdx.x; q < P; q += blockDim.x)
        if (q != r && hist[q]) atomicAdd(&counts[q], (unsigned long long)hist[q]);
    } else {
      for (int q = threadIdx.x; q <= P; q += blockDim.x) {
        if (!hist[q]) continue;
        base[q] = q == P ? atomicAdd(touched_len, (unsigned long long)hist[q])
                         : atomicAdd(&cursors[q], (unsigned long long)hist[q]);
      }
      __syncthreads();
      if (slot == P) {  // owned: local id
        touched[base[P] + pos] = sh >= 0 ? (d >> sh) : d / P;
      } else if (slot >= 0) {
        const unsigned long long at = base[slot] + pos;
        send[2 * at] = (unsigned long long)(uint32_t)d;
        send[2 * at + 1] = sent_key[d];
        atomicAnd(&sent[d >> 5], ~(1u << (d & 31)));
      }
    }
    __syncthreads();
  }
}

// exclusive scan of the P message counts -> cursors; counts in words
__global__ void k_dsssp_offsets(const unsigned long long* __restrict__ counts, int P,
                                unsigned long long* __restrict__ cursors,
                                int64_t* __restrict__ send_counts) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    unsigned long long acc = 0;
    for (int q = 0; q < P; ++q) {
      cursors[q] = acc;
      send_counts[q] = 2 * (int64_t)counts[q];
      acc += counts[q];
    }
  }
}

// owners relax received offers; improved vertices enqueued once
__global__ void k_dsssp_apply(const unsigned long long* __restrict__ recv, int64_t nmsg, int P,
                              int sh, unsigned long long* __restrict__ dp,
                              uint32_t* __restrict__ dist, uint32_t* __restrict__ mark,
                              int32_t* __restrict__ touched,
                              unsigned long long* __restrict__ touched_len) {
  const int lane = threadIdx.x & 31;
  for (int64_t b0 = (blockIdx.x * (int64_t)blockDim.x) ; b0 < nmsg;
       b0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = b0 + threadIdx.x;
    bool emit = false;
    int32_t l = 0;
    if (i < nmsg) {
      const int32_t d = (int32_t)recv[2 * i];
      const unsigned long long key = recv[2 * i + 1];
      l = sh >= 0 ? (d >> sh) : d / P;
      const uint32_t nd = (uint32_t)(key >> 32);
      if (nd < dist[l]) {
        atomicMin(&dp[l], key);
        atomicMin(&dist[l], nd);
        const uint32_t bit = 1u << (l & 31);
        emit = !(atomicOr(&mark[l >> 5], bit) & bit);
      }
    }
    const unsigned em = __ballot_sync(0xffffffffu, emit);
    if (em) {
      unsigned long long at = 0;
      if (lane == 0) at = atomicAdd(touched_len, (unsigned long long)__popc(em));
      at = __shfl_sync(0xffffffffu, at, 0);
      if (emit) touched[at + __popc(em & ((1u << lane) - 1))] = l;
    }
  }
}

__global__ void k_dsssp_seed(unsigned long long* dp, uint32_t* dist, int32_t l, int32_t src,
                             int32_t* near) {
  dp[l] = (unsigned long long)(uint32_t)-1;  // dist 0, pred -1
  dist[l] = 0u;
  near[0] = l;
  (void)src;
}

// level counters for the host allreduce: near (next), far, slots, touched
__global__ void k_dsssp_stats(const Counters* __restrict__ C, int nxt, int64_t* __restrict__ st) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    const int64_t v[4] = {(int64_t)C[nxt].out_len, (int64_t)C[3].aux0, (int64_t)C[2].total,
                          (int64_t)C[4].out_len};
    for (int k = 0; k < 4; ++k) st[k] = st[4 + k] = v[k];
  }
}

}  // namespace gfx

using namespace gfx;

extern "C" {

int gfx_dist_partition_weights(gfx_graph* g, int P, int r, const int64_t* lrow_d, int32_t* lw_d) {
  GFX_REQUIRE(g && lrow_d, "gfx_dist_partition_weights: null argument");
  GFX_REQUIRE(g->w, "the graph has no weights");
  GFX_REQUIRE(P >= 1 && P <= 64 && r >= 0 && r < P, "bad partition P=%d r=%d", P, r);
  gfx_ctx* ctx = g->ctx;
  GFX_CK(cudaSetDevice(ctx->device));
  const int64_t nl = g->n > r ? (g->n - r + P - 1) / P : 0;
  if (nl > 0)
    GFX_LAUNCH(k_part_weights, grid_for(nl * 32, 256, ctx->sm_count * 16), 256, 0, ctx->stream,
               g->row, g->w, P, r, nl, lrow_d, lw_d);
  GFX_CK(cudaGetLastError());
  GFX_CK(cudaStreamSynchronize(ctx->stream));
  return GFX_OK;
}

int gfx_dsssp_create(gfx_ctx* ctx, int64_t n, int P, int r, const int64_t* lrow_d,
                     const int32_t* lcol_d, const int32_t* lw_d, int64_t n_local,
                     int64_t m_local, gfx_dsssp** out) {
  GFX_REQUIRE(ctx && out && lrow_d && (m_local == 0 || (lcol_d && lw_d)),
              "gfx_dsssp_create: null argument");
  GFX_REQUIRE(P >= 1 && P <= 64 && r >= 0 && r < P, "bad partition P=%d r=%d", P, r);
  GFX_REQUIRE(n_local == (n > r ? (n - r + P - 1) / P : 0), "n_local does not match the partition");
  GFX_REQUIRE(n < (int64_t)INT32_MAX, "vertex ids must fit int32");
  GFX_CK(cudaSetDevice(ctx->device));
  gfx_graph* lg = nullptr;
  GFX_TRY(gfx_graph_create(ctx, n_local, m_local, lrow_d, lcol_d, lw_d, GFX_GRAPH_UNDIRECTED,
                           &lg));
  auto* ds = new gfx_dsssp();
  ds->ctx = ctx;
  ds->lg = lg;
  ds->P = P;
  ds->r = r;
  ds->sh = (P & (P - 1)) == 0 ? __builtin_ctz((unsigned)P) : -1;
  ds->n = n;
  ds->nl = n_local;
  ds->ml = m_local;
  ds->wl = (n_local + 31) / 32;
  const int64_t nl1 = n_local + 64;
  int st = GFX_OK;
  auto alloc = [&](void** p, size_t bytes) {
    if (st == GFX_OK && cudaMalloc(p, bytes) != cudaSuccess) {
      set_error("gfx_dsssp_create: out of device memory");
      st = GFX_ENOMEM;
    }
  };
  alloc((void**)&ds->dp, nl1 * 8);
  alloc((void**)&ds->dist, (nl1 + ds->wl + 1) * 4);
  alloc((void**)&ds->sent_key, (n + 1) * 8);
  alloc((void**)&ds->sent, ((n + 31) / 32 + 1) * 4);
  alloc((void**)&ds->nearq[0], nl1 * 4);
  alloc((void**)&ds->nearq[1], nl1 * 4);
  alloc((void**)&ds->touched, nl1 * 4);
  alloc((void**)&ds->emit, (n_local + m_local + 64) * 4);
  alloc((void**)&ds->far, (2 * nl1) * 4);
  alloc((void**)&ds->fkey, (2 * nl1) * 4);
  alloc((void**)&ds->far2, (2 * nl1) * 4);
  alloc((void**)&ds->fkey2, (2 * nl1) * 4);
  alloc((void**)&ds->scan, (nl1 + 2) * 8);
  alloc((void**)&ds->rowbase, nl1 * 8);
  alloc((void**)&ds->part, part_capacity(m_local, n_local) * 4);
  alloc((void**)&ds->C, 8 * sizeof(Counters));
  alloc((void**)&ds->cursors, 2 * 65 * 8);
  if (st != GFX_OK) {
    gfx_dsssp_destroy(ds);
    return st;
  }
  ds->mark = ds->dist + nl1;
  *out = ds;
  return GFX_OK;
}

int gfx_dsssp_destroy(gfx_dsssp* ds) {
  if (!ds) return GFX_OK;
  cudaSetDevice(ds->ctx->device);
  cudaStreamSynchronize(ds->ctx->stream);
  void* ps[] = {ds->dp, ds->dist, ds->sent_key, ds->sent, ds->nearq[0], ds->nearq[1], ds->touched,
                ds->emit, ds->far, ds->fkey, ds->far2, ds->fkey2, ds->scan, ds->rowbase,
                ds->part, ds->C, ds->cursors};
  for (void* p : ps)
    if (p) cudaFree(p);
  if (ds->lg) gfx_graph_destroy(ds->lg);
  delete ds;
  return GFX_OK;
}

int gfx_dsssp_bind(gfx_dsssp* ds, void* send_d, int64_t send_cap_words, void* recv_d,
                   int64_t recv_cap_words, int64_t* send_counts_d, int64_t* stats_d) {
  GFX_REQUIRE(ds && send_d && recv_d && send_counts_d && stats_d, "gfx_dsssp_bind: null argument");
  ds->send = static_cast<unsigned long long*>(send_d);
  ds->recv = static_cast<unsigned long long*>(recv_d);
  ds->send_cap = send_cap_words;
  ds->recv_cap = recv_cap_words;
  ds->send_counts = send_counts_d;
  ds->stats = stats_d;
  return GFX_OK;
}

int gfx_dsssp_reset(gfx_dsssp* ds, int64_t source, int64_t* near_local) {
  GFX_REQUIRE(ds && near_local, "gfx_dsssp_reset: null argument");
  GFX_REQUIRE(source >= 0 && source < ds->n, "source %lld out of range", (long long)source);
  gfx_ctx* ctx = ds->ctx;
  GFX_CK(cudaSetDevice(ctx->device));
  const int64_t nl = ds->nl;
  GFX_CK(cudaMemsetAsync(ds->dp, 0xFF, (nl + 1) * 8, ctx->stream));
  GFX_CK(cudaMemsetAsync(ds->dist, 0xFF, (nl + 64) * 4, ctx->stream));
  GFX_CK(cudaMemsetAsync(ds->mark, 0, (ds->wl + 1) * 4, ctx->stream));
  GFX_CK(cudaMemsetAsync(ds->sent_key, 0xFF, (ds->n + 1) * 8, ctx->stream));
  GFX_CK(cudaMemsetAsync(ds->sent, 0, ((ds->n + 31) / 32 + 1) * 4, ctx->stream));
  GFX_CK(cudaMemsetAsync(ds->C, 0, 8 * sizeof(Counters), ctx->stream));
  ds->cur = 0;
  *near_local = 0;
  if (source % ds->P == ds->r) {
    const int32_t l = (int32_t)(source / ds->P);
    GFX_LAUNCH(k_dsssp_seed, 1, 1, 0, ctx->stream, ds->dp, ds->dist, l, (int32_t)source,
               ds->nearq[0]);
    const unsigned long long one = 1;
    GFX_CK(cudaMemcpyAsync(&ds->C[0].out_len, &one, 8, cudaMemcpyHostToDevice, ctx->stream));
    *near_local = 1;
  }
  GFX_CK(cudaGetLastError());
  GFX_CK(cudaStreamSynchronize(ctx->stream));
  return GFX_OK;
}

int gfx_dsssp_relax(gfx_dsssp* ds) {
  GFX_NVTX("gfx_dsssp_relax");
  GFX_REQUIRE(ds && ds->send, "gfx_dsssp_relax: engine not bound");
  gfx_ctx* ctx = ds->ctx;
  GFX_CK(cudaSetDevice(ctx->device));
  Counters* C = ds->C;
  const int cur = ds->cur, nxt = cur ^ 1;
  GFX_CK(cudaMemsetAsync(&C[2], 0, sizeof(Counters), ctx->stream));
  GFX_CK(cudaMemsetAsync(&C[4], 0, sizeof(Counters), ctx->stream));
  GFX_CK(cudaMemsetAsync(&C[nxt], 0, sizeof(Counters), ctx->stream));
  GFX_CK(cudaMemsetAsync(ds->cursors, 0, 2 * 65 * 8, ctx->stream));
  DistRelaxOp op{ds->dp, ds->dist, ds->mark, ds->sent_key, ds->sent, ds->P, ds->r, ds->sh, {}};
  if (ds->nl > 0)
    GFX_TRY(lb_advance(ds->lg, ds->nearq[cur], &C[cur].out_len, ds->nl, &C[2], ds->scan,
                       ds->rowbase, ds->part, op, ds->emit, &C[2].out_len));
  const int grid = grid_for(ds->nl + ds->ml + 64, 256, ctx->sm_count * 8);
  unsigned long long* counts = ds->cursors + 65;
  GFX_LAUNCH(k_dsssp_bucket<0>, grid, 256, 0, ctx->stream, ds->emit, &C[2].out_len, ds->P, ds->r,
             ds->sh, counts, ds->cursors, ds->sent_key, ds->sent, ds->send, ds->touched,
             &C[4].out_len);
  GFX_LAUNCH(k_dsssp_offsets, 1, 32, 0, ctx->stream, counts, ds->P, ds->cursors, ds->send_counts);
  GFX_LAUNCH(k_dsssp_bucket<1>, grid, 256, 0, ctx->stream, ds->emit, &C[2].out_len, ds->P, ds->r,
             ds->sh, counts, ds->cursors, ds->sent_key, ds->sent, ds->send, ds->touched,
             &C[4].out_len);
  GFX_CK(cudaGetLastError());
  return GFX_OK;
}

int gfx_dsssp_apply(gfx_dsssp* ds, int64_t nrecv_words) {
  GFX_NVTX("gfx_dsssp_apply");
  GFX_REQUIRE(ds && ds->recv, "gfx_dsssp_apply: engine not bound");
  GFX_REQUIRE(nrecv_words >= 0 && nrecv_words % 2 == 0 && nrecv_words <= ds->recv_cap,
              "bad received word count %lld", (long long)nrecv_words);
  gfx_ctx* ctx = ds->ctx;
  GFX_CK(cudaSetDevice(ctx->device));
  const int64_t nmsg = nrecv_words / 2;
  if (nmsg > 0)
    GFX_LAUNCH(k_dsssp_apply, grid_for(nmsg, 256, ctx->sm_count * 8), 256, 0, ctx->stream,
               ds->recv, nmsg, ds->P, ds->sh, ds->dp, ds->dist, ds->mark, ds->touched,
               &ds->C[4].out_len);
  GFX_CK(cudaGetLastError());
  return GFX_OK;
}

int gfx_dsssp_split(gfx_dsssp* ds, double threshold) {
  GFX_NVTX("gfx_dsssp_split");
  GFX_REQUIRE(ds && ds->stats, "gfx_dsssp_split: engine not bound");
  gfx_ctx* ctx = ds->ctx;
  GFX_CK(cudaSetDevice(ctx->device));
  Counters* C = ds->C;
  const int nxt = ds->cur ^ 1;
  GFX_LAUNCH(k_sssp_split, grid_for(ds->nl + 64, 256, ctx->sm_count * 8), 256, 0, ctx->stream,
             ds->touched, &C[4].out_len, ds->dist, ds->mark, threshold, ds->nearq[nxt],
             &C[nxt].out_len, ds->far, ds->fkey, &C[3].aux0);
  GFX_LAUNCH(k_dsssp_stats, 1, 32, 0, ctx->stream, C, nxt, ds->stats);
  GFX_CK(cudaGetLastError());
  ds->cur = nxt;
  return GFX_OK;
}

// advance_bucket (split = 1) or the stale-drop compaction (split = 0); far_local
// is the host's copy of this rank's far count (from the allreduced stats)
int gfx_dsssp_refar(gfx_dsssp* ds, double threshold, int split, int64_t far_local) {
  GFX_NVTX("gfx_dsssp_refar");
  GFX_REQUIRE(ds && ds->stats, "gfx_dsssp_refar: engine not bound");
  gfx_ctx* ctx = ds->ctx;
  GFX_CK(cudaSetDevice(ctx->device));
  Counters* C = ds->C;
  const int cur = ds->cur;
  if (split) GFX_CK(cudaMemsetAsync(&C[cur], 0, sizeof(Counters), ctx->stream));
  GFX_CK(cudaMemsetAsync(&C[3].aux1, 0, 8, ctx->stream));
  GFX_CK(cudaMemsetAsync(&C[2].total, 0, 8, ctx->stream));
  GFX_CK(cudaMemsetAsync(&C[4].out_len, 0, 8, ctx->stream));
  unsigned long long* sink = &C[5].out_len;  // split == 0 never writes near
  GFX_LAUNCH(k_sssp_refar, grid_for(far_local + 1, 256, ctx->sm_count * 8), 256, 0, ctx->stream,
             ds->far, ds->fkey, far_local, ds->dist, threshold, split, ds->nearq[cur],
             split ? &C[cur].out_len : sink, ds->far2, ds->fkey2, &C[3].aux1);
  GFX_CK(cudaMemcpyAsync(&C[3].aux0, &C[3].aux1, 8, cudaMemcpyDeviceToDevice, ctx->stream));
  std::swap(ds->far, ds->far2);
  std::swap(ds->fkey, ds->fkey2);
  GFX_LAUNCH(k_dsssp_stats, 1, 32, 0, ctx->stream, C, cur, ds->stats);
  GFX_CK(cudaGetLastError());
  return GFX_OK;
}

int gfx_dsssp_result(gfx_dsssp* ds, int32_t* dist_d, int32_t* preds_d) {
  GFX_REQUIRE(ds && dist_d && preds_d, "gfx_dsssp_result: null argument");
  gfx_ctx* ctx = ds->ctx;
  GFX_CK(cudaSetDevice(ctx->device));
  if (ds->nl > 0)
    GFX_LAUNCH(k_sssp_unpack, grid_for(ds->nl, 256, ctx->sm_count * 8), 256, 0, ctx->stream,
               ds->dp, ds->nl, dist_d, preds_d, 0);
  GFX_CK(cudaGetLastError());
  GFX_CK(cudaStreamSynchronize(ctx->stream));
  return GFX_OK;
}

}  // extern "C"
