// PageRank as a deterministic pull-gather SpMV on sm_100a.
//
// Reference: primitives/pagerank.py:30-91.  Each round: dangling mass of the
// active frontier, rank_next = (1-d)/n + d*dangling/n everywhere, then every
// active s scatters d*rank[s]/outdeg[s] to its out-neighbours (np.add.at),
// then the frontier keeps vertices with |rank_next - rank| >= epsilon.
//
// Here the scatter becomes a gather over in-neighbours (no fp64 atomics, so
// runs are reproducible): contrib[u] = d*rank[u]/outdeg[u] for active u (0
// otherwise), rank_next[v] = base + sum contrib[u] in ascending u.  Vertices
// with in-degree <= 16 are summed sequentially by one thread in exactly the
// reference's slot order (bit-identical terms and order); heavier rows are
// reduced by a whole warp (tolerance: L1 <= 1e-6, north_star).
#include <cuda_runtime.h>

#include <vector>

#include "gfx_device.cuh"
#include "gfx_internal.cuh"

namespace gfx {

constexpr int kPrBlock = 256;

// contrib + per-block dangling partial sums (deterministic order)
__global__ void __launch_bounds__(kPrBlock)
    k_pr_contrib(const int64_t* __restrict__ row, int64_t n, const double* __restrict__ rank,
                 const uint8_t* __restrict__ active, double damping, double* __restrict__ contrib,
                 double* __restrict__ partials, unsigned long long* __restrict__ edges) {
  __shared__ double s_warp[kPrBlock / 32];
  double dang = 0.0;
  unsigned long long work = 0;
  // kPrCu vertices per thread in flight (independent loads), each thread's
  // dangling terms still added in increasing v within the thread
  constexpr int kPrCu = 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v0 < n;
       v0 += kPrCu * stride) {
    int64_t r0[kPrCu], r1[kPrCu];
    double rk[kPrCu];
    uint8_t act[kPrCu];
#pragma unroll
    for (int k = 0; k < kPrCu; ++k) {
      const int64_t v = v0 + k * stride;
      r0[k] = r1[k] = 0;
      rk[k] = 0.0;
      act[k] = 0;
      if (v < n) {
        r0[k] = row[v];
        r1[k] = row[v + 1];
        rk[k] = rank[v];
        act[k] = active[v];
      }
    }
#pragma unroll
    for (int k = 0; k < kPrCu; ++k) {
      const int64_t v = v0 + k * stride;
      if (v >= n) break;
      const int64_t deg = r1[k] - r0[k];
      double c = 0.0;
      if (act[k]) {
        work += (unsigned long long)deg;
        if (deg == 0) dang = __dadd_rn(dang, rk[k]);
        else c = __ddiv_rn(__dmul_rn(damping, rk[k]), (double)deg);
      }
      contrib[v] = c;
    }
  }
  dang = warp_sum_f64(dang);
  work = warp_sum_u64(work);
  if ((threadIdx.x & 31) == 0) {
    s_warp[threadIdx.x >> 5] = dang;
    if (work) atomicAdd(edges, work);  // plan.total_output of the round
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kPrBlock / 32; ++w) t = __dadd_rn(t, s_warp[w]);
    partials[blockIdx.x] = t;
  }
}

// base = (1-d)/n + d*dangling/n (reference pagerank.py:68-69, same operation order)
__global__ void k_pr_base(const double* __restrict__ partials, int nparts, int64_t n,
                          double damping, double* __restrict__ base) {
  __shared__ double s[256];
  double t = 0.0;
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) t = __dadd_rn(t, partials[i]);
  s[threadIdx.x] = t;
  __syncthreads();
  if (threadIdx.x == 0) {
    double dm = 0.0;
    for (int i = 0; i < (int)blockDim.x; ++i) dm = __dadd_rn(dm, s[i]);
    const double nn = (double)n;
    *base = __dadd_rn(__ddiv_rn(__dadd_rn(1.0, -damping), nn), __ddiv_rn(__dmul_rn(damping, dm), nn));
  }
}

// Warp per 32 consecutive vertices.  Light rows (in-degree <= kPrLight):
// one lane per row, summed in the reference's slot order, with the row's
// column ids and then their contributions fetched kPrBatch at a time (the
// loads of a batch are in flight together; the adds stay sequential, so the
// terms and their order are the reference's).  Heavy rows: the whole warp,
// kPrBatch loads per lane in flight, tree-reduced (L1 <= 1e-6 tolerance).
constexpr int kPrLight = 16;
constexpr int kPrBatch = 8;
__global__ void __launch_bounds__(kPrBlock)
    k_pr_gather(const int64_t* __restrict__ rrow, const int32_t* __restrict__ rcol, int64_t n,
                const double* __restrict__ contrib, const double* __restrict__ base_p,
                double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const double base = *base_p;
  // a lane reads its row's column ids kPrBatch at a time: through L1, so the
  // row's sector is fetched from L2 once, not once per load (s24 20 rounds
  // 43.4 -> 42.9 ms against L1::no_allocate streaming)
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t grp = gw; grp * 32 < n; grp += nw) {
    const int64_t v = grp * 32 + lane;
    int64_t b = 0, e = 0;
    if (v < n) {
      b = rrow[v];
      e = rrow[v + 1];
    }
    const bool heavy = (e - b) > kPrLight;
    double s = base;
    if (v < n && !heavy) {
      for (int64_t p = b; p < e; p += kPrBatch) {
        int32_t u[kPrBatch];
        double c[kPrBatch];
#pragma unroll
        for (int k = 0; k < kPrBatch; ++k) u[k] = p + k < e ? __ldg(rcol + p + k) : -1;
#pragma unroll
        for (int k = 0; k < kPrBatch; ++k) c[k] = u[k] >= 0 ? contrib[u[k]] : 0.0;
#pragma unroll
        for (int k = 0; k < kPrBatch; ++k)
          if (u[k] >= 0) s = __dadd_rn(s, c[k]);
      }
    }
    if (v < n && !heavy) out[v] = s;  // heavy rows: k_pr_chunks + k_pr_heavy
  }
}

// Heavy rows (in-degree > kPrLight) are cut into chunks of kPrChunk slots
// (graph-constant table, built once): one warp sums a chunk (kPrBatch loads
// per lane in flight, tree-reduced) into partial[k] ...
constexpr int64_t kPrChunk = 1024;
__global__ void __launch_bounds__(kPrBlock)
    k_pr_chunks(const int64_t* __restrict__ cstart, int64_t nchunks, const int64_t* __restrict__ cend,
                const int32_t* __restrict__ rcol, const double* __restrict__ contrib,
                double* __restrict__ partial) {
  const int lane = threadIdx.x & 31;
  const unsigned long long pol = l2_evict_first_policy();
  for (int64_t k = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; k < nchunks;
       k += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t kb = cstart[k], ke = cend[k];
    double part = 0.0;
    for (int64_t p0 = kb; p0 < ke; p0 += 32 * kPrBatch) {
      int32_t u[kPrBatch];
      double c[kPrBatch];
#pragma unroll
      for (int j = 0; j < kPrBatch; ++j) {
        const int64_t p = p0 + j * 32 + lane;
        u[j] = p < ke ? ld_stream_i32(rcol + p, pol) : -1;
      }
#pragma unroll
      for (int j = 0; j < kPrBatch; ++j) c[j] = u[j] >= 0 ? contrib[u[j]] : 0.0;
#pragma unroll
      for (int j = 0; j < kPrBatch; ++j) part = __dadd_rn(part, c[j]);
    }
    part = warp_sum_f64(part);
    if (lane == 0) partial[k] = part;
  }
}

// ... and each heavy row adds its chunks' partials in chunk order (the
// result is reproducible run to run)
__global__ void __launch_bounds__(kPrBlock)
    k_pr_heavy(const int32_t* __restrict__ hrow, const int64_t* __restrict__ hfirst, int64_t nheavy,
               const double* __restrict__ partial, const double* __restrict__ base_p,
               double* __restrict__ out) {
  const double base = *base_p;
  for (int64_t h = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; h < nheavy;
       h += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int64_t k = hfirst[h]; k < hfirst[h + 1]; ++k) s = __dadd_rn(s, partial[k]);
    out[hrow[h]] = __dadd_rn(base, s);
  }
}

// frontier filter |rank_next - rank| >= eps (pagerank.py:81-85); counts actives
__global__ void __launch_bounds__(kPrBlock)
    k_pr_moved(const double* __restrict__ nxt, const double* __restrict__ cur, int64_t n,
               double eps, uint8_t* __restrict__ active, unsigned long long* __restrict__ cnt) {
  unsigned long long c = 0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    if (active[v]) {
      const bool keep = fabs(__dadd_rn(nxt[v], -cur[v])) >= eps;
      if (!keep) active[v] = 0;
      c += keep;
    }
  }
  c = warp_sum_u64(c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(cnt, c);
}

}  // namespace gfx

using namespace gfx;

extern "C" int gfx_pagerank(gfx_graph* g, double damping, double epsilon, int64_t max_iters,
                            double* rank_d, gfx_stats* stats) {
  GFX_NVTX("gfx_pagerank");
  GFX_REQUIRE(g && rank_d, "gfx_pagerank: null argument");
  GFX_REQUIRE(damping > 0.0 && damping < 1.0, "damping must be in (0, 1)");
  GFX_REQUIRE(epsilon >= 0.0, "epsilon must be >= 0");
  GFX_REQUIRE(g->rrow != nullptr, "pagerank on a directed graph needs the reverse adjacency");
  gfx_ctx* ctx = g->ctx;
  GFX_CK(cudaSetDevice(ctx->device));
  const int64_t n = g->n;
  if (n == 0) return GFX_OK;
  double *nxt, *contrib, *partials, *base;
  uint8_t* active;
  GFX_TRY(scratch_t(g, "pr_next", n, &nxt));
  GFX_TRY(scratch_t(g, "pr_contrib", n, &contrib));
  GFX_TRY(scratch_t(g, "pr_active", n, &active));
  const int cgrid = grid_for(n, kPrBlock, ctx->sm_count * 8);
  GFX_TRY(scratch_t(g, "pr_partials", cgrid + 1, &partials));
  GFX_TRY(scratch_t(g, "pr_base", 1, &base));
  Counters* C = g->counters + 2;
  auto* pin = static_cast<Counters*>(ctx->pinned);

  // graph-constant heavy-row chunk table (reverse adjacency), built once:
  // keep_pr_meta = {nheavy, nchunks}; rows, first chunk per row, chunk bounds
  int64_t nheavy = 0, nchunks = 0;
  int32_t* hrow = nullptr;
  int64_t *hfirst = nullptr, *cstart = nullptr, *cend = nullptr;
  double* partial = nullptr;
  {
    bool fresh = false;
    void* meta = nullptr;
    GFX_TRY(scratch(g, "keep_pr_meta", 16, &meta, &fresh));
    int64_t hm[2] = {0, 0};
    if (fresh) {
      std::vector<int64_t> rr((size_t)n + 1);
      GFX_CK(cudaMemcpyAsync(rr.data(), g->rrow, (n + 1) * 8, cudaMemcpyDeviceToHost, ctx->stream));
      GFX_CK(cudaStreamSynchronize(ctx->stream));
      std::vector<int32_t> rows;
      std::vector<int64_t> first, cs, ce;
      for (int64_t v = 0; v < n; ++v) {
        const int64_t b = rr[v], e = rr[v + 1];
        if (e - b <= kPrLight) continue;
        rows.push_back((int32_t)v);
        first.push_back((int64_t)cs.size());
        for (int64_t p = b; p < e; p += kPrChunk) {
          cs.push_back(p);
          ce.push_back(p + kPrChunk < e ? p + kPrChunk : e);
        }
      }
      first.push_back((int64_t)cs.size());
      hm[0] = (int64_t)rows.size();
      hm[1] = (int64_t)cs.size();
      void* q = nullptr;
      GFX_TRY(scratch(g, "keep_pr_rows", (rows.size() + 1) * 4, &q));
      GFX_CK(cudaMemcpy(q, rows.data(), rows.size() * 4, cudaMemcpyHostToDevice));
      GFX_TRY(scratch(g, "keep_pr_first", first.size() * 8, &q));
      GFX_CK(cudaMemcpy(q, first.data(), first.size() * 8, cudaMemcpyHostToDevice));
      GFX_TRY(scratch(g, "keep_pr_cs", (cs.size() + 1) * 8, &q));
      GFX_CK(cudaMemcpy(q, cs.data(), cs.size() * 8, cudaMemcpyHostToDevice));
      GFX_TRY(scratch(g, "keep_pr_ce", (ce.size() + 1) * 8, &q));
      GFX_CK(cudaMemcpy(q, ce.data(), ce.size() * 8, cudaMemcpyHostToDevice));
      GFX_CK(cudaMemcpy(meta, hm, 16, cudaMemcpyHostToDevice));
    } else {
      GFX_CK(cudaMemcpy(hm, meta, 16, cudaMemcpyDeviceToHost));
    }
    nheavy = hm[0];
    nchunks = hm[1];
    void* q = nullptr;
    GFX_TRY(scratch(g, "keep_pr_rows", (nheavy + 1) * 4, &q));
    hrow = static_cast<int32_t*>(q);
    GFX_TRY(scratch(g, "keep_pr_first", (nheavy + 1) * 8, &q));
    hfirst = static_cast<int64_t*>(q);
    GFX_TRY(scratch(g, "keep_pr_cs", (nchunks + 1) * 8, &q));
    cstart = static_cast<int64_t*>(q);
    GFX_TRY(scratch(g, "keep_pr_ce", (nchunks + 1) * 8, &q));
    cend = static_cast<int64_t*>(q);
    GFX_TRY(scratch_t(g, "pr_partial", nchunks + 1, &partial));
  }

  GFX_CK(cudaEventRecord(ctx->ev0, ctx->stream));
  GFX_TRY(fill_f64(ctx, rank_d, 1.0 / (double)n, n));
  GFX_CK(cudaMemsetAsync(active, 1, n, ctx->stream));
  GFX_CK(cudaMemsetAsync(C, 0, sizeof(Counters), ctx->stream));
  double* cur = rank_d;
  double* nx = nxt;
  int64_t it = 0, nactive = n;
  const int ggrid = grid_for((n + 31) / 32 * 32, kPrBlock, ctx->sm_count * 16);
  while (nactive > 0 && it < max_iters) {
    ++it;
    GFX_LAUNCH(k_pr_contrib, cgrid, kPrBlock, 0, ctx->stream, g->row, n, cur, active, damping,
               contrib, partials, &C->edges);
    GFX_LAUNCH(k_pr_base, 1, 256, 0, ctx->stream, partials, cgrid, n, damping, base);
    GFX_LAUNCH(k_pr_gather, ggrid, kPrBlock, 0, ctx->stream, g->rrow, g->rcol, n, contrib, base,
               nx);
    if (nchunks) {
      GFX_LAUNCH(k_pr_chunks, grid_for(nchunks * 32, kPrBlock, ctx->sm_count * 16), kPrBlock, 0,
                 ctx->stream, cstart, nchunks, cend, g->rcol, contrib, partial);
      GFX_LAUNCH(k_pr_heavy, grid_for(nheavy, kPrBlock, ctx->sm_count * 4), kPrBlock, 0,
                 ctx->stream, hrow, hfirst, nheavy, partial, base, nx);
    }
    if (epsilon > 0.0) {
      GFX_CK(cudaMemsetAsync(&C->out_len, 0, 8, ctx->stream));
      GFX_LAUNCH(k_pr_moved, cgrid, kPrBlock, 0, ctx->stream, nx, cur, n, epsilon, active,
                 &C->out_len);
      GFX_CK(cudaMemcpyAsync(pin, C, sizeof(Counters), cudaMemcpyDeviceToHost, ctx->stream));
      GFX_CK(cudaStreamSynchronize(ctx->stream));
      nactive = (int64_t)pin->out_len;
    }
    std::swap(cur, nx);
  }
  GFX_CK(cudaGetLastError());
  if (cur != rank_d)
    GFX_CK(cudaMemcpyAsync(rank_d, cur, n * sizeof(double), cudaMemcpyDeviceToDevice,
                           ctx->stream));
  GFX_CK(cudaEventRecord(ctx->ev1, ctx->stream));
  GFX_CK(cudaEventSynchronize(ctx->ev1));
  float ms = 0.f;
  GFX_CK(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
  GFX_CK(cudaMemcpyAsync(pin, C, sizeof(Counters), cudaMemcpyDeviceToHost, ctx->stream));
  GFX_CK(cudaStreamSynchronize(ctx->stream));
  if (stats) {
    *stats = gfx_stats{};
    stats->iterations = it;
    stats->edges_traversed = (int64_t)pin->edges;
    stats->device_ms = ms;
    // per round: col (4m) + row, contrib write/read, rank read/write (40n)
    stats->bytes_alg = it * (4 * g->m + 40 * n);
  }
  return GFX_OK;
}
