// Betweenness centrality (Brandes) with deterministic pull-gathers.
//
// Reference: primitives/bc.py:32-116.  Forward: level-synchronous BFS with a
// CAS claim, and per level sigma[d] += sigma[s] over every edge landing on
// the new level (np.add.at).  Backward: deepest level first, delta[s] +=
// sigma[s]/sigma[d] * (1 + delta[d]) over edges s -> d with d one level
// deeper; delta[source] = 0; bc += delta.
//
// Device: the forward BFS is the push LB expansion (gfx_bfs.cu) keeping every
// level's frontier; sigma and delta are then gathered level by level with no
// fp64 atomics: sigma[v] = sum of sigma over in-neighbours one level up,
// delta[v] = sum over out-neighbours one level down, each term computed as
// (sigma[v] / sigma[w]) * (1 + delta[w]) with round-to-nearest intrinsics (no
// FMA contraction).  Light rows (<= 32) are summed sequentially in ascending
// neighbour order -- the reference's slot order -- so their values are
// bit-identical; heavier rows use a warp reduction (rel <= 1e-5, north_star).
#include <cuda_runtime.h>

#include <cstdlib>
#include <vector>

#include "gfx_device.cuh"
#include "gfx_expand.cuh"
#include "gfx_internal.cuh"

namespace gfx {

// Each term loads everything it needs for neighbour u in one go (the label
// and the value arrays in parallel), then evaluates -- so a batch of
// neighbours costs two dependent round trips (column ids, then their data).
struct SigmaTerm {
  const int32_t* labels;
  const double* sigma;
  int32_t want;  // level of contributing neighbours
  struct V {
    int32_t l;
    double s;
  };
  __device__ V load(int32_t u) const { return V{labels[u], sigma[u]}; }
  __device__ double eval(int32_t, const V& x) const { return x.l == want ? x.s : 0.0; }
};

struct DeltaTerm {
  const int32_t* labels;
  const double* sigma;
  const double* delta;
  int32_t want;
  struct V {
    int32_t l;
    double s, d;
  };
  __device__ V load(int32_t u) const { return V{labels[u], sigma[u], delta[u]}; }
  __device__ double eval(int32_t v, const V& x) const {
    if (x.l != want) return 0.0;
    return __dmul_rn(__ddiv_rn(sigma[v], x.s), __dadd_rn(1.0, x.d));
  }
};

// out[v] = sum_{u in adj(v)} T(v, u) for v in items[0..cnt).  Light rows
// (<= kGatherLight): one lane per row, kGatherBatch neighbours' loads in
// flight, terms added sequentially in ascending neighbour order (the
// reference's slot order); heavy rows: the whole warp, kGatherBatch loads
// per lane in flight, tree-reduced.
constexpr int kGatherLight = 32;
constexpr int kGatherBatch = 8;
template <class T>
__global__ void __launch_bounds__(256)
    k_level_gather(const int32_t* __restrict__ items, int64_t cnt, const int64_t* __restrict__ rows,
                   const int32_t* __restrict__ cols, T term, double* __restrict__ out) {
  constexpr int B = kGatherBatch;
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t grp = gw; grp * 32 < cnt; grp += nw) {
    const int64_t i = grp * 32 + lane;
    int32_t v = 0;
    int64_t b = 0, e = 0;
    if (i < cnt) {
      v = items[i];
      b = rows[v];
      e = rows[v + 1];
    }
    const bool heavy = (e - b) > kGatherLight;
    double acc = 0.0;
    if (i < cnt && !heavy)
      for (int64_t p0 = b; p0 < e; p0 += B) {
        int32_t u[B];
        typename T::V x[B];
#pragma unroll
        for (int k = 0; k < B; ++k) u[k] = p0 + k < e ? ld_stream_i32(cols + p0 + k) : -1;
#pragma unroll
        for (int k = 0; k < B; ++k)
          if (u[k] >= 0) x[k] = term.load(u[k]);
#pragma unroll
        for (int k = 0; k < B; ++k) {
          if (u[k] < 0) continue;
          const double t = term.eval(v, x[k]);
          if (t != 0.0) acc = __dadd_rn(acc, t);
        }
      }
    unsigned hm = __ballot_sync(0xffffffffu, heavy);
    while (hm) {
      const int k = __ffs(hm) - 1;
      hm &= hm - 1;
      const int32_t kv = __shfl_sync(0xffffffffu, v, k);
      const int64_t kb = __shfl_sync(0xffffffffu, b, k), ke = __shfl_sync(0xffffffffu, e, k);
      double part = 0.0;
      for (int64_t p0 = kb; p0 < ke; p0 += 32 * B) {
        int32_t u[B];
        typename T::V x[B];
#pragma unroll
        for (int j = 0; j < B; ++j) {
          const int64_t p = p0 + j * 32 + lane;
          u[j] = p < ke ? ld_stream_i32(cols + p) : -1;
        }
#pragma unroll
        for (int j = 0; j < B; ++j)
          if (u[j] >= 0) x[j] = term.load(u[j]);
#pragma unroll
        for (int j = 0; j < B; ++j)
          if (u[j] >= 0) part = __dadd_rn(part, term.eval(kv, x[j]));
      }
      part = warp_sum_f64(part);
      if (lane == k) acc = part;
    }
    if (i < cnt) out[v] = acc;
  }
}

// Push forms, used on undirected graphs for a level whose neighbour level
// has fewer slots than the level itself (the load-balanced expansion then
// splits hubs across warps).  Forward: sigma values are path counts --
// integers held exactly in fp64 (< 2^53) -- so the atomic sums are exact in
// any order and the result is deterministic.  Backward: the terms are summed
// exactly in 128-bit fixed point (Fix128 below) and rounded once, so the
// push is deterministic too (GFX_BC_DELTA_PUSH=0 gathers every level).
struct SigmaPushOp {
  static constexpr bool kWeights = false, kSrcVal = false, kEmitEdge = false;
  static constexpr int kBatch = kVisitBatch;
  static constexpr int kMinBlocks = 3;
  const int32_t* labels;
  double* sigma;
  int32_t want;  // level of the receiving neighbours
  int32_t lv[kBatch];
  __device__ int32_t src_value(int32_t) const { return 0; }
  __device__ void prefetch(const int32_t* d) {
#pragma unroll
    for (int u = 0; u < kBatch; ++u) lv[u] = d[u] >= 0 ? labels[d[u]] : -1;
  }
  __device__ bool visit(int u, int32_t d, int32_t s, int32_t, int32_t, int64_t) {
    if (lv[u] == want) atomicAdd(&sigma[d], sigma[s]);
    return false;
  }
};

// Exact, order-independent accumulation of non-negative doubles: every term
// is converted EXACTLY to a 128-bit fixed-point number with 64 fractional
// bits (a 53-bit mantissa shifted into place; bits below 2^-64 are dropped
// per term, deterministically) and added with integer atomics -- the low
// word's carry propagated into the high word -- so the sum is the same
// whatever order the terms arrive in, and is then rounded to a double once.
struct Fix128 {
  unsigned long long lo, hi;
};
__device__ __forceinline__ Fix128 to_fix128(double t) {
  Fix128 f{0ull, 0ull};
  if (!(t > 0.0)) return f;
  int e;
  const double m = frexp(t, &e);  // t = m * 2^e, m in [0.5, 1)
  const unsigned long long mant = (unsigned long long)ldexp(m, 53);  // exact
  const int sh = e - 53 + 64;                                       // mant * 2^sh
  if (sh >= 128) return Fix128{~0ull, ~0ull};                       // saturate (not reached)
  if (sh >= 64) {
    f.hi = mant << (sh - 64);
  } else if (sh > 0) {
    f.lo = mant << sh;
    f.hi = mant >> (64 - sh);
  } else if (sh > -64) {
    f.lo = mant >> (-sh);
  }
  return f;
}
__device__ __forceinline__ void fix128_add(unsigned long long* acc, Fix128 f) {
  // acc[0] = low word, acc[1] = high word of this vertex's sum
  if (f.lo) {
    const unsigned long long old = atomicAdd(&acc[0], f.lo);
    if (old + f.lo < old) f.hi += 1ull;  // carry out of the low word
  }
  if (f.hi) atomicAdd(&acc[1], f.hi);
}

struct DeltaPushOp {  // frontier: level want + 1; receivers: neighbours at level want
  static constexpr bool kWeights = false, kSrcVal = false, kEmitEdge = false;
  static constexpr int kBatch = kVisitBatch;
  static constexpr int kMinBlocks = 3;
  const int32_t* labels;
  const double* sigma;
  const double* delta;
  unsigned long long* acc;  // 2 words per vertex (Fix128)
  int32_t want;
  int32_t lv[kBatch];
  __device__ int32_t src_value(int32_t) const { return 0; }
  __device__ void prefetch(const int32_t* d) {
#pragma unroll
    for (int u = 0; u < kBatch; ++u) lv[u] = d[u] >= 0 ? labels[d[u]] : -1;
  }
  __device__ bool visit(int u, int32_t s, int32_t w, int32_t, int32_t, int64_t) {
    if (lv[u] == want)
      fix128_add(acc + 2 * (int64_t)s,
                 to_fix128(__dmul_rn(__ddiv_rn(sigma[s], sigma[w]), __dadd_rn(1.0, delta[w]))));
    return false;
  }
};

// delta[v] = the level's fixed-point sums rounded once; accumulators cleared
__global__ void k_fix128_finish(const int32_t* __restrict__ items, int64_t cnt,
                                unsigned long long* __restrict__ acc, double* __restrict__ delta) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = items[i];
    const unsigned long long lo = acc[2 * (int64_t)v], hi = acc[2 * (int64_t)v + 1];
    delta[v] = __dadd_rn((double)hi, ldexp((double)lo, -64));
    acc[2 * (int64_t)v] = 0ull;
    acc[2 * (int64_t)v + 1] = 0ull;
  }
}

__global__ void k_bc_seed(double* sigma, int32_t src) { sigma[src] = 1.0; }

__global__ void k_bc_accumulate(const int32_t* __restrict__ items, int64_t cnt,
                                const double* __restrict__ delta, int32_t src,
                                double* __restrict__ bc) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = items[i];
    if (v != src) bc[v] = __dadd_rn(bc[v], delta[v]);
  }
}

}  // namespace gfx

using namespace gfx;

extern "C" int gfx_bc(gfx_graph* g, const int64_t* sources, int64_t num_sources, double* bc_d,
                      gfx_stats* stats) {
  GFX_NVTX("gfx_bc");
  GFX_REQUIRE(g && bc_d && (num_sources == 0 || sources), "gfx_bc: null argument");
  for (int64_t i = 0; i < num_sources; ++i)
    GFX_REQUIRE(sources[i] >= 0 && sources[i] < g->n, "source %lld out of range",
                (long long)sources[i]);
  GFX_REQUIRE(g->rrow != nullptr, "bc on a directed graph needs the reverse adjacency");
  gfx_ctx* ctx = g->ctx;
  GFX_CK(cudaSetDevice(ctx->device));
  const int64_t n = g->n;
  int32_t *labels, *preds;
  double *sigma, *delta;
  GFX_TRY(scratch_t(g, "bc_labels", n + 1, &labels));
  GFX_TRY(scratch_t(g, "bc_preds", n + 1, &preds));
  GFX_TRY(scratch_t(g, "bc_sigma", n + 1, &sigma));
  GFX_TRY(scratch_t(g, "bc_delta", n + 1, &delta));
  const int grid = ctx->sm_count * 8;
  int32_t* part;
  int64_t *scan, *rowbase;
  GFX_TRY(scratch_t(g, "q_scan", n + 2, &scan));
  GFX_TRY(scratch_t(g, "q_rowbase", n + 1, &rowbase));
  GFX_TRY(scratch_t(g, "q_part", part_capacity(g->m, g->n), &part));
  Counters* pc = g->counters + 2;  // push plans (C[2], C[3])
  // the backward push accumulates exactly in 128-bit fixed point (Fix128),
  // so BC values are bit-reproducible run to run; GFX_BC_DELTA_PUSH=0
  // forces the pull-gather on every level (diagnostic)
  const char* dp = std::getenv("GFX_BC_DELTA_PUSH");
  const bool delta_push = !(dp && dp[0] == '0');
  // forward levels from the direction-optimising persistent BFS (no host
  // round trip per level); GFX_BC_FWD=push restores the push-only level loop
  const char* fw = std::getenv("GFX_BC_FWD");
  const bool fwd_do = !(fw && fw[0] == 'p');
  unsigned long long* acc = nullptr;
  bool acc_fresh = false;
  GFX_TRY(scratch(g, "bc_fix128", (size_t)(n + 1) * 16, reinterpret_cast<void**>(&acc),
                  &acc_fresh));
  if (acc_fresh) GFX_CK(cudaMemsetAsync(acc, 0, (size_t)(n + 1) * 16, ctx->stream));
  int64_t iterations = 0, edges = 0;
  std::vector<int64_t> off;
  GFX_CK(cudaEventRecord(ctx->ev0, ctx->stream));
  for (int64_t si = 0; si < num_sources; ++si) {
    const int32_t src = (int32_t)sources[si];
    int32_t* order = nullptr;
    std::vector<int64_t> slots;
    if (fwd_do) GFX_TRY(bfs_do_levels(g, src, labels, preds, &off, &order, &slots));
    else GFX_TRY(bfs_push_levels(g, src, labels, preds, &off, &order, &slots));
    const bool undirected = (g->flags & GFX_GRAPH_UNDIRECTED) != 0;
    // push a level from its neighbour level when that is fewer slots
    auto push_from = [&](int64_t lvl, auto op) -> int {
      const int64_t cnt = off[lvl + 1] - off[lvl];
      const unsigned long long c = (unsigned long long)cnt;
      GFX_CK(cudaMemcpyAsync(&pc[0].out_len, &c, 8, cudaMemcpyHostToDevice, ctx->stream));
      GFX_CK(cudaMemsetAsync(&pc[1], 0, sizeof(Counters), ctx->stream));
      return lb_advance(g, order + off[lvl], &pc[0].out_len, cnt, &pc[1], scan, rowbase, part, op,
                        nullptr, &pc[1].out_len);
    };
    const int64_t L = (int64_t)off.size() - 1;  // levels 0..L-1 (last is empty)
    // forward: sigma level by level (bc.py:87-92)
    GFX_CK(cudaMemsetAsync(sigma, 0, n * sizeof(double), ctx->stream));
    GFX_LAUNCH(k_bc_seed, 1, 1, 0, ctx->stream, sigma, src);
    for (int64_t d = 1; d < L; ++d) {
      const int64_t cnt = off[d + 1] - off[d];
      if (cnt <= 0) continue;
      if (undirected && slots[d - 1] < slots[d]) {
        GFX_TRY(push_from(d - 1, SigmaPushOp{labels, sigma, (int32_t)d, {}}));
        continue;
      }
      SigmaTerm t{labels, sigma, (int32_t)(d - 1)};
      GFX_LAUNCH((k_level_gather<SigmaTerm>), grid_for(cnt * 32, 256, grid), 256, 0, ctx->stream,
                 order + off[d], cnt, g->rrow, g->rcol, t, sigma);
    }
    // backward: delta deepest level first (bc.py:98-116); the source's own
    // delta is 0 by definition (bc.py:110), so level 0 is not gathered
    GFX_CK(cudaMemsetAsync(delta, 0, n * sizeof(double), ctx->stream));
    for (int64_t d = L - 2; d >= 1; --d) {
      const int64_t cnt = off[d + 1] - off[d];
      if (cnt <= 0) continue;
      if (delta_push && undirected && d + 1 < (int64_t)slots.size() && slots[d + 1] < slots[d] &&
          off[d + 2] > off[d + 1]) {
        GFX_TRY(push_from(d + 1, DeltaPushOp{labels, sigma, delta, acc, (int32_t)d, {}}));
        GFX_LAUNCH(k_fix128_finish, grid_for(cnt, 256, grid), 256, 0, ctx->stream, order + off[d],
                   cnt, acc, delta);
        continue;
      }
      DeltaTerm t{labels, sigma, delta, (int32_t)(d + 1)};
      GFX_LAUNCH((k_level_gather<DeltaTerm>), grid_for(cnt * 32, 256, grid), 256, 0, ctx->stream,
                 order + off[d], cnt, g->row, g->col, t, delta);
    }
    const int64_t reached = off[L];
    GFX_LAUNCH(k_bc_accumulate, grid_for(reached, 256, grid), 256, 0, ctx->stream, order, reached,
               delta, src, bc_d);
    GFX_CK(cudaGetLastError());
    iterations += L - 1;
    int64_t er = 0, rc = 0;
    GFX_TRY(reached_stats(g, labels, &rc, &er));
    edges += er;
  }
  GFX_CK(cudaEventRecord(ctx->ev1, ctx->stream));
  GFX_CK(cudaEventSynchronize(ctx->ev1));
  float ms = 0.f;
  GFX_CK(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
  if (stats) {
    *stats = gfx_stats{};
    stats->iterations = iterations;
    stats->edges_traversed = edges;  // forward plans only (bc.py:67-68)
    stats->edges_reached = edges;
    stats->device_ms = ms;
  }
  return GFX_OK;
}
