// Connected components: lock-free union-find hooking over every undirected
// edge (one load-balanced pass), then full pointer jumping.
//
// Reference: primitives/cc.py:23-98 hooks component ids over an edge
// frontier with alternating parity and pointer-jumps after every round; its
// labels are arbitrary representatives.  Here every union
// hooks the larger root under the smaller one (atomicCAS on the root), so a
// tree's root is always its minimum vertex and the output is the canonical
// min-id labelling -- parity is bit-exact against the reference's labels
// canonicalised to min-id.  Path halving in find() only rewrites non-root
// parents to an ancestor, never racing with the root CAS.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "gfx_device.cuh"
#include "gfx_expand.cuh"
#include "gfx_internal.cuh"

namespace gfx {

__device__ __forceinline__ int32_t ld_parent(const int32_t* p, int32_t x) {
  int32_t v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p + x) : "memory");
  return v;
}

__device__ __forceinline__ int32_t cc_find(int32_t* p, int32_t x) {
  for (;;) {
    const int32_t y = ld_parent(p, x);
    if (y == x) return x;
    const int32_t z = ld_parent(p, y);
    if (z == y) return y;
    p[x] = z;  // halving: z is an ancestor of x, never a write to a root
    x = z;
  }
}

__device__ __forceinline__ void cc_unite(int32_t* p, int32_t a, int32_t b) {
  for (;;) {
    a = cc_find(p, a);
    b = cc_find(p, b);
    if (a == b) return;
    if (a < b) {
      const int32_t t = a;
      a = b;
      b = t;
    }
    // hook the larger root a under the smaller root b
    const int32_t old = atomicCAS(&p[a], a, b);
    if (old == a) return;
    a = old;
  }
}

struct CcHookOp {
  static constexpr bool kWeights = false, kSrcVal = false, kEmitEdge = false;
  static constexpr int kBatch = kVisitBatch;
  static constexpr int kMinBlocks = 2;
  int32_t* parent;
  __device__ int32_t src_value(int32_t) const { return 0; }
  __device__ void prefetch(const int32_t*) {}
  __device__ bool visit(int, int32_t d, int32_t s, int32_t, int32_t, int64_t) {
    if (s < d) cc_unite(parent, s, d);  // each undirected edge once (cc.py:44-47)
    return false;
  }
};

__global__ void k_iota(int32_t* __restrict__ p, int64_t n) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x)
    p[v] = (int32_t)v;
}

__global__ void k_cc_compress(int32_t* __restrict__ parent, int64_t n, int32_t* __restrict__ comp,
                              unsigned long long* __restrict__ nroots) {
  unsigned long long roots = 0;
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    int32_t r = (int32_t)v;
    for (int32_t q = parent[r]; q != r; q = parent[r]) r = q;
    comp[v] = r;
    roots += (r == (int32_t)v);
  }
  roots = warp_sum_u64(roots);
  if ((threadIdx.x & 31) == 0 && roots) atomicAdd(nroots, roots);
}

// ---------------------------------------------------------------------------
// Afforest-style shortcut (sampling then skipping the giant component):
// round r links every vertex to its r-th neighbour; after full compression
// the most frequent root among sampled vertices is the giant component c;
// only vertices outside c then link their remaining neighbours.  Every edge
// (v, u) leaving c is still processed from its non-c endpoint (the adjacency
// is symmetric), so the final partition is the same; unite keeps each
// tree's root at its minimum vertex, so labels stay canonical min-id.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256)
    k_cc_sample(const int64_t* __restrict__ row, const int32_t* __restrict__ col, int64_t n, int r,
                int32_t* __restrict__ parent) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = row[v];
    if (row[v + 1] - b > r) cc_unite(parent, (int32_t)v, col[b + r]);
  }
}

// full compression: parent[v] = root (roots are never rewritten)
__global__ void __launch_bounds__(256) k_cc_flatten(int32_t* __restrict__ parent, int64_t n) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    int32_t r = parent[v];
    while (true) {
      const int32_t q = ld_parent(parent, r);
      if (q == r) break;
      r = q;
    }
    parent[v] = r;
  }
}

// vertices outside the giant component link their remaining neighbours
// (from index `from`): light rows one lane each, heavy rows by the warp
__global__ void __launch_bounds__(256)
    k_cc_rest(const int64_t* __restrict__ row, const int32_t* __restrict__ col, int64_t n,
              int from, int32_t giant, int32_t* __restrict__ parent,
              unsigned long long* __restrict__ slots) {
  const int lane = threadIdx.x & 31;
  unsigned long long mine = 0;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t grp = gw; grp * 32 < n; grp += nw) {
    const int64_t v = grp * 32 + lane;
    int64_t b = 0, e = 0;
    if (v < n && cc_find(parent, (int32_t)v) != giant) {
      b = row[v] + from;
      e = row[v + 1];
    }
    const bool heavy = e - b > 32;
    if (e > b) mine += (unsigned long long)(e - b);
    if (!heavy)
      for (int64_t p = b; p < e; ++p) cc_unite(parent, (int32_t)v, col[p]);
    unsigned hm = __ballot_sync(0xffffffffu, heavy);
    while (hm) {
      const int k = __ffs(hm) - 1;
      hm &= hm - 1;
      const int32_t kv = (int32_t)(grp * 32 + k);
      const int64_t kb = __shfl_sync(0xffffffffu, b, k), ke = __shfl_sync(0xffffffffu, e, k);
      for (int64_t p = kb + lane; p < ke; p += 32) cc_unite(parent, kv, col[p]);
    }
  }
  mine = warp_sum_u64(mine);
  if (lane == 0 && mine) atomicAdd(slots, mine);
}

int iota_frontier(gfx_graph* g, int32_t** out) {
  bool fresh = false;
  void* p = nullptr;
  GFX_TRY(scratch(g, "keep_iota", (size_t)(g->n + 1) * 4, &p, &fresh));
  *out = static_cast<int32_t*>(p);
  if (fresh)
    GFX_LAUNCH(k_iota, grid_for(g->n, 256, g->ctx->sm_count * 8), 256, 0, g->ctx->stream, *out,
               g->n);
  return GFX_OK;
}

}  // namespace gfx

using namespace gfx;

extern "C" int gfx_cc(gfx_graph* g, int32_t* comp_d, int64_t* num_components, gfx_stats* stats) {
  GFX_NVTX("gfx_cc");
  GFX_REQUIRE(g && comp_d && num_components, "gfx_cc: null argument");
  GFX_REQUIRE(g->flags & GFX_GRAPH_UNDIRECTED, "cc expects an undirected graph");
  gfx_ctx* ctx = g->ctx;
  GFX_CK(cudaSetDevice(ctx->device));
  const int64_t n = g->n;
  if (n == 0) {
    *num_components = 0;
    return GFX_OK;
  }
  int32_t *parent, *iota, *part;
  int64_t *scan, *rowbase;
  GFX_TRY(scratch_t(g, "cc_parent", n, &parent));
  GFX_TRY(iota_frontier(g, &iota));
  GFX_TRY(scratch_t(g, "q_scan", n + 2, &scan));
  GFX_TRY(scratch_t(g, "q_rowbase", n + 1, &rowbase));
  GFX_TRY(scratch_t(g, "q_part", part_capacity(g->m, g->n), &part));
  Counters* C = g->counters;
  auto* pin = static_cast<Counters*>(ctx->pinned);

  GFX_CK(cudaEventRecord(ctx->ev0, ctx->stream));
  GFX_CK(cudaMemsetAsync(C, 0, 2 * sizeof(Counters), ctx->stream));
  const unsigned long long nn = (unsigned long long)n;
  GFX_CK(cudaMemcpyAsync(&C[0].out_len, &nn, 8, cudaMemcpyHostToDevice, ctx->stream));
  const int grid = grid_for(n, 256, ctx->sm_count * 8);
  GFX_LAUNCH(k_iota, grid, 256, 0, ctx->stream, parent, n);
  const bool afforest = getenv("GFX_CC_PLAIN") == nullptr;
  if (afforest) {
    constexpr int kRounds = 2;
    for (int r = 0; r < kRounds; ++r)
      GFX_LAUNCH(k_cc_sample, grid, 256, 0, ctx->stream, g->row, g->col, n, r, parent);
    GFX_LAUNCH(k_cc_flatten, grid, 256, 0, ctx->stream, parent, n);
    // the giant component: the most frequent root among 1024 evenly spaced
    // vertices with at least one edge... sampled on the host
    constexpr int kSample = 1024;
    int32_t* samp = nullptr;
    GFX_TRY(scratch_t(g, "cc_sample", kSample, &samp));
    const int64_t stride = n / kSample > 0 ? n / kSample : 1;
    GFX_CK(cudaMemcpy2DAsync(samp, 4, parent, stride * 4, 4, std::min<int64_t>(kSample, n),
                             cudaMemcpyDeviceToDevice, ctx->stream));
    std::vector<int32_t> hs((size_t)std::min<int64_t>(kSample, n));
    GFX_CK(cudaMemcpyAsync(hs.data(), samp, hs.size() * 4, cudaMemcpyDeviceToHost, ctx->stream));
    GFX_CK(cudaStreamSynchronize(ctx->stream));
    std::sort(hs.begin(), hs.end());
    int32_t giant = hs.empty() ? 0 : hs[0];
    size_t best = 0;
    for (size_t i = 0; i < hs.size();) {
      size_t j = i;
      while (j < hs.size() && hs[j] == hs[i]) ++j;
      if (j - i > best) {
        best = j - i;
        giant = hs[i];
      }
      i = j;
    }
    GFX_LAUNCH(k_cc_rest, grid_for(n, 256, ctx->sm_count * 16), 256, 0, ctx->stream, g->row,
               g->col, n, kRounds, giant, parent, &C[1].aux1);
  } else {
    CcHookOp op{parent};
    GFX_TRY(lb_advance(g, iota, &C[0].out_len, n, &C[1], scan, rowbase, part, op, nullptr,
                       &C[1].out_len));
  }
  GFX_LAUNCH(k_cc_compress, grid, 256, 0, ctx->stream, parent, n, comp_d, &C[1].aux0);
  GFX_CK(cudaGetLastError());
  GFX_CK(cudaEventRecord(ctx->ev1, ctx->stream));
  GFX_CK(cudaMemcpyAsync(pin, C, 2 * sizeof(Counters), cudaMemcpyDeviceToHost, ctx->stream));
  GFX_CK(cudaStreamSynchronize(ctx->stream));
  float ms = 0.f;
  GFX_CK(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
  *num_components = (int64_t)pin[1].aux0;
  if (stats) {
    *stats = gfx_stats{};
    stats->iterations = 1;
    stats->edges_traversed = g->m / 2;  // each undirected edge hooked once (reference plan)
    stats->device_ms = ms;
    if (afforest) {
      // two sampling rounds (row pair + one col per vertex), flatten and
      // final compress (parent read/write), and the slots the non-giant
      // vertices linked
      const int64_t rest = (int64_t)pin[1].aux1;
      stats->work_slots = 2 * n + rest;
      stats->bytes_alg = 2 * 20 * n + 16 * n + 16 * n + 4 * rest;
    } else {
      stats->work_slots = g->m;
      // one hook pass (col + row) + parent init/compress
      stats->bytes_alg = 4 * g->m + 16 * n;
    }
  }
  return GFX_OK;
}
