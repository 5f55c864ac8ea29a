// Kernel-level experiment entry point (used by tools/expand_lab.py to break
// the push expansion's time into streaming / probing / claiming parts).
// Not on any product path.
#include <cuda_runtime.h>

#include "gfx_device.cuh"
#include "gfx_expand.cuh"
#include "gfx_internal.cuh"

namespace gfx {

// variant 0 / 3: stream the adjacency only (no functor memory traffic),
// 16 / 8 column loads in flight per lane
template <int KB>
struct StreamOpT {
  static constexpr bool kWeights = false, kSrcVal = false, kEmitEdge = false;
  static constexpr int kBatch = KB;
  static constexpr int kMinBlocks = 3;
  int32_t sentinel;
  __device__ int32_t src_value(int32_t) const { return 0; }
  __device__ void prefetch(const int32_t*) {}
  __device__ bool visit(int, int32_t d, int32_t, int32_t, int32_t, int64_t) {
    return d == sentinel;  // never true for valid ids; keeps the load live
  }
};

// variant 1: stream + visited-bit probe, no atomics (emits unvisited slots)
struct ProbeOp {
  static constexpr bool kWeights = false, kSrcVal = false, kEmitEdge = false;
  static constexpr int kBatch = kVisitBatch;
  static constexpr int kMinBlocks = 3;
  const uint32_t* visited;
  uint32_t wv[kBatch];
  __device__ int32_t src_value(int32_t) const { return 0; }
  __device__ void prefetch(const int32_t* d) {
#pragma unroll
    for (int u = 0; u < kBatch; ++u) wv[u] = d[u] >= 0 ? visited[d[u] >> 5] : 0xffffffffu;
  }
  __device__ bool visit(int u, int32_t d, int32_t, int32_t, int32_t, int64_t) {
    return !((wv[u] >> (d & 31)) & 1u);
  }
};

// variant 2: full claim (as BfsClaimOp) on a private visited copy
struct ClaimOp {
  static constexpr bool kWeights = false, kSrcVal = false, kEmitEdge = false;
  static constexpr int kBatch = kVisitBatch;
  static constexpr int kMinBlocks = 3;
  uint32_t* visited;
  int32_t* labels;
  int32_t depth;
  uint32_t wv[kBatch];
  __device__ int32_t src_value(int32_t) const { return 0; }
  __device__ void prefetch(const int32_t* d) {
#pragma unroll
    for (int u = 0; u < kBatch; ++u) wv[u] = d[u] >= 0 ? visited[d[u] >> 5] : 0xffffffffu;
  }
  __device__ bool visit(int u, int32_t d, int32_t, int32_t, int32_t, int64_t) {
    const uint32_t bit = 1u << (d & 31);
    if (wv[u] & bit) return false;
    if (atomicOr(&visited[d >> 5], bit) & bit) return false;
    labels[d] = depth;
    return true;
  }
};

__global__ void k_visited_from_labels(const int32_t* __restrict__ labels, int64_t n,
                                      int32_t below, uint32_t* __restrict__ bm, int64_t words) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < words * 32;
       i += (int64_t)gridDim.x * blockDim.x) {
    const bool v = i < n && labels[i] < below;
    const unsigned b = __ballot_sync(0xffffffffu, v);
    if ((threadIdx.x & 31) == 0) bm[i >> 5] = b;
  }
}

}  // namespace gfx

using namespace gfx;

extern "C" int gfx_debug_expand(gfx_graph* g, const int32_t* F_d, int64_t nf, int variant,
                                        int32_t* labels_d, int32_t depth, float* ms,
                                        int64_t* out_count) {
  GFX_REQUIRE(g && F_d && ms && out_count && labels_d, "gfx_debug_expand: null argument");
  gfx_ctx* ctx = g->ctx;
  GFX_CK(cudaSetDevice(ctx->device));
  const int64_t n = g->n;
  int32_t *part, *out;
  int64_t *scan, *rowbase;
  uint32_t* vis;
  GFX_TRY(scratch_t(g, "q_scan", n + 2, &scan));
  GFX_TRY(scratch_t(g, "q_rowbase", n + 1, &rowbase));
  GFX_TRY(scratch_t(g, "q_part", part_capacity(g->m, g->n), &part));
  GFX_TRY(scratch_t(g, "dbg_out", g->m + 1, &out));
  GFX_TRY(scratch_t(g, "dbg_vis", g->words, &vis));
  Counters* C = g->counters;
  GFX_CK(cudaMemsetAsync(C, 0, 2 * sizeof(Counters), ctx->stream));
  const unsigned long long nn = (unsigned long long)nf;
  GFX_CK(cudaMemcpyAsync(&C[0].out_len, &nn, 8, cudaMemcpyHostToDevice, ctx->stream));
  GFX_LAUNCH(k_visited_from_labels, grid_for(g->words * 32, 256, ctx->sm_count * 8), 256, 0,
             ctx->stream, labels_d, n, depth, vis, g->words);
  GFX_CK(cudaEventRecord(ctx->ev0, ctx->stream));
  int st = GFX_OK;
  if (variant == 0) {
    StreamOpT<16> op{-7};
    st = lb_advance(g, F_d, &C[0].out_len, nf, &C[1], scan, rowbase, part, op, out, &C[1].out_len);
  } else if (variant == 3) {
    StreamOpT<8> op{-7};
    st = lb_advance(g, F_d, &C[0].out_len, nf, &C[1], scan, rowbase, part, op, out, &C[1].out_len);
  } else if (variant == 1) {
    ProbeOp op{vis, {}};
    st = lb_advance(g, F_d, &C[0].out_len, nf, &C[1], scan, rowbase, part, op, out, &C[1].out_len);
  } else {
    ClaimOp op{vis, labels_d, depth, {}};
    st = lb_advance(g, F_d, &C[0].out_len, nf, &C[1], scan, rowbase, part, op, out, &C[1].out_len);
  }
  if (st != GFX_OK) return st;
  GFX_CK(cudaEventRecord(ctx->ev1, ctx->stream));
  GFX_CK(cudaEventSynchronize(ctx->ev1));
  GFX_CK(cudaEventElapsedTime(ms, ctx->ev0, ctx->ev1));
  unsigned long long cnt = 0;
  GFX_CK(cudaMemcpy(&cnt, &C[1].out_len, 8, cudaMemcpyDeviceToHost));
  *out_count = (int64_t)cnt;
  return GFX_OK;
}
