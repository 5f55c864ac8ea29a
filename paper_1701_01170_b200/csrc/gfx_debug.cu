// Kernel-level experiment entry point (used by tools/expand_lab.py to break
// the push expansion's time into streaming / probing / claiming parts).
// Not on any product path.
#include <cooperative_groups.h>
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

// grid-barrier microbenchmark: cg::grid sync vs a flag barrier (per-block
// arrival words polled by block 0, one release word)
__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void flag_barrier(unsigned* flags, unsigned* gen, unsigned g) {
  __syncthreads();
  if (threadIdx.x == 0) st_rel(&flags[blockIdx.x * 32], g);
  if (blockIdx.x == 0) {
    for (unsigned i = threadIdx.x; i < gridDim.x; i += blockDim.x)
      while (ld_acq(&flags[i * 32]) != g) {
      }
    __syncthreads();
    if (threadIdx.x == 0) st_rel(gen, g);
  } else if (threadIdx.x == 0) {
    while (ld_acq(gen) != g) {
    }
  }
  if (threadIdx.x == 0) __threadfence();
  __syncthreads();
}

__global__ void k_gridsync_bench(int variant, int iters, unsigned* flags, unsigned* gen,
                                 unsigned* sink) {
  cooperative_groups::grid_group grid = cooperative_groups::this_grid();
  unsigned acc = 0;
  __shared__ unsigned sh[4];
  volatile unsigned* ctr = gen + 8;  // four level counters on one line
  for (int i = 0; i < iters; ++i) {
    if (variant == 1) flag_barrier(flags, gen, (unsigned)i + 1);
    else grid.sync();
    if (variant == 2) {  // every thread reads the counters (the level-end pattern)
      acc += ctr[0] + ctr[1] + ctr[2] + ctr[3];
    } else if (variant == 3) {  // thread 0 reads them, the block shares them
      if (threadIdx.x == 0)
        for (int k = 0; k < 4; ++k) sh[k] = ctr[k];
      __syncthreads();
      acc += sh[0] + sh[1] + sh[2] + sh[3];
      __syncthreads();
    }
    acc += flags[(blockIdx.x * 7 + i) % gridDim.x * 32];
  }
  if (acc == 0xdeadbeef) sink[0] = acc;
}

// same-address atomic throughput: every warp's lane 0 adds `iters` times to
// one counter (variant 0, with return value), to one counter without using
// the result (variant 1: RED), or to its own 128-byte line (variant 2)
__global__ void k_atomic_bench(int variant, int iters, unsigned long long* ctr,
                               unsigned long long* sink) {
  if ((threadIdx.x & 31) != 0) return;
  const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  unsigned long long acc = 0;
  for (int i = 0; i < iters; ++i) {
    if (variant == 0) acc += atomicAdd(ctr, 1ull);
    else if (variant == 1) atomicAdd(ctr, 1ull);
    else acc += atomicAdd(ctr + 16 * (wid & 1023), 1ull);
  }
  if (acc == 0xdeadbeefull) sink[0] = acc;
}

// dependent-load latency: one thread chases next = buf[next] through a
// random cyclic permutation of `span` words (stride-randomised), timing
// `iters` hops with clock64
__global__ void k_chase(const uint32_t* __restrict__ buf, int iters, long long* out,
                        uint32_t start) {
  uint32_t x = start;
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = buf[x];
  const long long t1 = clock64();
  out[0] = t1 - t0;
  out[1] = x;
}

}  // namespace gfx

using namespace gfx;

// cycles per dependent load over a chase buffer prepared by the caller
extern "C" int gfx_debug_chase(gfx_ctx* ctx, const uint32_t* buf_d, int iters, uint32_t start,
                               double* cycles_per_load) {
  GFX_REQUIRE(ctx && buf_d && cycles_per_load && iters > 0, "gfx_debug_chase: bad argument");
  GFX_CK(cudaSetDevice(ctx->device));
  long long* out = nullptr;
  GFX_CK(cudaMalloc(&out, 16));
  k_chase<<<1, 1, 0, ctx->stream>>>(buf_d, iters, out, start);  // warm (TLB, L2)
  k_chase<<<1, 1, 0, ctx->stream>>>(buf_d, iters, out, start);
  long long h[2];
  GFX_CK(cudaMemcpyAsync(h, out, 16, cudaMemcpyDeviceToHost, ctx->stream));
  GFX_CK(cudaStreamSynchronize(ctx->stream));
  GFX_CK(cudaFree(out));
  *cycles_per_load = (double)h[0] / iters;
  return GFX_OK;
}

extern "C" int gfx_debug_gridsync(gfx_ctx* ctx, int variant, int blocks, int threads, int iters,
                                  float* us_per_sync) {
  GFX_REQUIRE(ctx && us_per_sync && blocks > 0 && threads > 0, "gfx_debug_gridsync: bad argument");
  GFX_CK(cudaSetDevice(ctx->device));
  unsigned* buf = nullptr;
  GFX_CK(cudaMalloc(&buf, (size_t)(blocks + 2) * 32 * 4));
  GFX_CK(cudaMemset(buf, 0, (size_t)(blocks + 2) * 32 * 4));
  unsigned* flags = buf;
  unsigned* gen = buf + (size_t)blocks * 32;
  unsigned* sink = gen + 32;
  void* args[] = {&variant, &iters, &flags, &gen, &sink};
  int one = 1;
  void* args1[] = {&variant, &one, &flags, &gen, &sink};
  GFX_CK(cudaLaunchCooperativeKernel((const void*)k_gridsync_bench, dim3(blocks), dim3(threads),
                                     args1, 0, ctx->stream));
  GFX_CK(cudaMemsetAsync(buf, 0, (size_t)(blocks + 2) * 32 * 4, ctx->stream));
  GFX_CK(cudaEventRecord(ctx->ev0, ctx->stream));
  GFX_CK(cudaLaunchCooperativeKernel((const void*)k_gridsync_bench, dim3(blocks), dim3(threads),
                                     args, 0, ctx->stream));
  GFX_CK(cudaEventRecord(ctx->ev1, ctx->stream));
  GFX_CK(cudaEventSynchronize(ctx->ev1));
  float ms = 0.f;
  GFX_CK(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
  *us_per_sync = ms * 1000.f / iters;
  GFX_CK(cudaFree(buf));
  return GFX_OK;
}

// ns per atomic over `blocks` x 256 threads (one atomic per warp per iteration)
extern "C" int gfx_debug_atomics(gfx_ctx* ctx, int variant, int blocks, int iters,
                                 double* ns_per_atomic) {
  GFX_REQUIRE(ctx && ns_per_atomic && blocks > 0 && iters > 0, "gfx_debug_atomics: bad argument");
  GFX_CK(cudaSetDevice(ctx->device));
  unsigned long long* buf = nullptr;
  GFX_CK(cudaMalloc(&buf, (1024 * 16 + 16) * 8));
  GFX_CK(cudaMemsetAsync(buf, 0, (1024 * 16 + 16) * 8, ctx->stream));
  k_atomic_bench<<<blocks, 256, 0, ctx->stream>>>(variant, 1, buf, buf + 1024 * 16);
  GFX_CK(cudaEventRecord(ctx->ev0, ctx->stream));
  k_atomic_bench<<<blocks, 256, 0, ctx->stream>>>(variant, iters, buf, buf + 1024 * 16);
  GFX_CK(cudaEventRecord(ctx->ev1, ctx->stream));
  GFX_CK(cudaEventSynchronize(ctx->ev1));
  float ms = 0.f;
  GFX_CK(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
  *ns_per_atomic = ms * 1e6 / ((double)blocks * 8 * iters);
  GFX_CK(cudaFree(buf));
  return GFX_OK;
}

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
