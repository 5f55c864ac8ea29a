// Load-balanced push expansion template (the device `advance`).
//
// Reference semantics: operators.py:218-266 (advance, push) with the LB plan
// of load_balance.py:157-176.  One CTA owns one tile of kTile consecutive
// OUTPUT slots of the frontier's expansion (tiles come from the fused degree
// scan, so hubs are split across many CTAs and every CTA does the same work).
//
//   stage : warps copy every adjacency segment overlapping the tile into
//           shared memory with coalesced 4-byte cp.async (LDGSTS), plus the
//           owning source id (and weights / a per-source value when the
//           functor needs them);
//   visit : each thread walks slots j, j+B, ... of the tile and calls the
//           functor; it returns whether the slot's output id is emitted;
//   emit  : emitted ids are staged in shared memory and appended with ONE
//           global atomicAdd per tile, then written coalesced.
//
// Functor interface (see gfx_bfs.cu / gfx_sssp.cu / gfx_operators.cu):
//   static constexpr bool kWeights;    stage w[e]
//   static constexpr bool kSrcVal;     stage src_value(v) per slot
//   static constexpr bool kEmitEdge;   emit edge ids instead of dst ids
//   __device__ int32_t src_value(int32_t v) const;
//   __device__ void prefetch(const int32_t d[4]);   // issue loads for 4 slots
//   __device__ bool visit(int u, int32_t dst, int32_t src, int32_t w,
//                         int32_t sval, int64_t edge);  // u = slot of prefetch
#pragma once

#include "gfx_device.cuh"
#include "gfx_internal.cuh"

namespace gfx {

constexpr int kExpandBlock = 256;

template <class Op>
constexpr int expand_smem_bytes() {
  return kTile * 4 * (3 + (Op::kWeights ? 1 : 0) + (Op::kSrcVal ? 1 : 0) + (Op::kEmitEdge ? 1 : 0));
}

template <class Op>
__global__ void __launch_bounds__(kExpandBlock)
    k_lb_expand(const int32_t* __restrict__ F, const unsigned long long* __restrict__ nf_d,
                const int64_t* __restrict__ scan, const int64_t* __restrict__ rowbase,
                const int32_t* __restrict__ part, const Counters* __restrict__ plan,
                const int32_t* __restrict__ col, const int32_t* __restrict__ wgt, Op op,
                int32_t* __restrict__ out, unsigned long long* __restrict__ out_len) {
  extern __shared__ int32_t smem[];
  int32_t* buf = smem;               // [kTile] destination ids
  int32_t* owner = smem + kTile;     // [kTile] source ids
  int32_t* obuf = smem + 2 * kTile;  // [kTile] emitted ids
  int32_t* extra = smem + 3 * kTile;
  int32_t* wbuf = Op::kWeights ? extra : nullptr;
  if (Op::kWeights) extra += kTile;
  int32_t* sval = Op::kSrcVal ? extra : nullptr;
  if (Op::kSrcVal) extra += kTile;
  int32_t* ebuf = Op::kEmitEdge ? extra : nullptr;  // low 32 bits of edge ids (E kinds)
  __shared__ int s_cnt;
  __shared__ unsigned long long s_gbase;

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t ntiles = (int64_t)plan->ntiles;
  const int64_t total = (int64_t)plan->total;
  const int64_t nf = (int64_t)*nf_d;
  if (threadIdx.x == 0) s_cnt = 0;
  __syncthreads();
  Op o = op;  // mutable copy: functors keep per-thread prefetch registers

  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t s0 = t * kTile;
    const int64_t s1 = min(s0 + (int64_t)kTile, total);
    const int64_t i0 = part[t];
    const int64_t i1 = (t + 1 < ntiles) ? (int64_t)part[t + 1] : nf - 1;

    // ---- stage
    for (int64_t ib = i0 + (int64_t)warp * 32; ib <= i1; ib += kExpandBlock) {
      const int64_t i = ib + lane;
      int64_t lo = 0, len = 0, src_base = 0;
      int32_t v = 0, sv = 0;
      if (i <= i1) {
        const int64_t sc = scan[i], sc1 = scan[i + 1];
        lo = max(sc, s0);
        const int64_t hi = min(sc1, s1);
        len = hi > lo ? hi - lo : 0;
        src_base = rowbase[i] + (lo - sc);
        v = F[i];
        if (Op::kSrcVal && len > 0) sv = o.src_value(v);
      }
      unsigned mask = __ballot_sync(0xffffffffu, len > 0);
      while (mask) {
        const int k = __ffs(mask) - 1;
        mask &= mask - 1;
        const int klo = (int)(__shfl_sync(0xffffffffu, lo, k) - s0);
        const int klen = (int)__shfl_sync(0xffffffffu, len, k);
        const int64_t kbase = __shfl_sync(0xffffffffu, src_base, k);
        const int32_t kv = __shfl_sync(0xffffffffu, v, k);
        const int32_t ksv = Op::kSrcVal ? __shfl_sync(0xffffffffu, sv, k) : 0;
        for (int j = lane; j < klen; j += 32) {
          cp_async4(&buf[klo + j], &col[kbase + j]);
          if (Op::kWeights) cp_async4(&wbuf[klo + j], &wgt[kbase + j]);
          owner[klo + j] = kv;
          if (Op::kSrcVal) sval[klo + j] = ksv;
          if (Op::kEmitEdge) ebuf[klo + j] = (int32_t)(kbase + j);
        }
      }
    }
    cp_async_wait_all();
    __syncthreads();

    // ---- visit (4 slots in flight per thread)
    const int nslots = (int)(s1 - s0);
    for (int jb = 0; jb < nslots; jb += kExpandBlock * 4) {
      int32_t d[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int j = jb + u * kExpandBlock + threadIdx.x;
        d[u] = j < nslots ? buf[j] : -1;
      }
      o.prefetch(d);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int j = jb + u * kExpandBlock + threadIdx.x;
        bool emit = false;
        int32_t outv = 0;
        if (d[u] >= 0) {
          const int32_t w = Op::kWeights ? wbuf[j] : 1;
          const int32_t sv = Op::kSrcVal ? sval[j] : 0;
          const int64_t edge = Op::kEmitEdge ? (int64_t)(uint32_t)ebuf[j] : 0;
          emit = o.visit(u, d[u], owner[j], w, sv, edge);
          outv = Op::kEmitEdge ? ebuf[j] : d[u];
        }
        const unsigned wm = __ballot_sync(0xffffffffu, emit);
        if (wm) {
          int base = 0;
          if (lane == 0) base = atomicAdd(&s_cnt, __popc(wm));
          base = __shfl_sync(0xffffffffu, base, 0);
          if (emit) obuf[base + __popc(wm & ((1u << lane) - 1))] = outv;
        }
      }
    }
    __syncthreads();
    const int cnt = s_cnt;
    if (cnt > 0) {
      if (threadIdx.x == 0) s_gbase = atomicAdd(out_len, (unsigned long long)cnt);
      __syncthreads();
      const unsigned long long gb = s_gbase;
      for (int j = threadIdx.x; j < cnt; j += kExpandBlock) out[gb + j] = obuf[j];
    }
    __syncthreads();
    if (threadIdx.x == 0) s_cnt = 0;
    __syncthreads();
  }
}

template <class Op>
int set_expand_smem() {
  static bool done = false;
  if (done) return GFX_OK;
  GFX_CK(cudaFuncSetAttribute(k_lb_expand<Op>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              expand_smem_bytes<Op>()));
  done = true;
  return GFX_OK;
}

// CTAs per SM that fit the functor's shared-memory footprint
template <class Op>
inline int expand_ctas_per_sm() {
  const int per = expand_smem_bytes<Op>() + 1024;
  int k = (227 * 1024) / per;
  return k < 1 ? 1 : (k > 8 ? 8 : k);
}

// scan + expand over queue F (size at *nf_d), emitting into out / *out_len
template <class Op>
int lb_advance(gfx_graph* g, const int32_t* F, const unsigned long long* nf_d, int64_t nf_max,
               Counters* plan_ctr, int64_t* scan, int64_t* rowbase, int32_t* part, const Op& op,
               int32_t* out, unsigned long long* out_len) {
  gfx_ctx* ctx = g->ctx;
  GFX_TRY(launch_degree_scan(g, F, nf_d, nf_max, g->row, scan, rowbase, part, plan_ctr));
  GFX_TRY(set_expand_smem<Op>());
  const int grid = ctx->sm_count * expand_ctas_per_sm<Op>();
  GFX_LAUNCH((k_lb_expand<Op>), grid, kExpandBlock, expand_smem_bytes<Op>(), ctx->stream, 
      F, nf_d, scan, rowbase, part, plan_ctr, g->col, g->w, op, out, out_len);
  GFX_CK(cudaGetLastError());
  return GFX_OK;
}

}  // namespace gfx
