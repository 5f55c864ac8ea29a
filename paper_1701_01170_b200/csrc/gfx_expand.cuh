// Load-balanced push expansion template (the device `advance`).
//
// Reference semantics: operators.py:218-266 (advance, push) with the LB plan
// of load_balance.py:157-176.  One CTA owns one tile of kTile consecutive
// OUTPUT slots of the frontier's expansion (tiles come from the fused degree
// scan, so hubs are split across many CTAs and every CTA does the same work).
//
// Per tile (in passes of <= kPassItems frontier items):
//   items : each thread loads one item's (scan, delta = row[v] - scan, v)
//           into shared memory and drops a marker at the item's first slot;
//   owner : a CTA-wide inclusive max-scan over the markers gives every slot
//           its owning item (load-balancing search without binary search);
//   visit : thread t handles slots t, t+B, ... (consecutive lanes read
//           consecutive column ids: coalesced), 4 slots in flight per thread,
//           col id = col[delta[item] + slot]; the functor decides emission;
//   emit  : emitted ids are staged in shared memory and appended with ONE
//           global atomicAdd per tile, then written coalesced.
//
// Functor interface (gfx_bfs.cu / gfx_sssp.cu / gfx_operators.cu):
//   static constexpr bool kWeights;    load w[e]
//   static constexpr bool kSrcVal;     per-item src_value(v)
//   static constexpr bool kEmitEdge;   emit edge ids instead of dst ids
//   __device__ int32_t src_value(int32_t v) const;
//   __device__ void prefetch(const int32_t d[kVisitBatch]);
//   __device__ bool visit(int u, int32_t dst, int32_t src, int32_t w,
//                         int32_t sval, int64_t edge);   // u = prefetch slot
#pragma once

#include "gfx_device.cuh"
#include "gfx_internal.cuh"

namespace gfx {

constexpr int kExpandBlock = 256;
constexpr int kPassItems = 1024;
constexpr int kSlotsPerThread = kTile / kExpandBlock;  // 16
constexpr int kVisitBatch = 8;  // slots (column loads) in flight per thread

struct ExpandSmem {
  int64_t delta[kPassItems];   // row[v] - scan[i]: col index = delta + global slot
  int32_t src[kPassItems];     // frontier id
  int32_t sval[kPassItems];    // functor per-source value
  int16_t owner[kTile];        // slot -> item (relative to the pass)
  int32_t obuf[kTile];         // emitted ids
  int32_t warp_max[kExpandBlock / 32];
  int cnt;
  unsigned long long gbase;
};

// All tiles t = cta, cta + ncta, ... of one expansion (S.cnt must be 0 on
// entry; it is 0 again on exit).  Shared by the standalone kernel and the
// persistent BFS kernel.
template <class Op>
__device__ __forceinline__ void expand_tiles(ExpandSmem& S, Op& o, const int32_t* __restrict__ F,
                                             int64_t nf, const int64_t* __restrict__ scan,
                                             const int64_t* __restrict__ rowbase,
                                             const int32_t* __restrict__ part, int64_t ntiles,
                                             int64_t total, const int32_t* __restrict__ col,
                                             const int32_t* __restrict__ wgt,
                                             int32_t* __restrict__ out,
                                             unsigned long long* __restrict__ out_len,
                                             int64_t cta, int64_t ncta) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int64_t t = cta; t < ntiles; t += ncta) {
    const int64_t s0 = t * kTile;
    const int64_t s1 = min(s0 + (int64_t)kTile, total);
    const int64_t i0 = part[t];
    const int64_t i1 = (t + 1 < ntiles) ? (int64_t)part[t + 1] : nf - 1;

    for (int64_t pa = i0; pa <= i1; pa += kPassItems) {
      const int64_t pb = min(pa + kPassItems - 1, i1);
      // slot range of this pass, clipped to the tile
      const int64_t sl = max(scan[pa], s0);
      const int64_t sh = min(scan[pb + 1], s1);
      const int nsl = (int)max(sh - sl, (int64_t)0);
      __syncthreads();  // previous pass / tile fully consumed
      for (int j = tid; j < nsl; j += kExpandBlock) S.owner[j] = -1;
      __syncthreads();
      for (int64_t i = pa + tid; i <= pb; i += kExpandBlock) {
        const int r = (int)(i - pa);
        const int64_t sc = scan[i], sc1 = scan[i + 1];
        const int32_t v = F[i];
        S.delta[r] = rowbase[i] - sc;
        S.src[r] = v;
        const int64_t lo = max(sc, sl), hi = min(sc1, sh);
        if (hi > lo) {
          S.owner[lo - sl] = (int16_t)r;
          if (Op::kSrcVal) S.sval[r] = o.src_value(v);
        }
      }
      __syncthreads();
      // inclusive max-scan of owner[0..nsl): kSlotsPerThread consecutive per thread
      {
        int16_t loc[kSlotsPerThread];
        const int base = tid * kSlotsPerThread;
        int run = -1;
#pragma unroll
        for (int k = 0; k < kSlotsPerThread; ++k) {
          const int j = base + k;
          const int x = j < nsl ? S.owner[j] : -1;
          run = x > run ? x : run;
          loc[k] = (int16_t)run;
        }
        int incl = run;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, off);
          if (lane >= off) incl = y > incl ? y : incl;
        }
        if (lane == 31) S.warp_max[warp] = incl;
        int excl = __shfl_up_sync(0xffffffffu, incl, 1);
        if (lane == 0) excl = -1;
        __syncthreads();
        int wpre = -1;
        for (int w = 0; w < warp; ++w) wpre = S.warp_max[w] > wpre ? S.warp_max[w] : wpre;
        const int pre = wpre > excl ? wpre : excl;
#pragma unroll
        for (int k = 0; k < kSlotsPerThread; ++k) {
          const int j = base + k;
          if (j < nsl) S.owner[j] = (int16_t)(loc[k] > pre ? loc[k] : pre);
        }
      }
      __syncthreads();

      // ---- visit: kVisitBatch slots in flight per thread
      for (int jb = 0; jb < nsl; jb += kExpandBlock * kVisitBatch) {
        int32_t d[kVisitBatch], it[kVisitBatch], w[kVisitBatch];
        int64_t e[kVisitBatch];
#pragma unroll
        for (int u = 0; u < kVisitBatch; ++u) {
          const int j = jb + u * kExpandBlock + tid;
          it[u] = j < nsl ? S.owner[j] : -1;
          e[u] = it[u] >= 0 ? S.delta[it[u]] + sl + j : 0;
        }
#pragma unroll
        for (int u = 0; u < kVisitBatch; ++u) {
          d[u] = it[u] >= 0 ? ld_stream_i32(col + e[u]) : -1;
          if (Op::kWeights) w[u] = it[u] >= 0 ? ld_stream_i32(wgt + e[u]) : 0;
        }
        o.prefetch(d);
#pragma unroll
        for (int u = 0; u < kVisitBatch; ++u) {
          bool emit = false;
          if (d[u] >= 0) {
            const int32_t sv = Op::kSrcVal ? S.sval[it[u]] : 0;
            emit = o.visit(u, d[u], S.src[it[u]], Op::kWeights ? w[u] : 1, sv, e[u]);
          }
          const unsigned wm = __ballot_sync(0xffffffffu, emit);
          if (wm) {
            int b = 0;
            if (lane == 0) b = atomicAdd(&S.cnt, __popc(wm));
            b = __shfl_sync(0xffffffffu, b, 0);
            if (emit)
              S.obuf[b + __popc(wm & ((1u << lane) - 1))] =
                  Op::kEmitEdge ? (int32_t)e[u] : d[u];
          }
        }
      }
    }
    __syncthreads();
    const int cnt = S.cnt;
    if (cnt > 0) {
      if (tid == 0) S.gbase = atomicAdd(out_len, (unsigned long long)cnt);
      __syncthreads();
      const unsigned long long gb = S.gbase;
      for (int j = tid; j < cnt; j += kExpandBlock) out[gb + j] = S.obuf[j];
      __syncthreads();
      if (tid == 0) S.cnt = 0;
    }
  }
  __syncthreads();
}

template <class Op>
__global__ void __launch_bounds__(kExpandBlock)
    k_lb_expand(const int32_t* __restrict__ F, const unsigned long long* __restrict__ nf_d,
                const int64_t* __restrict__ scan, const int64_t* __restrict__ rowbase,
                const int32_t* __restrict__ part, const Counters* __restrict__ plan,
                const int32_t* __restrict__ col, const int32_t* __restrict__ wgt, Op op,
                int32_t* __restrict__ out, unsigned long long* __restrict__ out_len) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  ExpandSmem& S = *reinterpret_cast<ExpandSmem*>(smem_raw);
  if (threadIdx.x == 0) S.cnt = 0;
  __syncthreads();
  Op o = op;  // mutable copy: functors keep per-thread prefetch registers
  expand_tiles(S, o, F, (int64_t)*nf_d, scan, rowbase, part, (int64_t)plan->ntiles,
               (int64_t)plan->total, col, wgt, out, out_len, blockIdx.x, gridDim.x);
}

template <class Op>
constexpr int expand_smem_bytes() {
  return (int)sizeof(ExpandSmem);
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

// CTAs per SM that fit the shared-memory footprint
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
  GFX_LAUNCH((k_lb_expand<Op>), grid, kExpandBlock, expand_smem_bytes<Op>(), ctx->stream, F,
             nf_d, scan, rowbase, part, plan_ctr, g->col, g->w, op, out, out_len);
  GFX_CK(cudaGetLastError());
  return GFX_OK;
}

}  // namespace gfx
