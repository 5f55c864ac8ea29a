// Generic operators with the closed device-functor registry.
//
// Reference: operators.py:218-266 (advance), :269-307 (pull_expand), :360-384
// (filter_frontier), :392-456 (advance_filter_fused), :485-525
// (segmented_intersect), :528-533 (compute).  The reference takes arbitrary
// Python callables over whole id arrays; here the functors the six primitives
// pass (SURVEY 8(b) functor table) are a closed registry (include/gfx.h
// GFX_FN_*) that runs fused inside the load-balanced warp-tile expansion of
// the primitives.  Arbitrary callables take the staged path (gfx_opgen.cu).
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <cuda_runtime.h>

#include "gfx_device.cuh"
#include "gfx_expand.cuh"
#include "gfx_internal.cuh"

namespace gfx {

// relax passes of GFX_FN_SSSP_RELAX (see run_advance)
enum RelaxPass : int { kRelaxNone = 0, kRelaxMin = 1, kRelaxWin = 2 };

// one registry functor with its bound arrays
struct RegFn {
  int fid;
  int32_t* labels;
  int32_t* preds;
  int32_t value;
  double* f0;
  double* f1;
  double scalar;
};

__host__ inline RegFn make_fn(int fid, const gfx_functor_args* a) {
  RegFn f{fid, nullptr, nullptr, 0, nullptr, nullptr, 0.0};
  if (a) {
    f.labels = a->labels_d;
    f.preds = a->preds_d;
    f.value = (int32_t)a->value;
    f.f0 = a->f0_d;
    f.f1 = a->f1_d;
    f.scalar = a->scalar;
  }
  return f;
}

// vertex_cond functors (filter / fused image test); x is a vertex id, or an
// edge id for GFX_FN_CC_SAME_COMP
__device__ __forceinline__ bool vertex_cond(const RegFn& f, int64_t x, const int64_t* row,
                                            const int32_t* col, int64_t n) {
  switch (f.fid) {
    case GFX_FN_NONE:
      return true;
    case GFX_FN_LABEL_EQ:
    case GFX_FN_SSSP_STAMP:
      return f.labels[x] == f.value;
    case GFX_FN_LABEL_NE:
      return f.labels[x] != f.value;
    case GFX_FN_PR_MOVED:
      return fabs(f.f1[x] - f.f0[x]) >= f.scalar;
    case GFX_FN_CC_SAME_COMP: {  // comp[edge_sources[e]] != comp[col[e]]
      int64_t lo = 0, hi = n;    // largest v with row[v] <= e
      while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (row[mid] <= x) lo = mid;
        else hi = mid;
      }
      return f.labels[lo] != f.labels[col[x]];
    }
    default:
      return false;
  }
}

template <bool EMIT_EDGE, bool WEIGHTS>
struct RegistryOp {
  static constexpr bool kWeights = WEIGHTS, kSrcVal = false, kEmitEdge = EMIT_EDGE;
  static constexpr int kBatch = 4;
  static constexpr int kMinBlocks = 2;
  RegFn f;
  int pass;               // RelaxPass for GFX_FN_SSSP_RELAX
  const int32_t* pre;     // pre-call label snapshot (relax passes)
  const int64_t* row;
  const int32_t* col;
  int64_t n;
  RegFn vf;               // fused: vertex_cond on the image
  uint32_t* seen;         // fused: cull bitmap over the output domain (nullable)
  __device__ int32_t src_value(int32_t) const { return 0; }
  __device__ void prefetch(const int32_t*) {}

  __device__ bool cond(int32_t d, int32_t s, int32_t w) {
    switch (f.fid) {
      case GFX_FN_NONE:
        return true;
      case GFX_FN_BFS_CLAIM:  // compare_and_swap(labels, d, UNVISITED, depth) + preds[d] = s
      case GFX_FN_BC_CLAIM: {
        if (f.labels[d] != GFX_UNVISITED) return false;
        if (atomicCAS(&f.labels[d], GFX_UNVISITED, f.value) != GFX_UNVISITED) return false;
        if (f.preds) f.preds[d] = s;
        return true;
      }
      case GFX_FN_BFS_IDEMP: {  // labels[d] == UNVISITED; _set_depth (duplicates allowed)
        if (f.labels[d] != GFX_UNVISITED) return false;
        f.labels[d] = f.value;
        if (f.preds) f.preds[d] = s;
        return true;
      }
      case GFX_FN_SSSP_RELAX: {
        // values = pre[s] + w (pre-call snapshot, so both passes agree);
        // pass 1 lowers labels[d]; pass 2 reports the atomic_min winners --
        // strictly below the pre-call value AND equal to the post-call
        // minimum (operators.py:111-124) -- and only they set preds
        const int32_t ls = pre[s];
        if (ls == GFX_UNVISITED) return false;
        const int32_t nd = ls + w;
        if (nd >= pre[d]) return false;
        if (pass == kRelaxMin) {
          if (nd < f.labels[d]) atomicMin(&f.labels[d], nd);
          return false;
        }
        if (nd != f.labels[d]) return false;
        if (f.preds) f.preds[d] = s;
        return true;
      }
      case GFX_FN_TC_ORIENT: {  // deg[s] > deg[d] or (== and s < d)
        const int64_t ds = row[s + 1] - row[s], dd = row[d + 1] - row[d];
        return ds > dd || (ds == dd && s < d);
      }
      case GFX_FN_LABEL_EQ:
        return f.labels[d] == f.value;
      case GFX_FN_LABEL_NE:
        return f.labels[d] != f.value;
      case GFX_FN_BC_SIGMA:  // labels[d] == depth; sigma[d] += sigma[s]
        if (f.labels[d] != f.value) return false;
        atomicAdd(&f.f0[d], f.f0[s]);
        return true;
      case GFX_FN_BC_DELTA:  // labels[d] == lvl + 1; delta[s] += sigma[s]/sigma[d]*(1+delta[d])
        if (f.labels[d] != f.value) return false;
        atomicAdd(&f.f1[s], f.f0[s] / f.f0[d] * (1.0 + f.f1[d]));
        return true;
      case GFX_FN_PR_SCATTER: {  // rank_next[d] += damping * rank[s] / outdeg[s]
        const double od = (double)(row[s + 1] - row[s]);
        atomicAdd(&f.f1[d], f.scalar * f.f0[s] / od);
        return true;
      }
      default:
        return false;
    }
  }

  __device__ bool visit(int, int32_t d, int32_t s, int32_t w, int32_t, int64_t edge) {
    if (!cond(d, s, w)) return false;
    const int64_t x = EMIT_EDGE ? edge : (int64_t)d;
    if (vf.fid != GFX_FN_NONE && !vertex_cond(vf, x, row, col, n)) return false;
    if (seen) {
      const uint32_t bit = 1u << (x & 31);
      if (seen[x >> 5] & bit) return false;
      if (atomicOr(&seen[x >> 5], bit) & bit) return false;
    }
    return true;
  }
};

__global__ void k_edge_targets(const int32_t* __restrict__ edges, int64_t n,
                               const int32_t* __restrict__ col, int32_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = col[edges[i]];
}

// filter: mark survivors in a bitmap over the id domain
__global__ void k_filter_mark(const int32_t* __restrict__ in, int64_t n, RegFn f,
                              const int64_t* __restrict__ row, const int32_t* __restrict__ col,
                              int64_t nv, uint32_t* __restrict__ bm) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = in[i];
    if (vertex_cond(f, v, row, col, nv)) atomicOr(&bm[v >> 5], 1u << (v & 31));
  }
}

__global__ void k_vertex_mask(const int32_t* __restrict__ in, int64_t n, RegFn f,
                              const int64_t* __restrict__ row, const int32_t* __restrict__ col,
                              int64_t nv, uint8_t* __restrict__ mask) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    mask[i] = vertex_cond(f, in[i], row, col, nv);
}

__global__ void k_word_popc(const uint32_t* __restrict__ bm, int64_t words,
                            int64_t* __restrict__ cnt) {
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < words;
       w += (int64_t)gridDim.x * blockDim.x)
    cnt[w] = __popc(bm[w]);
}

// ordered (ascending) bitmap -> id list
__global__ void k_word_emit(const uint32_t* __restrict__ bm, int64_t words,
                            const int64_t* __restrict__ off, int32_t* __restrict__ out) {
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < words;
       w += (int64_t)gridDim.x * blockDim.x) {
    uint32_t x = bm[w];
    int64_t k = off[w];
    while (x) {
      const int b = __ffs(x) - 1;
      x &= x - 1;
      out[k++] = (int32_t)(w * 32 + b);
    }
  }
}

__global__ void k_compute(const int32_t* __restrict__ in, int64_t n, int fid,
                          int32_t* __restrict__ labels, int64_t* __restrict__ acc, int64_t value) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = in[i];
    if (fid == GFX_FN_SET_LABEL) labels[v] = (int32_t)value;
    else if (fid == GFX_FN_ADD_I64) atomicAdd((unsigned long long*)&acc[v], (unsigned long long)value);
  }
}

// pull probe, one warp per unvisited vertex: 32 in-neighbours per step,
// ballot, stop at the first hit (the lowest reverse slot wins, i.e. the
// sequential ascending early exit of SURVEY 8(d))
__global__ void k_pull_probe(const int32_t* __restrict__ U, int64_t nu,
                             const int64_t* __restrict__ rrow, const int32_t* __restrict__ rcol,
                             RegFn f, uint8_t* __restrict__ hit,
                             unsigned long long* __restrict__ probes) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  unsigned long long my_probes = 0;
  for (int64_t i = gw; i < nu; i += nw) {
    const int32_t u = U[i];
    const int64_t b = rrow[u], e = rrow[u + 1];
    int32_t found = -1;
    int64_t used = e - b;
    for (int64_t j = b; j < e; j += 32) {
      bool ok = false;
      int32_t s = -1;
      if (j + lane < e) {
        s = rcol[j + lane];
        ok = f.labels[s] == f.value - 1;  // BFS_PULL cond labels[s] == depth - 1
      }
      const unsigned m = __ballot_sync(0xffffffffu, ok);
      if (m) {
        const int k = __ffs(m) - 1;
        found = __shfl_sync(0xffffffffu, s, k);
        used = j - b + k + 1;
        break;
      }
    }
    if (lane == 0) {
      hit[i] = found >= 0;
      if (found >= 0) {  // _set_depth
        f.labels[u] = f.value;
        if (f.preds) f.preds[u] = found;
      }
      my_probes += (unsigned long long)used;
    }
  }
  if (lane == 0 && my_probes) atomicAdd(probes, my_probes);
}

__global__ void k_flags_invert(const uint8_t* __restrict__ in, int64_t n, uint8_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = !in[i];
}

// ordered intersection lists: thread per pair, merge in ascending order
__global__ void k_intersect_list(const int32_t* __restrict__ us, const int32_t* __restrict__ vs,
                                 int64_t npairs, const int64_t* __restrict__ rows,
                                 const int32_t* __restrict__ cols, const int64_t* __restrict__ off,
                                 int32_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npairs;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = rows[us[i]], ae = rows[us[i] + 1], b = rows[vs[i]], be = rows[vs[i] + 1];
    int64_t k = off[i];
    while (a < ae && b < be) {
      const int32_t x = cols[a], y = cols[b];
      if (x == y) out[k++] = x;
      a += (x <= y);
      b += (y <= x);
    }
  }
}

template <bool E, bool W>
static int run_advance(gfx_graph* g, const int32_t* F, int64_t nin, const RegFn& f,
                       const RegFn& vf, uint32_t* seen, int32_t* out, int64_t cap,
                       int64_t* nout, int64_t* edges) {
  gfx_ctx* ctx = g->ctx;
  int32_t* part;
  int64_t *scan, *rowbase;
  GFX_TRY(scratch_t(g, "q_scan", nin + 2, &scan));
  GFX_TRY(scratch_t(g, "q_rowbase", nin + 1, &rowbase));
  GFX_TRY(scratch_t(g, "q_part", part_capacity(g->m, nin), &part));
  Counters* C = g->counters;
  auto* pin = static_cast<Counters*>(ctx->pinned);
  GFX_CK(cudaMemsetAsync(C, 0, 2 * sizeof(Counters), ctx->stream));
  const unsigned long long nn = (unsigned long long)nin;
  GFX_CK(cudaMemcpyAsync(&C[0].out_len, &nn, 8, cudaMemcpyHostToDevice, ctx->stream));
  GFX_TRY(launch_degree_scan(g, F, &C[0].out_len, nin, g->row, scan, rowbase, part, &C[1]));
  GFX_CK(cudaMemcpyAsync(pin, &C[1], sizeof(Counters), cudaMemcpyDeviceToHost, ctx->stream));
  GFX_CK(cudaStreamSynchronize(ctx->stream));
  const int64_t total = (int64_t)pin->total;
  GFX_REQUIRE(total <= cap, "advance output capacity %lld < expansion size %lld", (long long)cap,
              (long long)total);
  GFX_REQUIRE(!E || g->m < (int64_t)INT32_MAX, "edge-id output needs m < 2^31");
  using Op = RegistryOp<E, W>;
  Op op{f, kRelaxNone, nullptr, g->row, g->col, g->n, vf, seen};
  GFX_TRY(set_expand_smem<Op>());
  const int grid = ctx->sm_count * 2;
  if (f.fid == GFX_FN_SSSP_RELAX) {
    // pass 1 (scatter-min) and pass 2 (winners) over the same plan, both
    // reading the pre-call snapshot
    int32_t* pre;
    GFX_TRY(scratch_t(g, "op_relax_pre", g->n + 1, &pre));
    GFX_CK(cudaMemcpyAsync(pre, f.labels, g->n * sizeof(int32_t), cudaMemcpyDeviceToDevice,
                           ctx->stream));
    op.pre = pre;
    op.pass = kRelaxMin;
    GFX_LAUNCH((k_lb_expand<Op>), grid, kExpandBlock, expand_smem_bytes(), ctx->stream, F,
               &C[0].out_len, scan, rowbase, part, &C[1], g->col, g->w, op, out, &C[1].out_len);
    op.pass = kRelaxWin;
  }
  GFX_LAUNCH((k_lb_expand<Op>), grid, kExpandBlock, expand_smem_bytes(), ctx->stream, F,
             &C[0].out_len, scan, rowbase, part, &C[1], g->col, g->w, op, out, &C[1].out_len);
  GFX_CK(cudaGetLastError());
  GFX_CK(cudaMemcpyAsync(pin, &C[1], sizeof(Counters), cudaMemcpyDeviceToHost, ctx->stream));
  GFX_CK(cudaStreamSynchronize(ctx->stream));
  *nout = (int64_t)pin->out_len;
  if (edges) *edges = total;
  return GFX_OK;
}

static bool is_advance_fn(int fid) {
  switch (fid) {
    case GFX_FN_NONE: case GFX_FN_BFS_CLAIM: case GFX_FN_BFS_IDEMP: case GFX_FN_SSSP_RELAX:
    case GFX_FN_TC_ORIENT: case GFX_FN_LABEL_EQ: case GFX_FN_LABEL_NE: case GFX_FN_BC_CLAIM:
    case GFX_FN_BC_SIGMA: case GFX_FN_BC_DELTA: case GFX_FN_PR_SCATTER:
      return true;
    default:
      return false;
  }
}

static bool is_vertex_fn(int fid) {
  switch (fid) {
    case GFX_FN_NONE: case GFX_FN_LABEL_EQ: case GFX_FN_LABEL_NE: case GFX_FN_PR_MOVED:
    case GFX_FN_CC_SAME_COMP: case GFX_FN_SSSP_STAMP:
      return true;
    default:
      return false;
  }
}

static int check_fn_args(gfx_graph* g, const RegFn& f) {
  switch (f.fid) {
    case GFX_FN_NONE: case GFX_FN_TC_ORIENT:
      return GFX_OK;
    case GFX_FN_SSSP_RELAX:
      GFX_REQUIRE(g->w, "SSSP relax needs edge weights");
      GFX_REQUIRE(f.labels, "functor %d needs labels", f.fid);
      return GFX_OK;
    case GFX_FN_BC_SIGMA:
      GFX_REQUIRE(f.labels && f.f0, "BC_SIGMA needs labels and sigma");
      return GFX_OK;
    case GFX_FN_BC_DELTA:
      GFX_REQUIRE(f.labels && f.f0 && f.f1, "BC_DELTA needs labels, sigma and delta");
      return GFX_OK;
    case GFX_FN_PR_SCATTER: case GFX_FN_PR_MOVED:
      GFX_REQUIRE(f.f0 && f.f1, "functor %d needs rank and rank_next", f.fid);
      return GFX_OK;
    default:
      GFX_REQUIRE(f.labels, "functor %d needs labels", f.fid);
      return GFX_OK;
  }
}

// edge frontiers expand the edge's destination (load_balance.py:94-102)
static int expansion_items(gfx_graph* g, const int32_t* fin, int64_t nin, int kind,
                           const int32_t** F) {
  *F = fin;
  if (kind == GFX_KIND_E2V || kind == GFX_KIND_E2E) {
    int32_t* tgt = nullptr;
    GFX_TRY(scratch_t(g, "op_targets", nin + 1, &tgt));
    GFX_LAUNCH(k_edge_targets, grid_for(nin, 256, g->ctx->sm_count * 8), 256, 0, g->ctx->stream,
               fin, nin, g->col, tgt);
    *F = tgt;
  }
  return GFX_OK;
}

static int dispatch_advance(gfx_graph* g, const int32_t* F, int64_t nin, int kind,
                            const RegFn& f, const RegFn& vf, uint32_t* seen, int32_t* out,
                            int64_t cap, int64_t* nout, int64_t* edges) {
  const bool emit_edge = kind == GFX_KIND_V2E || kind == GFX_KIND_E2E;
  const bool weights = f.fid == GFX_FN_SSSP_RELAX;
  if (emit_edge)
    return weights ? run_advance<true, true>(g, F, nin, f, vf, seen, out, cap, nout, edges)
                   : run_advance<true, false>(g, F, nin, f, vf, seen, out, cap, nout, edges);
  return weights ? run_advance<false, true>(g, F, nin, f, vf, seen, out, cap, nout, edges)
                 : run_advance<false, false>(g, F, nin, f, vf, seen, out, cap, nout, edges);
}

static int select_flagged(gfx_graph* g, const int32_t* in, const uint8_t* flags, int64_t n,
                          int32_t* out, int64_t* nsel, const char* tag) {
  gfx_ctx* ctx = g->ctx;
  int64_t* cnt;
  GFX_TRY(scratch_t(g, "op_sel_cnt", 2, &cnt));
  size_t tb = 0;
  GFX_CK(cub::DeviceSelect::Flagged(nullptr, tb, in, flags, out, cnt, n, ctx->stream));
  void* tmp = nullptr;
  GFX_TRY(scratch(g, tag, tb + 16, &tmp));
  GFX_CK(cub::DeviceSelect::Flagged(tmp, tb, in, flags, out, cnt, n, ctx->stream));
  count_launch();
  GFX_CK(cudaMemcpyAsync(nsel, cnt, 8, cudaMemcpyDeviceToHost, ctx->stream));
  return GFX_OK;
}

}  // namespace gfx

using namespace gfx;

extern "C" {

int gfx_advance(gfx_graph* g, const int32_t* fin_d, int64_t nin, int kind, int functor_id,
                const gfx_functor_args* args, int32_t* fout_d, int64_t fout_cap, int64_t* nout,
                int64_t* edges) {
  GFX_NVTX("gfx_advance");
  GFX_REQUIRE(g && nout && (nin == 0 || (fin_d && fout_d)), "gfx_advance: null argument");
  GFX_REQUIRE(kind >= GFX_KIND_V2V && kind <= GFX_KIND_E2E, "unknown advance kind %d", kind);
  GFX_REQUIRE(is_advance_fn(functor_id), "functor %d is not an advance functor of the registry",
              functor_id);
  const RegFn f = make_fn(functor_id, args);
  GFX_TRY(check_fn_args(g, f));
  GFX_CK(cudaSetDevice(g->ctx->device));
  *nout = 0;
  if (edges) *edges = 0;
  if (nin == 0) return GFX_OK;
  const int32_t* F;
  GFX_TRY(expansion_items(g, fin_d, nin, kind, &F));
  return dispatch_advance(g, F, nin, kind, f, make_fn(GFX_FN_NONE, nullptr), nullptr, fout_d,
                          fout_cap, nout, edges);
}

int gfx_advance_fused(gfx_graph* g, const int32_t* fin_d, int64_t nin, int kind, int cond_id,
                      const gfx_functor_args* cond_args, int vcond_id,
                      const gfx_functor_args* vcond_args, int32_t* fout_d, int64_t fout_cap,
                      int64_t* nout, int64_t* edges) {
  GFX_NVTX("gfx_advance_fused");
  GFX_REQUIRE(g && nout && (nin == 0 || (fin_d && fout_d)), "gfx_advance_fused: null argument");
  GFX_REQUIRE(kind >= GFX_KIND_V2V && kind <= GFX_KIND_E2E, "unknown advance kind %d", kind);
  GFX_REQUIRE(is_advance_fn(cond_id) && cond_id != GFX_FN_SSSP_RELAX,
              "functor %d is not a fused-advance functor of the registry", cond_id);
  GFX_REQUIRE(is_vertex_fn(vcond_id) && vcond_id != GFX_FN_CC_SAME_COMP,
              "functor %d is not a vertex functor of the registry", vcond_id);
  const RegFn f = make_fn(cond_id, cond_args), vf = make_fn(vcond_id, vcond_args);
  GFX_TRY(check_fn_args(g, f));
  GFX_TRY(check_fn_args(g, vf));
  gfx_ctx* ctx = g->ctx;
  GFX_CK(cudaSetDevice(ctx->device));
  *nout = 0;
  if (edges) *edges = 0;
  if (nin == 0) return GFX_OK;
  const bool emit_edge = kind == GFX_KIND_V2E || kind == GFX_KIND_E2E;
  const int64_t domain = emit_edge ? g->m : g->n;
  const int64_t words = (domain + 31) / 32 + 1;
  uint32_t* seen;
  GFX_TRY(scratch_t(g, "op_fused_seen", words, &seen));
  GFX_CK(cudaMemsetAsync(seen, 0, words * 4, ctx->stream));
  const int32_t* F;
  GFX_TRY(expansion_items(g, fin_d, nin, kind, &F));
  return dispatch_advance(g, F, nin, kind, f, vf, seen, fout_d, fout_cap, nout, edges);
}

int gfx_pull_advance(gfx_graph* g, const int32_t* fin_d, int64_t nin, int functor_id,
                     const gfx_functor_args* args, int32_t* active_d, int64_t* nactive,
                     int32_t* rest_d, int64_t* nrest, int64_t* edges) {
  GFX_NVTX("gfx_pull_advance");
  GFX_REQUIRE(g && nactive && nrest && (nin == 0 || (fin_d && active_d && rest_d)),
              "gfx_pull_advance: null argument");
  GFX_REQUIRE(functor_id == GFX_FN_BFS_PULL, "functor %d is not a pull functor of the registry",
              functor_id);
  GFX_REQUIRE(args && args->labels_d, "BFS_PULL needs labels");
  GFX_REQUIRE(g->rrow && g->rcol, "pull advance needs the reverse adjacency");
  gfx_ctx* ctx = g->ctx;
  GFX_CK(cudaSetDevice(ctx->device));
  *nactive = *nrest = 0;
  if (edges) *edges = 0;
  if (nin == 0) return GFX_OK;
  uint8_t *hit, *miss;
  GFX_TRY(scratch_t(g, "op_pull_hit", nin + 1, &hit));
  GFX_TRY(scratch_t(g, "op_pull_miss", nin + 1, &miss));
  Counters* C = g->counters;
  GFX_CK(cudaMemsetAsync(C, 0, sizeof(Counters), ctx->stream));
  const RegFn f = make_fn(functor_id, args);
  GFX_LAUNCH(k_pull_probe, grid_for(nin * 32, 256, ctx->sm_count * 16), 256, 0, ctx->stream,
             fin_d, nin, g->rrow, g->rcol, f, hit, &C->edges);
  GFX_LAUNCH(k_flags_invert, grid_for(nin, 256, ctx->sm_count * 8), 256, 0, ctx->stream, hit, nin,
             miss);
  auto* pin = static_cast<int64_t*>(ctx->pinned);
  GFX_TRY(select_flagged(g, fin_d, hit, nin, active_d, &pin[0], "op_pull_sel_a"));
  GFX_CK(cudaStreamSynchronize(ctx->stream));
  const int64_t na = pin[0];
  GFX_TRY(select_flagged(g, fin_d, miss, nin, rest_d, &pin[1], "op_pull_sel_r"));
  GFX_CK(cudaMemcpyAsync(&pin[2], &C->edges, 8, cudaMemcpyDeviceToHost, ctx->stream));
  GFX_CK(cudaGetLastError());
  GFX_CK(cudaStreamSynchronize(ctx->stream));
  *nactive = na;
  *nrest = pin[1];
  if (edges) *edges = pin[2];
  return GFX_OK;
}

int gfx_filter(gfx_graph* g, const int32_t* fin_d, int64_t nin, int mode, int functor_id,
               const gfx_functor_args* args, int64_t domain, int32_t* fout_d, int64_t* nout) {
  GFX_NVTX("gfx_filter");
  GFX_REQUIRE(g && nout && (nin == 0 || (fin_d && fout_d)), "gfx_filter: null argument");
  GFX_REQUIRE(mode == GFX_FILTER_EXACT || mode == GFX_FILTER_INEXACT, "unknown filter mode %d", mode);
  GFX_REQUIRE(is_vertex_fn(functor_id), "functor %d is not a filter functor of the registry",
              functor_id);
  const RegFn f = make_fn(functor_id, args);
  GFX_TRY(check_fn_args(g, f));
  GFX_REQUIRE(domain > 0 && domain < (int64_t)INT32_MAX, "bad id domain %lld", (long long)domain);
  gfx_ctx* ctx = g->ctx;
  GFX_CK(cudaSetDevice(ctx->device));
  *nout = 0;
  if (nin == 0) return GFX_OK;
  // survivors deduplicated and sorted (np.unique, operators.py:378-379);
  // the Python layer runs the INEXACT heuristics (gfx_cull_stage) instead
  const int64_t words = (domain + 31) / 32;
  uint32_t* bm;
  int64_t *cnt, *off;
  GFX_TRY(scratch_t(g, "op_bm", words + 1, &bm));
  GFX_TRY(scratch_t(g, "op_cnt", words + 1, &cnt));
  GFX_TRY(scratch_t(g, "op_off", words + 1, &off));
  GFX_CK(cudaMemsetAsync(bm, 0, (words + 1) * 4, ctx->stream));
  const int grid = ctx->sm_count * 8;
  GFX_LAUNCH(k_filter_mark, grid_for(nin, 256, grid), 256, 0, ctx->stream, fin_d, nin, f, g->row,
             g->col, g->n, bm);
  GFX_LAUNCH(k_word_popc, grid_for(words + 1, 256, grid), 256, 0, ctx->stream, bm, words + 1, cnt);
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, off, words + 1, ctx->stream);
  void* tmp = nullptr;
  GFX_TRY(scratch(g, "op_scan_tmp", tb, &tmp));
  cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, off, words + 1, ctx->stream);
  count_launch();
  GFX_LAUNCH(k_word_emit, grid_for(words, 256, grid), 256, 0, ctx->stream, bm, words, off, fout_d);
  GFX_CK(cudaGetLastError());
  int64_t total = 0;
  GFX_CK(cudaMemcpyAsync(&total, off + words, 8, cudaMemcpyDeviceToHost, ctx->stream));
  GFX_CK(cudaStreamSynchronize(ctx->stream));
  *nout = total;
  return GFX_OK;
}

int gfx_vertex_mask(gfx_graph* g, const int32_t* fin_d, int64_t nin, int functor_id,
                    const gfx_functor_args* args, uint8_t* mask_d) {
  GFX_REQUIRE(g && (nin == 0 || (fin_d && mask_d)), "gfx_vertex_mask: null argument");
  GFX_REQUIRE(is_vertex_fn(functor_id), "functor %d is not a vertex functor of the registry",
              functor_id);
  const RegFn f = make_fn(functor_id, args);
  GFX_TRY(check_fn_args(g, f));
  GFX_CK(cudaSetDevice(g->ctx->device));
  if (nin == 0) return GFX_OK;
  GFX_LAUNCH(k_vertex_mask, grid_for(nin, 256, g->ctx->sm_count * 8), 256, 0, g->ctx->stream,
             fin_d, nin, f, g->row, g->col, g->n, mask_d);
  GFX_CK(cudaGetLastError());
  GFX_CK(cudaStreamSynchronize(g->ctx->stream));
  return GFX_OK;
}

int gfx_compute(gfx_graph* g, const int32_t* fin_d, int64_t nin, int functor_id,
                const gfx_functor_args* args, int64_t* acc_d) {
  GFX_NVTX("gfx_compute");
  GFX_REQUIRE(g && (nin == 0 || fin_d), "gfx_compute: null argument");
  GFX_REQUIRE(functor_id == GFX_FN_SET_LABEL || functor_id == GFX_FN_ADD_I64,
              "functor %d is not a compute functor of the registry", functor_id);
  GFX_REQUIRE(functor_id != GFX_FN_SET_LABEL || (args && args->labels_d), "SET_LABEL needs labels");
  GFX_REQUIRE(functor_id != GFX_FN_ADD_I64 || acc_d, "ADD_I64 needs an int64 array");
  GFX_CK(cudaSetDevice(g->ctx->device));
  if (nin == 0) return GFX_OK;
  GFX_LAUNCH(k_compute, grid_for(nin, 256, g->ctx->sm_count * 8), 256, 0, g->ctx->stream, fin_d,
             nin, functor_id, args ? args->labels_d : nullptr, acc_d, args ? args->value : 0);
  GFX_CK(cudaGetLastError());
  GFX_CK(cudaStreamSynchronize(g->ctx->stream));
  return GFX_OK;
}

int gfx_segmented_intersect_list(gfx_graph* g, const int32_t* u_d, const int32_t* v_d,
                                 int64_t num_pairs, const int64_t* offsets_d, int32_t* out_d) {
  GFX_REQUIRE(g && (num_pairs == 0 || (u_d && v_d && offsets_d && out_d)),
              "gfx_segmented_intersect_list: null argument");
  GFX_CK(cudaSetDevice(g->ctx->device));
  if (num_pairs == 0) return GFX_OK;
  GFX_LAUNCH(k_intersect_list, grid_for(num_pairs, 256, g->ctx->sm_count * 8), 256, 0,
             g->ctx->stream, u_d, v_d, num_pairs, g->row, g->col, offsets_d, out_d);
  GFX_CK(cudaGetLastError());
  GFX_CK(cudaStreamSynchronize(g->ctx->stream));
  return GFX_OK;
}

}  // extern "C"
