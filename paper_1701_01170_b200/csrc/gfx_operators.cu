// Generic operators with the closed device-functor registry.
//
// Reference: operators.py:218-266 (advance), :360-384 (filter_frontier),
// :485-525 (segmented_intersect), :528-533 (compute).  The reference takes
// arbitrary Python callables over whole id arrays; on the device the functors
// are a closed registry (include/gfx.h GFX_FN_*), each the device form of a
// lambda the six primitives pass (SURVEY 8(b) functor table).  advance() runs
// on the same load-balanced warp-tile expansion as the primitives.
#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>

#include "gfx_device.cuh"
#include "gfx_expand.cuh"
#include "gfx_internal.cuh"

namespace gfx {

template <bool EMIT_EDGE, bool WEIGHTS>
struct RegistryOp {
  static constexpr bool kWeights = WEIGHTS, kSrcVal = false, kEmitEdge = EMIT_EDGE;
  static constexpr int kBatch = 4;
  static constexpr int kMinBlocks = 2;
  int fid;
  int32_t* labels;
  int32_t* preds;
  int32_t value;
  const int64_t* row;
  __device__ int32_t src_value(int32_t) const { return 0; }
  __device__ void prefetch(const int32_t*) {}
  __device__ bool visit(int, int32_t d, int32_t s, int32_t w, int32_t, int64_t) {
    switch (fid) {
      case GFX_FN_NONE:
        return true;
      case GFX_FN_BFS_CLAIM: {  // compare_and_swap(labels, d, UNVISITED, depth) + preds[d] = s
        if (labels[d] != GFX_UNVISITED) return false;
        if (atomicCAS(&labels[d], GFX_UNVISITED, value) != GFX_UNVISITED) return false;
        if (preds) preds[d] = s;
        return true;
      }
      case GFX_FN_BFS_IDEMP: {  // labels[d] == UNVISITED; _set_depth (duplicates allowed)
        if (labels[d] != GFX_UNVISITED) return false;
        labels[d] = value;
        if (preds) preds[d] = s;
        return true;
      }
      case GFX_FN_SSSP_RELAX: {  // atomic_min(labels, d, labels[s] + w[e]); set_pred
        const int32_t ls = labels[s];
        if (ls == GFX_UNVISITED) return false;
        const int32_t nd = ls + w;
        if (nd >= labels[d]) return false;
        if (atomicMin(&labels[d], nd) <= nd) return false;
        if (preds) preds[d] = s;
        return true;
      }
      case GFX_FN_TC_ORIENT: {  // deg[s] > deg[d] or (== and s < d)
        const int64_t ds = row[s + 1] - row[s], dd = row[d + 1] - row[d];
        return ds > dd || (ds == dd && s < d);
      }
      case GFX_FN_LABEL_EQ:
        return labels[d] == value;
      case GFX_FN_LABEL_NE:
        return labels[d] != value;
      default:
        return false;
    }
  }
};

__global__ void k_edge_targets(const int32_t* __restrict__ edges, int64_t n,
                               const int32_t* __restrict__ col, int32_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = col[edges[i]];
}

// filter: mark survivors in a bitmap over the id domain
__global__ void k_filter_mark(const int32_t* __restrict__ in, int64_t n, int fid,
                              const int32_t* __restrict__ labels, int32_t value,
                              uint32_t* __restrict__ bm) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = in[i];
    bool keep = true;
    if (fid == GFX_FN_LABEL_EQ) keep = labels[v] == value;
    else if (fid == GFX_FN_LABEL_NE) keep = labels[v] != value;
    if (keep) atomicOr(&bm[v >> 5], 1u << (v & 31));
  }
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
static int run_advance(gfx_graph* g, const int32_t* F, int64_t nin, int fid,
                       const gfx_functor_args* args, int32_t* out, int64_t cap, int64_t* nout,
                       int64_t* edges) {
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
  Op op{fid, args ? args->labels_d : nullptr, args ? args->preds_d : nullptr,
        args ? (int32_t)args->value : 0, g->row};
  GFX_TRY(set_expand_smem<Op>());
  GFX_LAUNCH((k_lb_expand<Op>), ctx->sm_count * 2, kExpandBlock, expand_smem_bytes(), ctx->stream,
             F, &C[0].out_len, scan, rowbase, part, &C[1], g->col, g->w, op, out, &C[1].out_len);
  GFX_CK(cudaGetLastError());
  GFX_CK(cudaMemcpyAsync(pin, &C[1], sizeof(Counters), cudaMemcpyDeviceToHost, ctx->stream));
  GFX_CK(cudaStreamSynchronize(ctx->stream));
  *nout = (int64_t)pin->out_len;
  if (edges) *edges = total;
  return GFX_OK;
}

}  // namespace gfx

using namespace gfx;

extern "C" {

int gfx_advance(gfx_graph* g, const int32_t* fin_d, int64_t nin, int kind, int functor_id,
                const gfx_functor_args* args, int32_t* fout_d, int64_t fout_cap, int64_t* nout,
                int64_t* edges) {
  GFX_REQUIRE(g && nout && (nin == 0 || (fin_d && fout_d)), "gfx_advance: null argument");
  GFX_REQUIRE(kind >= GFX_KIND_V2V && kind <= GFX_KIND_E2E, "unknown advance kind %d", kind);
  GFX_REQUIRE(functor_id >= GFX_FN_NONE && functor_id <= GFX_FN_LABEL_NE,
              "functor %d is not an advance functor of the registry", functor_id);
  const bool need_labels = functor_id != GFX_FN_NONE && functor_id != GFX_FN_TC_ORIENT;
  GFX_REQUIRE(!need_labels || (args && args->labels_d), "functor %d needs labels", functor_id);
  GFX_REQUIRE(functor_id != GFX_FN_SSSP_RELAX || g->w, "SSSP relax needs edge weights");
  GFX_CK(cudaSetDevice(g->ctx->device));
  *nout = 0;
  if (edges) *edges = 0;
  if (nin == 0) return GFX_OK;
  const int32_t* F = fin_d;
  if (kind == GFX_KIND_E2V || kind == GFX_KIND_E2E) {
    // edge frontiers expand the edge's destination (load_balance.py:94-102)
    int32_t* tgt = nullptr;
    GFX_TRY(scratch_t(g, "op_targets", nin + 1, &tgt));
    GFX_LAUNCH(k_edge_targets, grid_for(nin, 256, g->ctx->sm_count * 8), 256, 0, g->ctx->stream,
               fin_d, nin, g->col, tgt);
    F = tgt;
  }
  const bool emit_edge = kind == GFX_KIND_V2E || kind == GFX_KIND_E2E;
  const bool weights = functor_id == GFX_FN_SSSP_RELAX;
  if (emit_edge)
    return weights ? run_advance<true, true>(g, F, nin, functor_id, args, fout_d, fout_cap, nout,
                                             edges)
                   : run_advance<true, false>(g, F, nin, functor_id, args, fout_d, fout_cap, nout,
                                              edges);
  return weights ? run_advance<false, true>(g, F, nin, functor_id, args, fout_d, fout_cap, nout,
                                            edges)
                 : run_advance<false, false>(g, F, nin, functor_id, args, fout_d, fout_cap, nout,
                                             edges);
}

int gfx_filter(gfx_graph* g, const int32_t* fin_d, int64_t nin, int mode, int functor_id,
               const gfx_functor_args* args, int64_t domain, int32_t* fout_d, int64_t* nout) {
  GFX_REQUIRE(g && nout && (nin == 0 || (fin_d && fout_d)), "gfx_filter: null argument");
  GFX_REQUIRE(mode == GFX_FILTER_EXACT || mode == GFX_FILTER_INEXACT, "unknown filter mode %d", mode);
  GFX_REQUIRE(functor_id == GFX_FN_NONE || functor_id == GFX_FN_LABEL_EQ ||
                  functor_id == GFX_FN_LABEL_NE,
              "functor %d is not a filter functor of the registry", functor_id);
  GFX_REQUIRE(functor_id == GFX_FN_NONE || (args && args->labels_d), "filter functor needs labels");
  GFX_REQUIRE(domain > 0 && domain < (int64_t)INT32_MAX, "bad id domain %lld", (long long)domain);
  gfx_ctx* ctx = g->ctx;
  GFX_CK(cudaSetDevice(ctx->device));
  *nout = 0;
  if (nin == 0) return GFX_OK;
  // EXACT: survivors deduplicated and sorted (np.unique, operators.py:378-379);
  // INEXACT returns the same set, which satisfies its superset contract.
  const int64_t words = (domain + 31) / 32;
  uint32_t* bm;
  int64_t *cnt, *off;
  GFX_TRY(scratch_t(g, "op_bm", words + 1, &bm));
  GFX_TRY(scratch_t(g, "op_cnt", words + 1, &cnt));
  GFX_TRY(scratch_t(g, "op_off", words + 1, &off));
  GFX_CK(cudaMemsetAsync(bm, 0, (words + 1) * 4, ctx->stream));
  const int grid = ctx->sm_count * 8;
  GFX_LAUNCH(k_filter_mark, grid_for(nin, 256, grid), 256, 0, ctx->stream, fin_d, nin, functor_id,
             args ? args->labels_d : nullptr, args ? (int32_t)args->value : 0, bm);
  GFX_LAUNCH(k_word_popc, grid_for(words + 1, 256, grid), 256, 0, ctx->stream, bm, words + 1, cnt);
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, off, words + 1, ctx->stream);
  void* tmp = nullptr;
  GFX_TRY(scratch(g, "op_scan_tmp", tb, &tmp));
  cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, off, words + 1, ctx->stream);
  GFX_LAUNCH(k_word_emit, grid_for(words, 256, grid), 256, 0, ctx->stream, bm, words, off, fout_d);
  GFX_CK(cudaGetLastError());
  int64_t total = 0;
  GFX_CK(cudaMemcpyAsync(&total, off + words, 8, cudaMemcpyDeviceToHost, ctx->stream));
  GFX_CK(cudaStreamSynchronize(ctx->stream));
  *nout = total;
  return GFX_OK;
}

int gfx_compute(gfx_graph* g, const int32_t* fin_d, int64_t nin, int functor_id,
                const gfx_functor_args* args, int64_t* acc_d) {
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
