// Building blocks of the staged operator path and the batched atomics.
//
// The reference operators take Python callables over whole id arrays and run
// them between a gather and a commit (operators.py:10-15, 161-215).  Here a
// callable functor runs on DEVICE tensors: these kernels materialise the
// expansion triples in slot order (_gather, operators.py:161-197), compact
// them by the callable's mask, mark pull hits, reproduce the INEXACT culling
// heuristics exactly (operators.py:315-357), and implement the batched atomic
// helpers functors mutate problem data with (operators.py:111-153).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <cuda_runtime.h>

#include "gfx_device.cuh"
#include "gfx_internal.cuh"

namespace gfx {

#define GRID_STRIDE(i, n)                                                   \
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n); \
       i += (int64_t)gridDim.x * blockDim.x)

// expansion degree of item i (vertex, or the head of an edge)
__global__ void k_item_degrees(const int32_t* __restrict__ fin, int64_t n, int edge_input,
                               const int32_t* __restrict__ col, const int64_t* __restrict__ rows,
                               int64_t* __restrict__ deg) {
  GRID_STRIDE(i, n + 1) {
    if (i == n) {
      deg[i] = 0;
    } else {
      const int64_t v = edge_input ? (int64_t)col[fin[i]] : (int64_t)fin[i];
      deg[i] = rows[v + 1] - rows[v];
    }
  }
}

// slot-parallel gather: each slot finds its item by binary search in scan
__global__ void k_gather(const int32_t* __restrict__ fin, int64_t nin, int edge_input,
                         const int32_t* __restrict__ fcol, const int64_t* __restrict__ rows,
                         const int32_t* __restrict__ cols, const int64_t* __restrict__ eids,
                         const int64_t* __restrict__ scan, int64_t total, int64_t* __restrict__ a,
                         int64_t* __restrict__ b, int64_t* __restrict__ e,
                         int32_t* __restrict__ rep) {
  GRID_STRIDE(k, total) {
    int64_t lo = 0, hi = nin;  // largest i with scan[i] <= k (scan[nin] = total > k)
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (scan[mid] <= k) lo = mid;
      else hi = mid;
    }
    const int64_t v = edge_input ? (int64_t)fcol[fin[lo]] : (int64_t)fin[lo];
    const int64_t j = rows[v] + (k - scan[lo]);
    a[k] = v;
    b[k] = cols[j];
    e[k] = eids ? eids[j] : j;
    if (rep) rep[k] = (int32_t)lo;
  }
}

__global__ void k_iota64(int64_t* __restrict__ p, int64_t n) {
  GRID_STRIDE(i, n) p[i] = i;
}

__global__ void k_col_histogram(const int32_t* __restrict__ col, int64_t m,
                                int64_t* __restrict__ cnt) {
  GRID_STRIDE(i, m) atomicAdd((unsigned long long*)&cnt[col[i]], 1ull);
}

// rcol[j] = source vertex of forward slot reid[j]
__global__ void k_slot_sources(const int64_t* __restrict__ reid, int64_t m,
                               const int64_t* __restrict__ row, int64_t n,
                               int32_t* __restrict__ rcol) {
  GRID_STRIDE(j, m) {
    const int64_t e = reid[j];
    int64_t lo = 0, hi = n;
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (row[mid] <= e) lo = mid;
      else hi = mid;
    }
    rcol[j] = (int32_t)lo;
  }
}

__global__ void k_mark_items(const uint8_t* __restrict__ mask, const int32_t* __restrict__ rep,
                             int64_t k, uint8_t* __restrict__ hits) {
  GRID_STRIDE(i, k) if (mask[i]) hits[rep[i]] = 1;
}

__global__ void k_invert(const uint8_t* __restrict__ in, int64_t n, uint8_t* __restrict__ out) {
  GRID_STRIDE(i, n) out[i] = !in[i];
}

// StatusBitmap.test_and_set: reads precede writes within the batch
__global__ void k_bits_test(const uint32_t* __restrict__ w, const int64_t* __restrict__ ids,
                            int64_t k, uint8_t* __restrict__ fresh) {
  GRID_STRIDE(i, k) fresh[i] = !((w[ids[i] >> 5] >> (ids[i] & 31)) & 1u);
}
__global__ void k_bits_set(uint32_t* __restrict__ w, const int64_t* __restrict__ ids, int64_t k) {
  GRID_STRIDE(i, k) atomicOr(&w[ids[i] >> 5], 1u << (ids[i] & 31));
}
template <class T>
__global__ void k_eq_flags(const T* __restrict__ a, int64_t n, T v, uint8_t* __restrict__ f) {
  GRID_STRIDE(i, n) f[i] = a[i] == v;
}

// ---- INEXACT culling (operators.py:315-357) -------------------------------
// bitmask stage: an item survives iff no EARLIER batch held its id
// (_cull_bitmask reads the seen bits before marking the batch)
__global__ void k_first_batch(const int64_t* __restrict__ items, int64_t n, int64_t batch,
                              int64_t* __restrict__ first) {
  GRID_STRIDE(i, n) atomicMin((long long*)&first[items[i]], (long long)(i / batch));
}
__global__ void k_bitmask_keep(const int64_t* __restrict__ items, int64_t n, int64_t batch,
                               const int64_t* __restrict__ first, uint8_t* __restrict__ keep) {
  GRID_STRIDE(i, n) keep[i] = first[items[i]] == i / batch;
}
// history stage: one thread replays one batch in order with a direct-mapped
// table (slot = id mod size): an item is dropped when the previous item of
// its slot in this batch carried the same id (_cull_history's stable sort by
// slot compares exactly those neighbours)
__global__ void k_history_keep(const int64_t* __restrict__ items, int64_t n, int64_t table,
                               int64_t batch, int64_t* __restrict__ tab,
                               uint8_t* __restrict__ keep) {
  const int64_t nb = (n + batch - 1) / batch;
  int64_t* t = tab + (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * table;  // per thread
  GRID_STRIDE(bi, nb) {
    for (int64_t s = 0; s < table; ++s) t[s] = -1;
    const int64_t lo = bi * batch, hi = min(lo + batch, n);
    for (int64_t i = lo; i < hi; ++i) {
      const int64_t x = items[i];
      const int64_t s = x % table;
      keep[i] = t[s] != x;
      t[s] = x;
    }
  }
}

// ---- batched atomics --------------------------------------------------------
template <class T>
__device__ __forceinline__ void atomic_min_t(T* p, T v);
template <>
__device__ __forceinline__ void atomic_min_t<int32_t>(int32_t* p, int32_t v) { atomicMin(p, v); }
template <>
__device__ __forceinline__ void atomic_min_t<int64_t>(int64_t* p, int64_t v) {
  atomicMin((long long*)p, (long long)v);
}
template <class T>
__device__ __forceinline__ void atomic_add_t(T* p, T v) { atomicAdd(p, v); }
template <>
__device__ __forceinline__ void atomic_add_t<int64_t>(int64_t* p, int64_t v) {
  atomicAdd((unsigned long long*)p, (unsigned long long)v);
}

template <class T>
__global__ void k_amin_pre(const T* __restrict__ arr, const int64_t* __restrict__ idx, int64_t k,
                           T* __restrict__ pre) {
  GRID_STRIDE(i, k) pre[i] = arr[idx[i]];
}
template <class T>
__global__ void k_amin(T* __restrict__ arr, const int64_t* __restrict__ idx,
                       const T* __restrict__ vals, const T* __restrict__ pre, int64_t k) {
  GRID_STRIDE(i, k) if (vals[i] < pre[i]) atomic_min_t(&arr[idx[i]], vals[i]);
}
template <class T>
__global__ void k_amin_won(const T* __restrict__ arr, const int64_t* __restrict__ idx,
                           const T* __restrict__ vals, const T* __restrict__ pre, int64_t k,
                           uint8_t* __restrict__ won) {
  GRID_STRIDE(i, k) won[i] = vals[i] < pre[i] && vals[i] == arr[idx[i]];
}
template <class T>
__global__ void k_aadd(T* __restrict__ arr, const int64_t* __restrict__ idx,
                       const T* __restrict__ vals, T scalar, int64_t k) {
  GRID_STRIDE(i, k) atomic_add_t(&arr[idx[i]], vals ? vals[i] : scalar);
}
// compare_and_swap: eligibility from the pre-call state, earliest occurrence wins
template <class T>
__global__ void k_cas_elig(const T* __restrict__ arr, const int64_t* __restrict__ idx, int64_t k,
                           T expected, uint8_t* __restrict__ won, int64_t* __restrict__ pos) {
  GRID_STRIDE(i, k) {
    const bool el = arr[idx[i]] == expected;
    won[i] = el;
    if (el) pos[idx[i]] = INT64_MAX;
  }
}
__global__ void k_cas_claim(const int64_t* __restrict__ idx, int64_t k,
                            const uint8_t* __restrict__ won, int64_t* __restrict__ pos) {
  GRID_STRIDE(i, k) if (won[i]) atomicMin((long long*)&pos[idx[i]], (long long)i);
}
template <class T>
__global__ void k_cas_store(T* __restrict__ arr, const int64_t* __restrict__ idx, int64_t k,
                            const T* __restrict__ vals, T scalar, uint8_t* __restrict__ won,
                            const int64_t* __restrict__ pos) {
  GRID_STRIDE(i, k) {
    if (won[i]) {
      const bool w = pos[idx[i]] == i;
      won[i] = w;
      if (w) arr[idx[i]] = vals ? vals[i] : scalar;
    }
  }
}

inline int grid_of(gfx_ctx* ctx, int64_t n) { return grid_for(n, 256, ctx->sm_count * 8); }

template <class T>
int run_atomic_min(gfx_ctx* ctx, T* arr, const int64_t* idx, const T* vals, int64_t k,
                   uint8_t* won, T* pre) {
  const int gr = grid_of(ctx, k);
  GFX_LAUNCH(k_amin_pre<T>, gr, 256, 0, ctx->stream, arr, idx, k, pre);
  GFX_LAUNCH(k_amin<T>, gr, 256, 0, ctx->stream, arr, idx, vals, pre, k);
  GFX_LAUNCH(k_amin_won<T>, gr, 256, 0, ctx->stream, arr, idx, vals, pre, k, won);
  return GFX_OK;
}

template <class T>
int run_cas(gfx_ctx* ctx, T* arr, const int64_t* idx, int64_t k, T expected, const T* vals,
            T scalar, uint8_t* won, int64_t* pos) {
  const int gr = grid_of(ctx, k);
  GFX_LAUNCH(k_cas_elig<T>, gr, 256, 0, ctx->stream, arr, idx, k, expected, won, pos);
  GFX_LAUNCH(k_cas_claim, gr, 256, 0, ctx->stream, idx, k, won, pos);
  GFX_LAUNCH(k_cas_store<T>, gr, 256, 0, ctx->stream, arr, idx, k, vals, scalar, won, pos);
  return GFX_OK;
}

}  // namespace gfx

using namespace gfx;

extern "C" {

int gfx_scan_offsets(gfx_graph* g, const int32_t* fin_d, int64_t nin, int edge_input, int reverse,
                     int64_t* scan_d, int64_t* total) {
  GFX_REQUIRE(g && scan_d && total && (nin == 0 || fin_d), "gfx_scan_offsets: null argument");
  const int64_t* rows = reverse ? g->rrow : g->row;
  GFX_REQUIRE(rows, "reverse scan needs the reverse adjacency");
  gfx_ctx* ctx = g->ctx;
  GFX_CK(cudaSetDevice(ctx->device));
  int64_t* deg;
  GFX_TRY(scratch_t(g, "op_deg", nin + 2, &deg));
  GFX_LAUNCH(k_item_degrees, grid_of(ctx, nin + 1), 256, 0, ctx->stream, fin_d, nin, edge_input,
             g->col, rows, deg);
  size_t tb = 0;
  GFX_CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, deg, scan_d, nin + 1, ctx->stream));
  void* tmp;
  GFX_TRY(scratch(g, "op_scan_tmp2", tb + 16, &tmp));
  GFX_CK(cub::DeviceScan::ExclusiveSum(tmp, tb, deg, scan_d, nin + 1, ctx->stream));
  count_launch();
  auto* pin = static_cast<int64_t*>(ctx->pinned);
  GFX_CK(cudaMemcpyAsync(pin, scan_d + nin, 8, cudaMemcpyDeviceToHost, ctx->stream));
  GFX_CK(cudaStreamSynchronize(ctx->stream));
  *total = pin[0];
  return GFX_OK;
}

int gfx_gather(gfx_graph* g, const int32_t* fin_d, int64_t nin, int edge_input, int reverse,
               const int64_t* scan_d, int64_t total, int64_t* a_d, int64_t* b_d, int64_t* e_d,
               int32_t* rep_d) {
  GFX_NVTX("gfx_gather");
  GFX_REQUIRE(g && (total == 0 || (fin_d && scan_d && a_d && b_d && e_d)),
              "gfx_gather: null argument");
  GFX_REQUIRE(!reverse || (g->rrow && g->rcol && g->reid),
              "reverse gather needs gfx_graph_build_csc first");
  gfx_ctx* ctx = g->ctx;
  GFX_CK(cudaSetDevice(ctx->device));
  if (total == 0) return GFX_OK;
  GFX_LAUNCH(k_gather, grid_of(ctx, total), 256, 0, ctx->stream, fin_d, nin, edge_input, g->col,
             reverse ? g->rrow : g->row, reverse ? g->rcol : g->col, reverse ? g->reid : nullptr,
             scan_d, total, a_d, b_d, e_d, rep_d);
  GFX_CK(cudaGetLastError());
  GFX_CK(cudaStreamSynchronize(ctx->stream));
  return GFX_OK;
}

int gfx_graph_build_csc(gfx_graph* g, int64_t* rrow_d, int32_t* rcol_d, int64_t* reid_d) {
  GFX_NVTX("gfx_graph_build_csc");
  GFX_REQUIRE(g && rrow_d && (g->m == 0 || (rcol_d && reid_d)), "gfx_graph_build_csc: null argument");
  gfx_ctx* ctx = g->ctx;
  GFX_CK(cudaSetDevice(ctx->device));
  const int64_t n = g->n, m = g->m;
  int64_t* cnt;
  GFX_CK(cudaMallocAsync(&cnt, (n + 1) * 8, ctx->stream));
  GFX_CK(cudaMemsetAsync(cnt, 0, (n + 1) * 8, ctx->stream));
  if (m) GFX_LAUNCH(k_col_histogram, grid_of(ctx, m), 256, 0, ctx->stream, g->col, m, cnt);
  size_t tb = 0;
  GFX_CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, rrow_d, n + 1, ctx->stream));
  void* tmp;
  GFX_CK(cudaMallocAsync(&tmp, tb + 16, ctx->stream));
  GFX_CK(cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, rrow_d, n + 1, ctx->stream));
  count_launch();
  GFX_CK(cudaFreeAsync(tmp, ctx->stream));
  GFX_CK(cudaFreeAsync(cnt, ctx->stream));
  if (m) {
    // stable radix sort of (col, forward slot): argsort(col, kind="stable")
    int64_t* slots;
    int32_t* keys_out;
    GFX_CK(cudaMallocAsync(&slots, m * 8, ctx->stream));
    GFX_CK(cudaMallocAsync(&keys_out, m * 4, ctx->stream));
    GFX_LAUNCH(k_iota64, grid_of(ctx, m), 256, 0, ctx->stream, slots, m);
    int bits = 1;
    while (bits < 31 && (int64_t{1} << bits) < n) ++bits;
    tb = 0;
    GFX_CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, g->col, keys_out, slots, reid_d, m, 0,
                                           bits, ctx->stream));
    GFX_CK(cudaMallocAsync(&tmp, tb + 16, ctx->stream));
    GFX_CK(cub::DeviceRadixSort::SortPairs(tmp, tb, g->col, keys_out, slots, reid_d, m, 0, bits,
                                           ctx->stream));
    count_launch();
    GFX_CK(cudaFreeAsync(tmp, ctx->stream));
    GFX_CK(cudaFreeAsync(keys_out, ctx->stream));
    GFX_CK(cudaFreeAsync(slots, ctx->stream));
    GFX_LAUNCH(k_slot_sources, grid_of(ctx, m), 256, 0, ctx->stream, reid_d, m, g->row, n, rcol_d);
  }
  GFX_CK(cudaGetLastError());
  GFX_CK(cudaStreamSynchronize(ctx->stream));
  g->reid = reid_d;
  if (!(g->flags & GFX_GRAPH_UNDIRECTED)) return gfx_graph_set_reverse(g, rrow_d, rcol_d);
  return GFX_OK;
}

int gfx_select_i64(gfx_ctx* ctx, const int64_t* in_d, const uint8_t* flags_d, int64_t n,
                   int invert, int64_t* out_d, int64_t* nout) {
  GFX_REQUIRE(ctx && nout && (n == 0 || (in_d && flags_d && out_d)), "gfx_select_i64: null argument");
  GFX_CK(cudaSetDevice(ctx->device));
  *nout = 0;
  if (n == 0) return GFX_OK;
  const uint8_t* fl = flags_d;
  uint8_t* inv = nullptr;
  if (invert) {
    GFX_CK(cudaMallocAsync(&inv, n, ctx->stream));
    GFX_LAUNCH(k_invert, grid_of(ctx, n), 256, 0, ctx->stream, flags_d, n, inv);
    fl = inv;
  }
  int64_t* cnt;
  GFX_CK(cudaMallocAsync(&cnt, 8, ctx->stream));
  size_t tb = 0;
  GFX_CK(cub::DeviceSelect::Flagged(nullptr, tb, in_d, fl, out_d, cnt, n, ctx->stream));
  void* tmp;
  GFX_CK(cudaMallocAsync(&tmp, tb + 16, ctx->stream));
  GFX_CK(cub::DeviceSelect::Flagged(tmp, tb, in_d, fl, out_d, cnt, n, ctx->stream));
  count_launch();
  auto* pin = static_cast<int64_t*>(ctx->pinned);
  GFX_CK(cudaMemcpyAsync(pin, cnt, 8, cudaMemcpyDeviceToHost, ctx->stream));
  GFX_CK(cudaFreeAsync(tmp, ctx->stream));
  GFX_CK(cudaFreeAsync(cnt, ctx->stream));
  if (inv) GFX_CK(cudaFreeAsync(inv, ctx->stream));
  GFX_CK(cudaStreamSynchronize(ctx->stream));
  *nout = pin[0];
  return GFX_OK;
}

int gfx_bitmap_test_and_set(gfx_ctx* ctx, uint32_t* words_d, const int64_t* ids_d, int64_t k,
                            uint8_t* fresh_d) {
  GFX_REQUIRE(ctx && (k == 0 || (words_d && ids_d && fresh_d)),
              "gfx_bitmap_test_and_set: null argument");
  GFX_CK(cudaSetDevice(ctx->device));
  if (k == 0) return GFX_OK;
  GFX_LAUNCH(k_bits_test, grid_of(ctx, k), 256, 0, ctx->stream, words_d, ids_d, k, fresh_d);
  GFX_LAUNCH(k_bits_set, grid_of(ctx, k), 256, 0, ctx->stream, words_d, ids_d, k);
  GFX_CK(cudaGetLastError());
  GFX_CK(cudaStreamSynchronize(ctx->stream));
  return GFX_OK;
}

int gfx_unvisited(gfx_ctx* ctx, int dtype, const void* labels_d, int64_t n, int64_t sentinel,
                  int64_t* out_d, int64_t* nout) {
  GFX_REQUIRE(ctx && nout && (n == 0 || (labels_d && out_d)), "gfx_unvisited: null argument");
  GFX_REQUIRE(dtype == 0 || dtype == 1, "labels must be int32 or int64");
  GFX_CK(cudaSetDevice(ctx->device));
  *nout = 0;
  if (n == 0) return GFX_OK;
  uint8_t* fl;
  int64_t* ids;
  GFX_CK(cudaMallocAsync(&fl, n, ctx->stream));
  GFX_CK(cudaMallocAsync(&ids, n * 8, ctx->stream));
  if (dtype == 0)
    GFX_LAUNCH(k_eq_flags<int32_t>, grid_of(ctx, n), 256, 0, ctx->stream, (const int32_t*)labels_d,
               n, (int32_t)sentinel, fl);
  else
    GFX_LAUNCH(k_eq_flags<int64_t>, grid_of(ctx, n), 256, 0, ctx->stream, (const int64_t*)labels_d,
               n, sentinel, fl);
  GFX_LAUNCH(k_iota64, grid_of(ctx, n), 256, 0, ctx->stream, ids, n);
  const int st = gfx_select_i64(ctx, ids, fl, n, 0, out_d, nout);
  cudaFreeAsync(fl, ctx->stream);
  cudaFreeAsync(ids, ctx->stream);
  GFX_CK(cudaStreamSynchronize(ctx->stream));
  return st;
}

int gfx_mark_items(gfx_ctx* ctx, const uint8_t* mask_d, const int32_t* rep_d, int64_t k,
                   uint8_t* hits_d) {
  GFX_REQUIRE(ctx && (k == 0 || (mask_d && rep_d && hits_d)), "gfx_mark_items: null argument");
  GFX_CK(cudaSetDevice(ctx->device));
  if (k == 0) return GFX_OK;
  GFX_LAUNCH(k_mark_items, grid_of(ctx, k), 256, 0, ctx->stream, mask_d, rep_d, k, hits_d);
  GFX_CK(cudaGetLastError());
  GFX_CK(cudaStreamSynchronize(ctx->stream));
  return GFX_OK;
}

int gfx_cull_stage(gfx_ctx* ctx, const int64_t* items_d, int64_t n, int stage, int64_t domain,
                   int64_t table_or_batch, int64_t batch, uint8_t* keep_d) {
  GFX_REQUIRE(ctx && (n == 0 || (items_d && keep_d)), "gfx_cull_stage: null argument");
  GFX_REQUIRE(stage >= 0 && stage <= 2, "unknown cull stage %d", stage);
  GFX_REQUIRE(table_or_batch >= 1 && batch >= 1, "cull table/batch sizes must be >= 1");
  GFX_CK(cudaSetDevice(ctx->device));
  if (n == 0) return GFX_OK;
  if (stage == 0) {  // bitmask over [0, domain), batches of table_or_batch items
    GFX_REQUIRE(domain >= 1, "bitmask culling needs a positive id domain");
    int64_t* first;
    GFX_CK(cudaMallocAsync(&first, domain * 8, ctx->stream));
    GFX_CK(cudaMemsetAsync(first, 0x7f, domain * 8, ctx->stream));
    GFX_LAUNCH(k_first_batch, grid_of(ctx, n), 256, 0, ctx->stream, items_d, n, table_or_batch,
               first);
    GFX_LAUNCH(k_bitmask_keep, grid_of(ctx, n), 256, 0, ctx->stream, items_d, n, table_or_batch,
               first, keep_d);
    GFX_CK(cudaFreeAsync(first, ctx->stream));
  } else {  // history table of table_or_batch slots over batches of `batch` items
    const int64_t nb = (n + batch - 1) / batch;
    const int grid = grid_for(nb, 64, ctx->sm_count * 16);
    int64_t* tab;
    GFX_CK(cudaMallocAsync(&tab, (int64_t)grid * 64 * table_or_batch * 8, ctx->stream));
    GFX_LAUNCH(k_history_keep, grid, 64, 0, ctx->stream, items_d,
               n, table_or_batch, batch, tab, keep_d);
    GFX_CK(cudaFreeAsync(tab, ctx->stream));
  }
  GFX_CK(cudaGetLastError());
  GFX_CK(cudaStreamSynchronize(ctx->stream));
  return GFX_OK;
}

int gfx_atomic_min(gfx_ctx* ctx, int dtype, void* arr_d, const int64_t* idx_d, const void* vals_d,
                   int64_t k, uint8_t* won_d, void* pre_d) {
  GFX_REQUIRE(ctx && (k == 0 || (arr_d && idx_d && vals_d && won_d && pre_d)),
              "gfx_atomic_min: null argument");
  GFX_REQUIRE(dtype == 0 || dtype == 1, "atomic_min supports int32/int64 arrays (dtype %d)", dtype);
  GFX_CK(cudaSetDevice(ctx->device));
  if (k) {
    if (dtype == 0)
      GFX_TRY(run_atomic_min<int32_t>(ctx, (int32_t*)arr_d, idx_d, (const int32_t*)vals_d, k,
                                      won_d, (int32_t*)pre_d));
    else
      GFX_TRY(run_atomic_min<int64_t>(ctx, (int64_t*)arr_d, idx_d, (const int64_t*)vals_d, k,
                                      won_d, (int64_t*)pre_d));
  }
  GFX_CK(cudaGetLastError());
  GFX_CK(cudaStreamSynchronize(ctx->stream));
  return GFX_OK;
}

int gfx_atomic_add(gfx_ctx* ctx, int dtype, void* arr_d, const int64_t* idx_d, const void* vals_d,
                   double scalar, int64_t k) {
  GFX_REQUIRE(ctx && (k == 0 || (arr_d && idx_d)), "gfx_atomic_add: null argument");
  GFX_REQUIRE(dtype >= 0 && dtype <= 3, "atomic_add: unknown dtype %d", dtype);
  GFX_CK(cudaSetDevice(ctx->device));
  if (k) {
    const int gr = grid_of(ctx, k);
    switch (dtype) {
      case 0:
        GFX_LAUNCH(k_aadd<int32_t>, gr, 256, 0, ctx->stream, (int32_t*)arr_d, idx_d,
                   (const int32_t*)vals_d, (int32_t)scalar, k);
        break;
      case 1:
        GFX_LAUNCH(k_aadd<int64_t>, gr, 256, 0, ctx->stream, (int64_t*)arr_d, idx_d,
                   (const int64_t*)vals_d, (int64_t)scalar, k);
        break;
      case 2:
        GFX_LAUNCH(k_aadd<float>, gr, 256, 0, ctx->stream, (float*)arr_d, idx_d,
                   (const float*)vals_d, (float)scalar, k);
        break;
      default:
        GFX_LAUNCH(k_aadd<double>, gr, 256, 0, ctx->stream, (double*)arr_d, idx_d,
                   (const double*)vals_d, scalar, k);
    }
  }
  GFX_CK(cudaGetLastError());
  GFX_CK(cudaStreamSynchronize(ctx->stream));
  return GFX_OK;
}

int gfx_compare_and_swap(gfx_ctx* ctx, int dtype, void* arr_d, const int64_t* idx_d, int64_t k,
                         int64_t expected, const void* vals_d, int64_t scalar, uint8_t* won_d,
                         int64_t* pos_d) {
  GFX_REQUIRE(ctx && (k == 0 || (arr_d && idx_d && won_d && pos_d)),
              "gfx_compare_and_swap: null argument");
  GFX_REQUIRE(dtype == 0 || dtype == 1, "compare_and_swap supports int32/int64 arrays");
  GFX_CK(cudaSetDevice(ctx->device));
  if (k) {
    if (dtype == 0)
      GFX_TRY(run_cas<int32_t>(ctx, (int32_t*)arr_d, idx_d, k, (int32_t)expected,
                               (const int32_t*)vals_d, (int32_t)scalar, won_d, pos_d));
    else
      GFX_TRY(run_cas<int64_t>(ctx, (int64_t*)arr_d, idx_d, k, expected, (const int64_t*)vals_d,
                               scalar, won_d, pos_d));
  }
  GFX_CK(cudaGetLastError());
  GFX_CK(cudaStreamSynchronize(ctx->stream));
  return GFX_OK;
}

}  // extern "C"
