// libgfx core: errors, context, graph handle, scratch, fills, and the fused
// degree-scan + tile partition shared by every load-balanced expansion.
#include <cuda_runtime.h>
#include <cstdlib>

#include <algorithm>
#include <atomic>
#include <cstring>

#include "gfx_device.cuh"
#include "gfx_internal.cuh"
#include "gfx_scan.cuh"

namespace gfx {

static thread_local std::string g_last_error;
static std::atomic<long long> g_launches{0};

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
}

int cuda_status(cudaError_t e, const char* what, const char* file, int line) {
  set_error("CUDA error %s (%s) at %s:%d in %s", cudaGetErrorName(e), cudaGetErrorString(e),
            file, line, what);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();  // clear sticky-free allocation error
    return GFX_ENOMEM;
  }
  return GFX_ECUDA;
}

int scratch(gfx_graph* g, const char* name, size_t bytes, void** out, bool* fresh) {
  auto& b = g->scratch[name];
  if (fresh) *fresh = false;
  if (b.bytes < bytes) {
    if (fresh) *fresh = true;
    if (b.ptr) {
      GFX_CK(cudaStreamSynchronize(g->ctx->stream));
      GFX_CK(cudaFree(b.ptr));
      b.ptr = nullptr;
      b.bytes = 0;
    }
    size_t want = std::max<size_t>(bytes, 256);
    GFX_CK(cudaMalloc(&b.ptr, want));
    b.bytes = want;
  }
  *out = b.ptr;
  return GFX_OK;
}

unsigned int next_epoch(gfx_graph* g, unsigned int** counter, bool* wrapped) {
  g->epoch = (g->epoch + 1) % kScanEpochs;
  *wrapped = false;
  if (g->epoch == 0) {
    // wrapped: every per-epoch counter and tile status must be cleared
    cudaMemsetAsync(g->tile_counters, 0, sizeof(unsigned int) * kScanEpochs, g->ctx->stream);
    g->epoch = 1;
    *wrapped = true;
  }
  *counter = g->tile_counters + g->epoch;
  return g->epoch;
}

int read_counters(gfx_graph* g, Counters* host) {
  auto* pin = static_cast<Counters*>(g->ctx->pinned);
  GFX_CK(cudaMemcpyAsync(pin, g->counters, sizeof(Counters), cudaMemcpyDeviceToHost,
                         g->ctx->stream));
  GFX_CK(cudaStreamSynchronize(g->ctx->stream));
  *host = *pin;
  return GFX_OK;
}

int zero_counters(gfx_graph* g) {
  GFX_CK(cudaMemsetAsync(g->counters, 0, sizeof(Counters), g->ctx->stream));
  return GFX_OK;
}

template <typename T>
__global__ void k_fill(T* __restrict__ p, T v, int64_t count) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; i < count; i += stride) p[i] = v;
}

int fill_i32(gfx_ctx* ctx, int32_t* p, int32_t v, int64_t count) {
  if (count <= 0) return GFX_OK;
  GFX_LAUNCH((k_fill<int32_t>), grid_for(count, 256, ctx->sm_count * 16), 256, 0, ctx->stream, p, v, count);
  GFX_CK(cudaGetLastError());
  return GFX_OK;
}

int fill_f64(gfx_ctx* ctx, double* p, double v, int64_t count) {
  if (count <= 0) return GFX_OK;
  GFX_LAUNCH((k_fill<double>), grid_for(count, 256, ctx->sm_count * 16), 256, 0, ctx->stream, p, v, count);
  GFX_CK(cudaGetLastError());
  return GFX_OK;
}

// Standalone fused degree scan (dynamic tile ids; see gfx_scan.cuh).
__global__ void __launch_bounds__(kScanBlock)
    k_degree_scan(const int32_t* __restrict__ F, const unsigned long long* __restrict__ nf_d,
                  const int64_t* __restrict__ row, int64_t* __restrict__ scan,
                  int64_t* __restrict__ rowbase, int32_t* __restrict__ part,
                  unsigned long long* status, unsigned int* tile_counter, unsigned epoch,
                  Counters* __restrict__ ctr) {
  const int64_t nf = (int64_t)*nf_d;
  const int64_t ntiles = nf > 0 ? (nf + kScanTileItems - 1) / kScanTileItems : 1;
  __shared__ unsigned s_tile;
  __shared__ ScanSmem sm;
  for (;;) {
    if (threadIdx.x == 0) s_tile = atomicAdd(tile_counter, 1u);
    __syncthreads();
    const int64_t tile = s_tile;
    if (tile >= ntiles) break;
    scan_tile(tile, ntiles, F, nf, row, scan, rowbase, part, status, epoch, ctr, sm);
  }
}

int launch_degree_scan(gfx_graph* g, const int32_t* F, const unsigned long long* nf_d,
                       int64_t nf_max, const int64_t* row, int64_t* scan, int64_t* rowbase,
                       int32_t* part, Counters* counters) {
  gfx_ctx* ctx = g->ctx;
  int64_t tiles_max = std::max<int64_t>(1, (nf_max + kScanTileItems - 1) / kScanTileItems);
  void* sp = nullptr;
  bool fresh = false;
  GFX_TRY(scratch(g, "scan_status", (size_t)tiles_max * 8, &sp, &fresh));
  auto* status = static_cast<unsigned long long*>(sp);
  unsigned int* tc = nullptr;
  bool wrapped = false;
  unsigned ep = next_epoch(g, &tc, &wrapped);
  if (fresh || wrapped) {
    // clear the whole (possibly larger) buffer so no stale tag survives
    GFX_CK(cudaMemsetAsync(status, 0, g->scratch["scan_status"].bytes, ctx->stream));
  }
  int grid = (int)std::min<int64_t>(tiles_max, (int64_t)ctx->sm_count * 4);
  GFX_LAUNCH(k_degree_scan, grid, kScanBlock, 0, ctx->stream, F, nf_d, row, scan, rowbase, part, status, tc,
                                                      ep, counters);
  GFX_CK(cudaGetLastError());
  return GFX_OK;
}

// graph-constant: bitmap of vertices with nonzero (in-)degree
__global__ void k_nonzero_bitmap(const int64_t* __restrict__ row, int64_t n, int64_t words,
                                 uint32_t* __restrict__ bm) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (; i < words * 32; i += stride) {
    bool nz = i < n && row[i + 1] > row[i];
    unsigned b = __ballot_sync(0xffffffffu, nz);
    if ((threadIdx.x & 31) == 0) bm[i >> 5] = b;
  }
}

// max out-degree -> out[0], number of vertices with out-degree > 0 -> out[-1]
__global__ void k_max_degree(const int64_t* __restrict__ row, int64_t n,
                             unsigned long long* __restrict__ out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  unsigned long long best = 0, nnz = 0;
  for (; i < n; i += stride) {
    unsigned long long d = (unsigned long long)(row[i + 1] - row[i]);
    best = d > best ? d : best;
    nnz += d > 0;
  }
  for (int o = 16; o; o >>= 1) {
    unsigned long long y = __shfl_xor_sync(0xffffffffu, best, o);
    best = y > best ? y : best;
    nnz += __shfl_xor_sync(0xffffffffu, nnz, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(out, best);
    atomicAdd(out - 1, nnz);
  }
}

int build_nonzero_bitmap(gfx_graph* g, const int64_t* row, const char* name) {
  uint32_t* bm = nullptr;
  GFX_TRY(scratch_t(g, name, (size_t)g->words, &bm));
  int64_t threads = g->words * 32;
  GFX_LAUNCH(k_nonzero_bitmap, grid_for(threads, 256, g->ctx->sm_count * 16), 256, 0, g->ctx->stream, 
      row, g->n, g->words, bm);
  GFX_CK(cudaGetLastError());
  return GFX_OK;
}

// Persisting-L2 access window on the stream for [base, base + bytes): random-
// probe targets (SSSP distances, PageRank contributions) stay L2-resident
// while the adjacency streams through with evict-first hints.  When bytes
// exceed the persisting capacity, hitRatio spreads the capacity over the
// whole window.  on == false removes the window and the carve-out.
void l2_window(gfx_ctx* ctx, void* base, size_t bytes, bool on) {
  static size_t max_persist = (size_t)-1;
  if (max_persist == (size_t)-1) {
    cudaDeviceProp prop{};
    if (cudaGetDeviceProperties(&prop, ctx->device) != cudaSuccess) {
      max_persist = 0;
    } else {
      max_persist = (size_t)prop.persistingL2CacheMaxSize;
    }
    cudaGetLastError();
  }
  if (!max_persist || getenv("GFX_NO_L2_PERSIST")) return;
  cudaStreamAttrValue attr{};
  if (on) {
    attr.accessPolicyWindow.base_ptr = base;
    static size_t max_window = 0;
    if (!max_window) {
      int w = 0;
      cudaDeviceGetAttribute(&w, cudaDevAttrMaxAccessPolicyWindowSize, ctx->device);
      max_window = w > 0 ? (size_t)w : max_persist;
    }
    const size_t win = bytes < max_window ? bytes : max_window;
    attr.accessPolicyWindow.num_bytes = win;
    attr.accessPolicyWindow.hitRatio = win <= max_persist ? 1.0f : (float)max_persist / (float)win;
    attr.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  } else {
    attr.accessPolicyWindow.num_bytes = 0;
  }
  // the set-aside is taken for the duration of the call only: a persisting
  // carve-out left behind would shrink L2 for every later kernel
  if (on) cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, max_persist);
  cudaStreamSetAttribute(ctx->stream, cudaStreamAttributeAccessPolicyWindow, &attr);
  if (!on) {
    cudaCtxResetPersistingL2Cache();
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, 0);
  }
  cudaGetLastError();
}

}  // namespace gfx

using namespace gfx;

extern "C" {

int gfx_version(void) { return 1; }

int64_t gfx_launch_count(void) { return (int64_t)g_launches.load(); }

int gfx_ctx_set_stats(gfx_ctx* c, int detail) {
  GFX_REQUIRE(c, "null ctx");
  c->stats_detail = detail;
  return GFX_OK;
}

int gfx_ctx_set_timing(gfx_ctx* c, int enabled) {
  GFX_REQUIRE(c, "null ctx");
  c->timing = enabled != 0;
  return GFX_OK;
}

const char* gfx_last_error(void) { return g_last_error.c_str(); }

int gfx_ctx_create(int device, void* stream, gfx_ctx** out) {
  GFX_REQUIRE(out != nullptr, "gfx_ctx_create: out is NULL");
  int ndev = 0;
  GFX_CK(cudaGetDeviceCount(&ndev));
  GFX_REQUIRE(device >= 0 && device < ndev, "gfx_ctx_create: device %d out of range (%d devices)",
              device, ndev);
  GFX_CK(cudaSetDevice(device));
  auto* c = new gfx_ctx();
  c->device = device;
  // NULL selects the legacy default stream, which orders with torch's
  // default stream (both are the context's NULL stream at driver level)
  c->stream = static_cast<cudaStream_t>(stream);
  GFX_CK(cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, device));
  GFX_CK(cudaEventCreate(&c->ev0));
  GFX_CK(cudaEventCreate(&c->ev1));
  GFX_CK(cudaEventCreate(&c->lev0));
  GFX_CK(cudaEventCreate(&c->lev1));
  GFX_CK(cudaMallocHost(&c->pinned, 4096));
  GFX_CK(cudaStreamSynchronize(c->stream));
  *out = c;
  return GFX_OK;
}

int gfx_ctx_destroy(gfx_ctx* c) {
  if (!c) return GFX_OK;
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  cudaFreeHost(c->pinned);
  cudaEventDestroy(c->ev0);
  cudaEventDestroy(c->ev1);
  cudaEventDestroy(c->lev0);
  cudaEventDestroy(c->lev1);
  if (c->own_stream) cudaStreamDestroy(c->stream);
  delete c;
  return GFX_OK;
}

int gfx_ctx_sync(gfx_ctx* c) {
  GFX_REQUIRE(c, "null ctx");
  GFX_CK(cudaStreamSynchronize(c->stream));
  return GFX_OK;
}

int gfx_ctx_sm_count(gfx_ctx* c) { return c ? c->sm_count : 0; }

int gfx_graph_create(gfx_ctx* ctx, int64_t n, int64_t m, const int64_t* row_d,
                     const int32_t* col_d, const int32_t* w_d, int flags, gfx_graph** out) {
  GFX_REQUIRE(ctx && out, "gfx_graph_create: null argument");
  GFX_REQUIRE(n >= 0 && n < (int64_t)INT32_MAX, "gfx_graph_create: n=%lld out of int32 range",
              (long long)n);
  GFX_REQUIRE(m >= 0, "gfx_graph_create: m < 0");
  GFX_REQUIRE(row_d != nullptr, "gfx_graph_create: row_offsets is NULL");
  GFX_REQUIRE(m == 0 || col_d != nullptr, "gfx_graph_create: column_indices is NULL");
  GFX_CK(cudaSetDevice(ctx->device));
  auto* g = new gfx_graph();
  g->ctx = ctx;
  g->n = n;
  g->m = m;
  g->row = row_d;
  g->col = col_d;
  g->w = w_d;
  g->flags = flags;
  g->words = (n + 31) / 32;
  if (flags & GFX_GRAPH_UNDIRECTED) {
    g->rrow = row_d;
    g->rcol = col_d;
  }
  int st = cudaMalloc(&g->counters, sizeof(Counters) * 4) == cudaSuccess ? GFX_OK : GFX_ENOMEM;
  if (st != GFX_OK) {
    delete g;
    set_error("gfx_graph_create: cannot allocate counters");
    return st;
  }
  cudaMemsetAsync(g->counters, 0, sizeof(Counters) * 4, ctx->stream);
  if (cudaMalloc(&g->tile_counters, sizeof(unsigned int) * kScanEpochs) != cudaSuccess) {
    cudaFree(g->counters);
    delete g;
    set_error("gfx_graph_create: cannot allocate tile counters");
    return GFX_ENOMEM;
  }
  cudaMemsetAsync(g->tile_counters, 0, sizeof(unsigned int) * kScanEpochs, ctx->stream);
  // max degree + nonzero bitmaps (graph constants)
  auto* pin = static_cast<unsigned long long*>(ctx->pinned);
  unsigned long long* dmax = reinterpret_cast<unsigned long long*>(g->counters) + 31;
  cudaMemsetAsync(dmax - 1, 0, 16, ctx->stream);
  if (n > 0) {
    GFX_LAUNCH(k_max_degree, grid_for(n, 256, ctx->sm_count * 8), 256, 0, ctx->stream, row_d, n, dmax);
    st = build_nonzero_bitmap(g, row_d, "nz_out");
    if (st != GFX_OK) {
      delete g;
      return st;
    }
  }
  cudaMemcpyAsync(pin, dmax - 1, 16, cudaMemcpyDeviceToHost, ctx->stream);
  cudaError_t e = cudaStreamSynchronize(ctx->stream);
  if (e != cudaSuccess) {
    delete g;
    return cuda_status(e, "graph create", __FILE__, __LINE__);
  }
  g->nnz_vertices = (int64_t)pin[0];
  g->max_deg = (int64_t)pin[1];
  *out = g;
  return GFX_OK;
}

int gfx_graph_set_reverse(gfx_graph* g, const int64_t* rrow_d, const int32_t* rcol_d) {
  GFX_REQUIRE(g && rrow_d && (g->m == 0 || rcol_d), "gfx_graph_set_reverse: null argument");
  g->rrow = rrow_d;
  g->rcol = rcol_d;
  if (g->n > 0) GFX_TRY(build_nonzero_bitmap(g, rrow_d, "nz_in"));
  GFX_CK(cudaStreamSynchronize(g->ctx->stream));
  return GFX_OK;
}

int gfx_graph_destroy(gfx_graph* g) {
  if (!g) return GFX_OK;
  cudaSetDevice(g->ctx->device);
  cudaStreamSynchronize(g->ctx->stream);
  for (auto& kv : g->scratch) cudaFree(kv.second.ptr);
  cudaFree(g->counters);
  cudaFree(g->tile_counters);
  delete g;
  return GFX_OK;
}

int64_t gfx_graph_max_degree(gfx_graph* g) { return g ? g->max_deg : -1; }

int gfx_graph_refresh(gfx_graph* g) {
  GFX_REQUIRE(g, "gfx_graph_refresh: null graph");
  gfx_ctx* ctx = g->ctx;
  GFX_CK(cudaSetDevice(ctx->device));
  // the caller rewrote the borrowed arrays in place (same n, m): recompute
  // every graph constant derived from them, keep the scratch allocations
  unsigned long long* dmax = reinterpret_cast<unsigned long long*>(g->counters) + 31;
  GFX_CK(cudaMemsetAsync(dmax - 1, 0, 16, ctx->stream));
  if (g->n > 0) {
    GFX_LAUNCH(k_max_degree, grid_for(g->n, 256, ctx->sm_count * 8), 256, 0, ctx->stream, g->row,
               g->n, dmax);
    GFX_TRY(build_nonzero_bitmap(g, g->row, "nz_out"));
    if (!(g->flags & GFX_GRAPH_UNDIRECTED) && g->rrow)
      GFX_TRY(build_nonzero_bitmap(g, g->rrow, "nz_in"));
    GFX_TRY(refresh_pull_heads(g));
  }
  g->m_oriented = -1;  // the oriented CSR (TC) is rebuilt on next use
  GFX_CK(cudaStreamSynchronize(ctx->stream));
  for (auto it = g->scratch.begin(); it != g->scratch.end();) {  // PageRank chunk table
    if (it->first.rfind("keep_pr_", 0) == 0) {
      cudaFree(it->second.ptr);
      it = g->scratch.erase(it);
    } else {
      ++it;
    }
  }
  g->w8_state = 0;     // and the compact weight copy (SSSP)
  auto* pin = static_cast<unsigned long long*>(ctx->pinned);
  GFX_CK(cudaMemcpyAsync(pin, dmax - 1, 16, cudaMemcpyDeviceToHost, ctx->stream));
  GFX_CK(cudaStreamSynchronize(ctx->stream));
  g->nnz_vertices = (int64_t)pin[0];
  g->max_deg = (int64_t)pin[1];
  return GFX_OK;
}

int gfx_graph_trim(gfx_graph* g) {
  GFX_REQUIRE(g, "null graph");
  GFX_CK(cudaStreamSynchronize(g->ctx->stream));
  for (auto it = g->scratch.begin(); it != g->scratch.end();) {
    if (it->first.rfind("nz_", 0) == 0 || it->first.rfind("keep_", 0) == 0) {
      ++it;
      continue;
    }
    cudaFree(it->second.ptr);
    it = g->scratch.erase(it);
  }
  return GFX_OK;
}

}  // extern "C"
