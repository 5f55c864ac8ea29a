// Internal declarations shared by the libgfx translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/gfx.h"
#include <nvtx3/nvToolsExt.h>

namespace gfx {

// ---------------------------------------------------------------------------
// error plumbing: thread-local message, status codes from gfx.h
// ---------------------------------------------------------------------------
void set_error(const char* fmt, ...);
int cuda_status(cudaError_t e, const char* what, const char* file, int line);

#define GFX_CK(call)                                                            \
  do {                                                                          \
    cudaError_t _e = (call);                                                    \
    if (_e != cudaSuccess) return ::gfx::cuda_status(_e, #call, __FILE__, __LINE__); \
  } while (0)

// NVTX range over a C-ABI entry point (header-only NVTX v3: a no-op unless a
// profiler injects itself, e.g. nsys / ncu --nvtx)
struct NvtxScope {
  explicit NvtxScope(const char* name) { nvtxRangePushA(name); }
  ~NvtxScope() { nvtxRangePop(); }
};
#define GFX_NVTX(name) ::gfx::NvtxScope gfx_nvtx_scope_(name)

// every kernel launch goes through GFX_LAUNCH so gfx_launch_count() is exact
void count_launch();
#define GFX_LAUNCH(K, G, B, S, ST, ...)       \
  do {                                        \
    K<<<(G), (B), (S), (ST)>>>(__VA_ARGS__);  \
    ::gfx::count_launch();                    \
  } while (0)

#define GFX_TRY(expr)            \
  do {                           \
    int _s = (expr);             \
    if (_s != GFX_OK) return _s; \
  } while (0)

#define GFX_REQUIRE(cond, ...)         \
  do {                                 \
    if (!(cond)) {                     \
      ::gfx::set_error(__VA_ARGS__);   \
      return GFX_EINVAL;               \
    }                                  \
  } while (0)

// ---------------------------------------------------------------------------
// device-side counters block (one per graph, mirrored in pinned host memory)
// ---------------------------------------------------------------------------
struct Counters {
  unsigned long long out_len;    // items appended to the output queue
  unsigned long long edges;      // expansion slots / in-degree sums this step
  unsigned long long total;      // scan total (expansion size)
  unsigned long long ntiles;     // expansion tiles
  unsigned long long aux0;       // kernel-specific
  unsigned long long aux1;
  unsigned long long aux2;
  unsigned long long aux3;
};

struct gfx_buffer {
  void* ptr = nullptr;
  size_t bytes = 0;
};

}  // namespace gfx

struct gfx_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int sm_count = 148;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  void* pinned = nullptr;  // 4 KB pinned host staging
  bool timing = false;     // per-iteration events
  int stats_detail = 1;    // 0: skip the statistics post-passes (E_r, pull edges)
  cudaEvent_t lev0 = nullptr, lev1 = nullptr;
};

struct gfx_graph {
  gfx_ctx* ctx = nullptr;
  int64_t n = 0, m = 0;
  const int64_t* row = nullptr;
  const int32_t* col = nullptr;
  const int32_t* w = nullptr;
  const int64_t* rrow = nullptr;  // reverse adjacency (== row/col if undirected)
  const int32_t* rcol = nullptr;
  const int64_t* reid = nullptr;  // forward slot of each reverse slot (gfx_graph_build_csc)
  int flags = 0;
  int64_t max_deg = 0;
  int64_t nnz_vertices = 0;       // vertices with out-degree > 0
  int64_t words = 0;              // ceil(n/32)
  std::unordered_map<std::string, gfx::gfx_buffer> scratch;
  gfx::Counters* counters = nullptr;  // device
  // oriented CSR for TC
  int64_t m_oriented = -1;
  // compact 8-bit copy of the weights (SSSP streams 5 instead of 8 bytes per
  // slot when every weight fits 0..255): 0 unknown, 1 built ("keep_w8"), 2 no
  int w8_state = 0;
  // decoupled look-back bookkeeping (per graph): epoch tags + per-epoch
  // dynamic tile counters, both cleared when the epoch wraps
  unsigned int epoch = 0;
  unsigned int* tile_counters = nullptr;
};

namespace gfx {

constexpr int kScanEpochs = 1 << 14;  // matches the 14-bit status tag

// lazily allocated, graph-owned scratch buffer (never shrinks)
int scratch(gfx_graph* g, const char* name, size_t bytes, void** out, bool* fresh = nullptr);
template <typename T>
inline int scratch_t(gfx_graph* g, const char* name, size_t count, T** out) {
  return scratch(g, name, count * sizeof(T), reinterpret_cast<void**>(out));
}

// next decoupled-look-back epoch; returns the per-epoch tile counter and
// whether the epoch wrapped (status buffers must then be cleared)
unsigned int next_epoch(gfx_graph* g, unsigned int** counter, bool* wrapped);

// read the counters block to host (stream-synchronous)
int read_counters(gfx_graph* g, Counters* host);
int zero_counters(gfx_graph* g);

// fills
int fill_i32(gfx_ctx* ctx, int32_t* p, int32_t v, int64_t count);
int fill_f64(gfx_ctx* ctx, double* p, double v, int64_t count);

// grid helpers
inline int grid_for(int64_t items, int block, int cap_blocks) {
  int64_t b = (items + block - 1) / block;
  if (b < 1) b = 1;
  if (b > cap_blocks) b = cap_blocks;
  return static_cast<int>(b);
}

// the degree-scan + tile partition used by every load-balanced expansion
// (reference load_balance.py:105-113 compute_scan_offsets and :157-176
// plan_lb_output, fused).  Inputs: frontier ids F[0..nf) (nf read from
// device *nf_d), CSR row offsets.  Outputs: scan[0..nf] exclusive prefix of
// degrees, rowbase[i] = row[F[i]], part[k] = item holding slot k*kTile,
// counters->total / ntiles.
constexpr int kTile = 512;           // expansion units per (warp) tile
// Each frontier item weighs kItemUnits units plus one per slot, so a tile
// never holds more than ~32 items (merge-path style: slots + items balanced)
constexpr int kItemUnits = 16;
inline int64_t part_capacity(int64_t m, int64_t n) {
  return (m + (int64_t)kItemUnits * (n + 1)) / kTile + 8;
}
constexpr int kScanBlock = 256;
constexpr int kScanItems = 8;        // items per thread in the scan
constexpr int kScanTileItems = kScanBlock * kScanItems;

// persisting-L2 window over a random-probe target (on/off, see gfx_core.cu)
void l2_window(gfx_ctx* ctx, void* base, size_t bytes, bool on);

// recompute the pull head array (first in-neighbour per vertex) if the
// graph has one (gfx_graph_refresh)
int refresh_pull_heads(gfx_graph* g);

// reached count and E_r from an int32 label array (UNVISITED = INT32_MAX)
int reached_stats(gfx_graph* g, const int32_t* labels, int64_t* reached, int64_t* edges);

// push-only BFS keeping each level's frontier: order[off[d], off[d+1])
// slots (optional): slots[d] = sum of out-degrees of level d
int bfs_push_levels(gfx_graph* g, int64_t source, int32_t* labels, int32_t* preds,
                    std::vector<int64_t>* off, int32_t** order_out,
                    std::vector<int64_t>* slots = nullptr);
// the same level lists from the direction-optimising persistent BFS
int bfs_do_levels(gfx_graph* g, int64_t source, int32_t* labels, int32_t* preds,
                  std::vector<int64_t>* off, int32_t** order_out,
                  std::vector<int64_t>* slots = nullptr);
// identity frontier 0..n-1 (graph-constant scratch)
int iota_frontier(gfx_graph* g, int32_t** out);

int launch_degree_scan(gfx_graph* g, const int32_t* F, const unsigned long long* nf_d,
                       int64_t nf_max, const int64_t* row, int64_t* scan,
                       int64_t* rowbase, int32_t* part, Counters* counters);

}  // namespace gfx
