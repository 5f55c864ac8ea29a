// Bit-exact GPU R-MAT generator + canonical CSR builder + weight assignment.
//
// Reproduces, bit for bit, the reference input pipeline
//   generate_rmat(S, ef, seed)           generators.py:22-52
//   coo_to_csr(make_undirected=True)     graph.py:158-203
//   assign_random_weights(g, lo, hi, s)  graph.py:227-246
// by replaying numpy's PCG64 stream (XSL-RR 128/64, state advanced before
// each output) with O(log k) jump-ahead, so every thread starts at its own
// stream position.  random() = (next64 >> 11) * 2^-53; integers() for a
// power-of-two range uses the buffered 32-bit Lemire path without rejection
// (low half of each 64-bit draw first).
//
// The canonical CSR is a radix sort of (src << S | dst) keys + unique, which
// is exactly lexsort + dedup; self loops map to the sentinel key
// (n-1, n-1), which can never be a real undirected edge and sorts last.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <cuda_runtime.h>

#include "gfx_device.cuh"
#include "gfx_internal.cuh"

namespace gfx {

typedef unsigned __int128 u128;

__host__ __device__ __forceinline__ u128 mk128(uint64_t hi, uint64_t lo) {
  return ((u128)hi << 64) | lo;
}

__host__ __device__ __forceinline__ u128 pcg_mult() {
  return mk128(0x2360ED051FC65DA4ULL, 0x4385DF649FCCF645ULL);
}

__host__ __device__ __forceinline__ uint64_t pcg_out(u128 s) {
  uint64_t x = (uint64_t)(s >> 64) ^ (uint64_t)s;
  unsigned r = (unsigned)(s >> 122);
  return (x >> r) | (x << ((64u - r) & 63u));
}

// jump parameters: after k steps, s' = A*s + C (pcg_advance_lcg_128)
struct Jump {
  u128 a, c;
};

__host__ __device__ inline Jump jump_params(uint64_t k, u128 inc) {
  u128 cur_mult = pcg_mult(), cur_plus = inc, acc_mult = 1, acc_plus = 0;
  while (k) {
    if (k & 1) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    k >>= 1;
  }
  return {acc_mult, acc_plus};
}

__host__ __device__ __forceinline__ u128 apply_jump(const Jump& j, u128 s) { return j.a * s + j.c; }

constexpr int kRmatEPT = 16;  // edges per thread per level

__global__ void __launch_bounds__(256)
    k_rmat_keys(int scale, uint64_t m, uint64_t s_hi, uint64_t s_lo, uint64_t i_hi,
                uint64_t i_lo, uint64_t jm_a_hi, uint64_t jm_a_lo, uint64_t jm_c_hi,
                uint64_t jm_c_lo, double c0, double c1, double c2, int undirected,
                uint64_t* __restrict__ keys) {
  const u128 inc = mk128(i_hi, i_lo);
  const u128 mult = pcg_mult();
  const Jump jm = {mk128(jm_a_hi, jm_a_lo), mk128(jm_c_hi, jm_c_lo)};
  const uint64_t sentinel = (scale >= 32) ? ~0ull : ((1ull << (2 * scale)) - 1);
  for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t * kRmatEPT < m;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t i0 = t * kRmatEPT;
    const int cnt = (int)min((uint64_t)kRmatEPT, m - i0);
    u128 s = apply_jump(jump_params(i0, inc), mk128(s_hi, s_lo));
    const Jump jlevel = (cnt == kRmatEPT) ? jm : jump_params(m - cnt, inc);
    uint32_t src[kRmatEPT], dst[kRmatEPT];
#pragma unroll
    for (int j = 0; j < kRmatEPT; ++j) src[j] = dst[j] = 0;
    for (int level = 0; level < scale; ++level) {
#pragma unroll
      for (int j = 0; j < kRmatEPT; ++j) {
        if (j < cnt) {
          s = s * mult + inc;
          const double u = (double)(pcg_out(s) >> 11) * (1.0 / 9007199254740992.0);
          const unsigned q = (u >= c0) + (u >= c1) + (u >= c2);
          src[j] = (src[j] << 1) | (q >> 1);
          dst[j] = (dst[j] << 1) | (q & 1u);
        }
      }
      s = apply_jump(jlevel, s);
    }
#pragma unroll
    for (int j = 0; j < kRmatEPT; ++j) {
      if (j < cnt) {
        const uint64_t a = src[j], b = dst[j];
        if (undirected) {
          const bool loop = a == b;
          keys[2 * (i0 + j)] = loop ? sentinel : ((a << scale) | b);
          keys[2 * (i0 + j) + 1] = loop ? sentinel : ((b << scale) | a);
        } else {
          keys[i0 + j] = (a << scale) | b;
        }
      }
    }
  }
}

__global__ void k_csr_cols(const uint64_t* __restrict__ keys, int64_t M, int scale,
                           int32_t* __restrict__ col) {
  const uint64_t mask = (1ull << scale) - 1;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M;
       i += (int64_t)gridDim.x * blockDim.x)
    col[i] = (int32_t)(keys[i] & mask);
}

__global__ void k_csr_rows(const uint64_t* __restrict__ keys, int64_t M, int scale, int64_t n,
                           int64_t* __restrict__ row) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v <= n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t target = (uint64_t)v << scale;
    int64_t lo = 0, hi = M;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (keys[mid] < target) lo = mid + 1; else hi = mid;
    }
    row[v] = lo;
  }
}

// ---- weights -------------------------------------------------------------
// first slot of v's row whose neighbour is > v (upper-triangle start)
__device__ __forceinline__ int64_t upper_start(const int64_t* row, const int32_t* col, int64_t v) {
  int64_t lo = row[v], hi = row[v + 1];
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (col[mid] <= v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__global__ void k_upper_counts(const int64_t* __restrict__ row, const int32_t* __restrict__ col,
                               int64_t n, int64_t* __restrict__ cnt) {
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x)
    cnt[v] = row[v + 1] - upper_start(row, col, v);
}

// upper slots of v get lo + bounded(u32[rank]) with rank = base[v] + k.
// One warp per row: lane l takes ranks base+l, base+l+32, ...; it jumps once
// to its first draw, then every 32 ranks = 16 draws is one precomputed jump.
__global__ void k_upper_weights(const int64_t* __restrict__ row, const int32_t* __restrict__ col,
                                int64_t n, const int64_t* __restrict__ base, uint64_t s_hi,
                                uint64_t s_lo, uint64_t i_hi, uint64_t i_lo, int64_t lo_w,
                                uint64_t range1, int32_t* __restrict__ w) {
  const u128 inc = mk128(i_hi, i_lo);
  const u128 s0 = mk128(s_hi, s_lo);
  const Jump j16 = jump_params(16, inc);
  const int lane = threadIdx.x & 31;
  for (int64_t v = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; v < n;
       v += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t us = upper_start(row, col, v), ue = row[v + 1];
    if (us + lane >= ue) continue;
    const int64_t rank = base[v] + lane;
    // state after rank/2 draws; one more step yields draw rank/2
    u128 s = apply_jump(jump_params((uint64_t)(rank >> 1), inc), s0);
    const bool high = rank & 1;
    for (int64_t e = us + lane; e < ue; e += 32) {
      const uint64_t x64 = pcg_out(s * pcg_mult() + inc);
      const uint32_t x = high ? (uint32_t)(x64 >> 32) : (uint32_t)x64;
      w[e] = (int32_t)(lo_w + (int64_t)(((uint64_t)x * range1) >> 32));
      s = apply_jump(j16, s);
    }
  }
}

// lower slots (s > d) copy the weight of their mirror slot (d -> s); one
// warp per row, lanes binary-search their own mirrors
__global__ void k_lower_weights(const int64_t* __restrict__ row, const int32_t* __restrict__ col,
                                int64_t n, int32_t* __restrict__ w) {
  const int lane = threadIdx.x & 31;
  for (int64_t v = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; v < n;
       v += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t us = upper_start(row, col, v);
    for (int64_t e = row[v] + lane; e < us; e += 32) {
      const int32_t d = col[e];
      int64_t lo = row[d], hi = row[d + 1];
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (col[mid] < v) lo = mid + 1; else hi = mid;
      }
      w[e] = w[lo];
    }
  }
}

}  // namespace gfx

using namespace gfx;

extern "C" int gfx_rmat_keys(gfx_ctx* ctx, int scale, int edge_factor, const double* cum3,
                             uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                             uint64_t inc_lo, int make_undirected, uint64_t* keys_d,
                             int64_t* num_keys) {
  GFX_NVTX("gfx_rmat_keys");
  GFX_REQUIRE(ctx && cum3 && keys_d && num_keys, "gfx_rmat_keys: null argument");
  GFX_REQUIRE(scale >= 1 && scale <= 30, "gfx_rmat_keys: scale must be in [1, 30]");
  GFX_REQUIRE(edge_factor >= 1, "gfx_rmat_keys: edge_factor must be >= 1");
  GFX_CK(cudaSetDevice(ctx->device));
  const uint64_t m = (uint64_t)edge_factor << scale;
  const int64_t nkeys = (int64_t)(make_undirected ? 2 * m : m);
  const u128 inc = mk128(inc_hi, inc_lo);
  const Jump jm = jump_params(m - kRmatEPT, inc);
  const uint64_t threads = (m + kRmatEPT - 1) / kRmatEPT;
  const int grid = grid_for((int64_t)threads, 256, ctx->sm_count * 32);
  GFX_LAUNCH(k_rmat_keys, grid, 256, 0, ctx->stream, 
      scale, m, state_hi, state_lo, inc_hi, inc_lo, (uint64_t)(jm.a >> 64), (uint64_t)jm.a,
      (uint64_t)(jm.c >> 64), (uint64_t)jm.c, cum3[0], cum3[1], cum3[2], make_undirected, keys_d);
  GFX_CK(cudaGetLastError());

  // radix sort on the 2*scale key bits, then unique
  uint64_t* alt = nullptr;
  GFX_CK(cudaMalloc(&alt, sizeof(uint64_t) * nkeys));
  cub::DoubleBuffer<uint64_t> db(keys_d, alt);
  size_t tmp_bytes = 0, tmp2 = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, db, nkeys, 0, 2 * scale, ctx->stream);
  int64_t* d_count = nullptr;
  cub::DeviceSelect::Unique(nullptr, tmp2, db.Current(), db.Alternate(), d_count, nkeys,
                            ctx->stream);
  tmp_bytes = tmp_bytes > tmp2 ? tmp_bytes : tmp2;
  void* tmp = nullptr;
  cudaError_t e = cudaMalloc(&tmp, tmp_bytes + 64);
  if (e != cudaSuccess) {
    cudaFree(alt);
    return cuda_status(e, "rmat sort temp", __FILE__, __LINE__);
  }
  d_count = reinterpret_cast<int64_t*>(static_cast<char*>(tmp) + ((tmp_bytes + 15) / 16) * 16);
  cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, db, nkeys, 0, 2 * scale, ctx->stream);
  uint64_t* sorted = db.Current();
  uint64_t* uniq = (sorted == keys_d) ? alt : keys_d;
  cub::DeviceSelect::Unique(tmp, tmp_bytes, sorted, uniq, d_count, nkeys, ctx->stream);
  int64_t count = 0;
  cudaMemcpyAsync(&count, d_count, 8, cudaMemcpyDeviceToHost, ctx->stream);
  e = cudaStreamSynchronize(ctx->stream);
  if (e == cudaSuccess && uniq != keys_d)
    e = cudaMemcpyAsync(keys_d, uniq, sizeof(uint64_t) * count, cudaMemcpyDeviceToDevice,
                        ctx->stream);
  uint64_t last = 0;
  if (e == cudaSuccess && count > 0 && make_undirected) {
    cudaMemcpyAsync(&last, keys_d + count - 1, 8, cudaMemcpyDeviceToHost, ctx->stream);
    e = cudaStreamSynchronize(ctx->stream);
    const uint64_t sentinel = (1ull << (2 * scale)) - 1;
    if (last == sentinel) --count;
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
  cudaFree(tmp);
  cudaFree(alt);
  if (e != cudaSuccess) return cuda_status(e, "rmat unique", __FILE__, __LINE__);
  *num_keys = count;
  return GFX_OK;
}

extern "C" int gfx_keys_to_csr(gfx_ctx* ctx, const uint64_t* keys_d, int64_t num_keys, int scale,
                               int64_t* row_d, int32_t* col_d) {
  GFX_NVTX("gfx_keys_to_csr");
  GFX_REQUIRE(ctx && keys_d && row_d && (num_keys == 0 || col_d), "gfx_keys_to_csr: null argument");
  GFX_CK(cudaSetDevice(ctx->device));
  const int64_t n = 1ll << scale;
  GFX_LAUNCH(k_csr_cols, grid_for(num_keys, 256, ctx->sm_count * 32), 256, 0, ctx->stream, 
      keys_d, num_keys, scale, col_d);
  GFX_LAUNCH(k_csr_rows, grid_for(n + 1, 256, ctx->sm_count * 32), 256, 0, ctx->stream, 
      keys_d, num_keys, scale, n, row_d);
  GFX_CK(cudaGetLastError());
  GFX_CK(cudaStreamSynchronize(ctx->stream));
  return GFX_OK;
}

extern "C" int gfx_assign_weights(gfx_graph* g, int64_t lo, int64_t hi, uint64_t state_hi,
                                  uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                                  int32_t* w_d) {
  GFX_NVTX("gfx_assign_weights");
  GFX_REQUIRE(g && w_d, "gfx_assign_weights: null argument");
  GFX_REQUIRE(lo >= 1 && lo <= hi, "need 1 <= lo <= hi");
  GFX_REQUIRE(g->flags & GFX_GRAPH_UNDIRECTED,
              "gfx_assign_weights: the device builder handles canonical undirected graphs");
  const uint64_t range1 = (uint64_t)(hi - lo) + 1;
  GFX_REQUIRE((range1 & (range1 - 1)) == 0 && range1 <= (1ull << 31),
              "gfx_assign_weights: the device stream replay needs a power-of-two range "
              "(numpy's Lemire sampler rejects otherwise); got [%lld, %lld]",
              (long long)lo, (long long)hi);
  gfx_ctx* ctx = g->ctx;
  GFX_CK(cudaSetDevice(ctx->device));
  const int64_t n = g->n;
  if (g->m == 0) return GFX_OK;
  int64_t* cnt = nullptr;
  GFX_TRY(scratch_t(g, "w_cnt", n + 1, &cnt));
  int64_t* base = nullptr;
  GFX_TRY(scratch_t(g, "w_base", n + 1, &base));
  const int grid = grid_for(n, 256, ctx->sm_count * 16);
  GFX_LAUNCH(k_upper_counts, grid, 256, 0, ctx->stream, g->row, g->col, n, cnt);
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, base, n, ctx->stream);
  void* tmp = nullptr;
  GFX_TRY(scratch(g, "w_scan_tmp", tb, &tmp));
  cub::DeviceScan::ExclusiveSum(tmp, tb, cnt, base, n, ctx->stream);
  if (range1 == 1) {
    GFX_TRY(fill_i32(ctx, w_d, (int32_t)lo, g->m));
  } else {
    const int wgrid = grid_for(n * 32, 256, ctx->sm_count * 16);
    GFX_LAUNCH(k_upper_weights, wgrid, 256, 0, ctx->stream, g->row, g->col, n, base, state_hi,
               state_lo, inc_hi, inc_lo, lo, range1, w_d);
    GFX_LAUNCH(k_lower_weights, wgrid, 256, 0, ctx->stream, g->row, g->col, n, w_d);
  }
  GFX_CK(cudaGetLastError());
  GFX_CK(cudaStreamSynchronize(ctx->stream));
  return GFX_OK;
}
