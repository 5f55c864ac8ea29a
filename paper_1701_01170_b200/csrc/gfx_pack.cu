// Compressed CSR column stream for host<->device transfer (PCIe-bound paths).
//
// The column ids of a CSR are sorted within rows, so consecutive slots differ
// by small amounts except at row starts.  The packed form stores the
// zigzag-encoded difference to the previous slot (globally, so decoding is one
// inclusive prefix sum) in a StreamVByte-like layout: per slot a 2-bit length
// code (1..4 bytes) in a control stream and the value's low bytes in a data
// stream, with the data byte offset of every 1024-slot block kept so blocks
// decode independently (one warp per block).  On R-MAT ef16 this is ~1.9
// bytes per slot instead of 4 (int32) or 8 (the reference's int64), so the
// host->device copy of a graph -- the end-to-end bound -- moves about half
// the bytes.  Decoding is two HBM-bandwidth passes on the device.
#include <algorithm>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>

#include "gfx_device.cuh"
#include "gfx_internal.cuh"

namespace gfx {

constexpr int kPackBlock = 1024;  // slots per independently decodable block

__device__ __forceinline__ uint32_t zz_len(uint32_t z) {
  return 1u + (z >= (1u << 8)) + (z >= (1u << 16)) + (z >= (1u << 24));
}

// zigzag of the difference to the previous element (int32 column ids, or
// int64 row offsets whose differences -- the degrees -- fit 32 bits)
template <class T>
__device__ __forceinline__ uint32_t zz_delta(const T* __restrict__ col, int64_t j) {
  const T prev = j ? col[j - 1] : T(0);
  const int32_t d = (int32_t)(col[j] - prev);
  return ((uint32_t)d << 1) ^ (uint32_t)(d >> 31);
}

// pass 1: data bytes per block (warp per block)
template <class T>
__global__ void k_pack_sizes(const T* __restrict__ col, int64_t m,
                             int64_t* __restrict__ bsize) {
  const int lane = threadIdx.x & 31;
  const int64_t nb = (m + kPackBlock - 1) / kPackBlock;
  for (int64_t b = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; b < nb;
       b += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t j0 = b * kPackBlock, j1 = min(j0 + kPackBlock, m);
    unsigned long long s = 0;
    for (int64_t j = j0 + lane; j < j1; j += 32) s += zz_len(zz_delta(col, j));
    s = warp_sum_u64(s);
    if (lane == 0) bsize[b] = (int64_t)s;
  }
}

// pass 2: control and data streams (warp per block; lanes take 32 slots at a
// time, a warp scan of the lengths places each value's bytes)
template <class T>
__global__ void k_pack_write(const T* __restrict__ col, int64_t m,
                             const int64_t* __restrict__ boff, uint8_t* __restrict__ ctrl,
                             uint8_t* __restrict__ data) {
  const int lane = threadIdx.x & 31;
  const int64_t nb = (m + kPackBlock - 1) / kPackBlock;
  for (int64_t b = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; b < nb;
       b += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t j0 = b * kPackBlock, j1 = min(j0 + kPackBlock, m);
    int64_t pos = boff[b];
    for (int64_t jb = j0; jb < j1; jb += 32) {
      const int64_t j = jb + lane;
      uint32_t z = 0, len = 0;
      if (j < j1) {
        z = zz_delta(col, j);
        len = zz_len(z);
      }
      int tot;
      const int off = warp_excl_scan((int)len, lane, &tot);
      for (uint32_t k = 0; k < len; ++k) data[pos + off + k] = (uint8_t)(z >> (8 * k));
      // 4 codes per control byte: lanes 4q..4q+3 -> byte (j >> 2)
      const uint32_t code = len ? len - 1 : 0;
      uint32_t packed = code << (2 * (lane & 3));
      packed |= __shfl_down_sync(0xffffffffu, packed, 1);
      packed |= __shfl_down_sync(0xffffffffu, packed, 2);
      if ((lane & 3) == 0 && j < j1) ctrl[j >> 2] = (uint8_t)packed;
      pos += tot;
    }
  }
}

// decode: warp per block -> zigzag deltas decoded to int32 differences
template <class T>
__global__ void k_unpack_deltas(const uint8_t* __restrict__ ctrl, const uint8_t* __restrict__ data,
                                const int64_t* __restrict__ boff, int64_t m, T* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t nb = (m + kPackBlock - 1) / kPackBlock;
  for (int64_t b = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; b < nb;
       b += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t j0 = b * kPackBlock, j1 = min(j0 + kPackBlock, m);
    int64_t pos = boff[b];
    for (int64_t jb = j0; jb < j1; jb += 32) {
      const int64_t j = jb + lane;
      uint32_t len = 0;
      if (j < j1) len = ((ctrl[j >> 2] >> (2 * (j & 3))) & 3u) + 1u;
      int tot;
      const int off = warp_excl_scan((int)len, lane, &tot);
      if (j < j1) {
        const uint8_t* p = data + pos + off;
        uint32_t z = p[0];
        if (len > 1) z |= (uint32_t)p[1] << 8;
        if (len > 2) z |= (uint32_t)p[2] << 16;
        if (len > 3) z |= (uint32_t)p[3] << 24;
        out[j] = (T)(int32_t)((z >> 1) ^ (0u - (z & 1u)));
      }
      pos += tot;
    }
  }
}

// ---- symmetric CSR from its upper triangle --------------------------------
// An undirected CSR (reference coo_to_csr with make_undirected: no self
// loops, no duplicates, rows sorted) is determined by its upper triangle U
// (each row's entries > the row id, i.e. every edge once).  Row u of the full
// CSR is [lower part: w < u with u in U(w), ascending] ++ [U(u)], so with the
// full row offsets `row` and U's own offsets `urow`:
//   upper slot j of row u  -> col[j + row[u+1] - urow[u+1]]
//   lower entries          = U transposed: the pairs (v = U[j], u) sorted by
//                            v, stable (u ascending within v) -> sorted index
//                            i of a pair with key v goes to col[i + urow[v]]
//                            (row[v] = lower entries before v + urow[v]).
// The transpose is one stable radix sort of (v, u) pairs over log2(n) bits.

// rowid[urow[u]] = u for every non-empty upper row (then a max-scan fills the rest)
// (every index derived from the host image is range-checked: a malformed
// image leaves wrong columns, never an out-of-bounds access)
__global__ void k_upper_row_starts(const int64_t* __restrict__ urow, int64_t n, int64_t mu,
                                   int32_t* __restrict__ rowid) {
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n;
       u += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = urow[u];
    if (urow[u + 1] > b && b >= 0 && b < mu) rowid[b] = (int32_t)u;
  }
}

__global__ void k_place_upper(const int64_t* __restrict__ row, const int64_t* __restrict__ urow,
                              const int32_t* __restrict__ ucol, const int32_t* __restrict__ rowid,
                              int64_t mu, int64_t m, int32_t* __restrict__ col) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < mu;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int32_t u = rowid[j];
    const int64_t dst = j + row[u + 1] - urow[u + 1];
    if (dst >= 0 && dst < m) col[dst] = ucol[j];
  }
}

__global__ void k_place_lower(const int64_t* __restrict__ urow, const uint32_t* __restrict__ key,
                              const int32_t* __restrict__ val, int64_t n, int64_t mu, int64_t m,
                              int32_t* __restrict__ col) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < mu;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t v = key[i];
    if ((int64_t)v >= n) continue;
    const int64_t dst = i + urow[v];
    if (dst >= 0 && dst < m) col[dst] = val[i];
  }
}

struct MaxI32 {
  __device__ __forceinline__ int32_t operator()(int32_t a, int32_t b) const { return a > b ? a : b; }
};

}  // namespace gfx

using namespace gfx;

template <class T>
static int pack_size_t(gfx_ctx* ctx, const T* col_d, int64_t m, int64_t* boff_d,
                       int64_t* data_bytes) {
  const int64_t nb = (m + kPackBlock - 1) / kPackBlock;
  int64_t* bsize;
  GFX_CK(cudaMallocAsync(&bsize, (nb + 1) * 8, ctx->stream));
  GFX_CK(cudaMemsetAsync(bsize + nb, 0, 8, ctx->stream));
  GFX_LAUNCH(k_pack_sizes<T>, grid_for(nb * 32, 256, ctx->sm_count * 16), 256, 0, ctx->stream,
             col_d, m, bsize);
  size_t tb = 0;
  GFX_CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, bsize, boff_d, nb + 1, ctx->stream));
  void* tmp;
  GFX_CK(cudaMallocAsync(&tmp, tb + 16, ctx->stream));
  GFX_CK(cub::DeviceScan::ExclusiveSum(tmp, tb, bsize, boff_d, nb + 1, ctx->stream));
  count_launch();
  auto* pin = static_cast<int64_t*>(ctx->pinned);
  GFX_CK(cudaMemcpyAsync(pin, boff_d + nb, 8, cudaMemcpyDeviceToHost, ctx->stream));
  GFX_CK(cudaFreeAsync(tmp, ctx->stream));
  GFX_CK(cudaFreeAsync(bsize, ctx->stream));
  GFX_CK(cudaStreamSynchronize(ctx->stream));
  *data_bytes = pin[0];
  return GFX_OK;
}

template <class T>
static int unpack_t(gfx_ctx* ctx, const uint8_t* ctrl_d, const uint8_t* data_d,
                    const int64_t* boff_d, int64_t m, T* col_d) {
  const int64_t nb = (m + kPackBlock - 1) / kPackBlock;
  GFX_LAUNCH(k_unpack_deltas<T>, grid_for(nb * 32, 256, ctx->sm_count * 16), 256, 0, ctx->stream,
             ctrl_d, data_d, boff_d, m, col_d);
  // prefix sum of the differences restores the values (for int32 columns the
  // wrap-around is harmless: every partial sum is a real column id)
  size_t tb = 0;
  GFX_CK(cub::DeviceScan::InclusiveSum(nullptr, tb, col_d, col_d, m, ctx->stream));
  void* tmp;
  GFX_CK(cudaMallocAsync(&tmp, tb + 16, ctx->stream));
  GFX_CK(cub::DeviceScan::InclusiveSum(tmp, tb, col_d, col_d, m, ctx->stream));
  count_launch();
  GFX_CK(cudaFreeAsync(tmp, ctx->stream));
  return GFX_OK;
}

extern "C" {

int gfx_csr_pack_size(gfx_ctx* ctx, const void* vals_d, int elem_bytes, int64_t m, int64_t* boff_d,
                      int64_t* data_bytes) {
  GFX_NVTX("gfx_csr_pack_size");
  GFX_REQUIRE(ctx && data_bytes && (m == 0 || (vals_d && boff_d)), "gfx_csr_pack_size: null argument");
  GFX_REQUIRE(elem_bytes == 4 || elem_bytes == 8, "elem_bytes must be 4 (int32) or 8 (int64)");
  GFX_CK(cudaSetDevice(ctx->device));
  *data_bytes = 0;
  if (m == 0) return GFX_OK;
  return elem_bytes == 4
             ? pack_size_t(ctx, static_cast<const int32_t*>(vals_d), m, boff_d, data_bytes)
             : pack_size_t(ctx, static_cast<const int64_t*>(vals_d), m, boff_d, data_bytes);
}

int gfx_csr_pack(gfx_ctx* ctx, const void* vals_d, int elem_bytes, int64_t m,
                 const int64_t* boff_d, uint8_t* ctrl_d, uint8_t* data_d) {
  GFX_NVTX("gfx_csr_pack");
  GFX_REQUIRE(ctx && (m == 0 || (vals_d && boff_d && ctrl_d && data_d)), "gfx_csr_pack: null argument");
  GFX_REQUIRE(elem_bytes == 4 || elem_bytes == 8, "elem_bytes must be 4 (int32) or 8 (int64)");
  GFX_CK(cudaSetDevice(ctx->device));
  if (m == 0) return GFX_OK;
  const int64_t nb = (m + kPackBlock - 1) / kPackBlock;
  GFX_CK(cudaMemsetAsync(ctrl_d, 0, (m + 3) / 4, ctx->stream));
  if (elem_bytes == 4)
    GFX_LAUNCH(k_pack_write<int32_t>, grid_for(nb * 32, 256, ctx->sm_count * 16), 256, 0,
               ctx->stream, static_cast<const int32_t*>(vals_d), m, boff_d, ctrl_d, data_d);
  else
    GFX_LAUNCH(k_pack_write<int64_t>, grid_for(nb * 32, 256, ctx->sm_count * 16), 256, 0,
               ctx->stream, static_cast<const int64_t*>(vals_d), m, boff_d, ctrl_d, data_d);
  GFX_CK(cudaGetLastError());
  GFX_CK(cudaStreamSynchronize(ctx->stream));
  return GFX_OK;
}

int gfx_csr_unpack(gfx_ctx* ctx, const uint8_t* ctrl_d, const uint8_t* data_d,
                   const int64_t* boff_d, int64_t m, void* vals_d, int elem_bytes, int sync) {
  GFX_NVTX("gfx_csr_unpack");
  GFX_REQUIRE(ctx && (m == 0 || (ctrl_d && data_d && boff_d && vals_d)),
              "gfx_csr_unpack: null argument");
  GFX_REQUIRE(elem_bytes == 4 || elem_bytes == 8, "elem_bytes must be 4 (int32) or 8 (int64)");
  GFX_CK(cudaSetDevice(ctx->device));
  if (m == 0) return GFX_OK;
  if (elem_bytes == 4) GFX_TRY(unpack_t(ctx, ctrl_d, data_d, boff_d, m, static_cast<int32_t*>(vals_d)));
  else GFX_TRY(unpack_t(ctx, ctrl_d, data_d, boff_d, m, static_cast<int64_t*>(vals_d)));
  GFX_CK(cudaGetLastError());
  if (sync) GFX_CK(cudaStreamSynchronize(ctx->stream));
  return GFX_OK;
}

int gfx_graph_rebuild_upper(gfx_graph* g, const int64_t* urow_d, const int32_t* ucol_d,
                            int64_t mu) {
  GFX_NVTX("gfx_graph_rebuild_upper");
  GFX_REQUIRE(g && (mu == 0 || (urow_d && ucol_d)), "gfx_graph_rebuild_upper: null argument");
  GFX_REQUIRE(g->flags & GFX_GRAPH_UNDIRECTED, "gfx_graph_rebuild_upper: undirected graphs only");
  GFX_REQUIRE(2 * mu == g->m, "gfx_graph_rebuild_upper: the upper triangle must hold m/2 slots");
  gfx_ctx* ctx = g->ctx;
  GFX_CK(cudaSetDevice(ctx->device));
  if (mu == 0) return GFX_OK;
  const int64_t n = g->n;
  int32_t* rowid;
  GFX_TRY(scratch_t(g, "up_rowid", mu, &rowid));
  // row ids of the upper slots: row starts, then an inclusive max-scan
  GFX_CK(cudaMemsetAsync(rowid, 0, mu * 4, ctx->stream));
  GFX_LAUNCH(k_upper_row_starts, grid_for(n, 256, ctx->sm_count * 8), 256, 0, ctx->stream, urow_d,
             n, mu, rowid);
  size_t tb_scan = 0;
  GFX_CK(cub::DeviceScan::InclusiveScan(nullptr, tb_scan, rowid, rowid, MaxI32(), mu, ctx->stream));
  void* tmp;
  GFX_TRY(scratch(g, "up_cub", tb_scan + 16, &tmp));
  GFX_CK(cub::DeviceScan::InclusiveScan(tmp, tb_scan, rowid, rowid, MaxI32(), mu, ctx->stream));
  count_launch();
  // upper slots straight to their place; the lower parts by the transpose
  int32_t* val_out;
  uint32_t* key_out;
  GFX_TRY(scratch_t(g, "up_key", mu, &key_out));
  GFX_TRY(scratch_t(g, "up_val", mu, &val_out));
  int bits = 1;
  while (bits < 31 && (int64_t(1) << bits) < n) ++bits;
  const uint32_t* key_in = reinterpret_cast<const uint32_t*>(ucol_d);
  size_t tb_sort = 0;
  GFX_CK(cub::DeviceRadixSort::SortPairs(nullptr, tb_sort, key_in, key_out, rowid, val_out, mu, 0,
                                         bits, ctx->stream));
  GFX_TRY(scratch(g, "up_sorttmp", tb_sort + 16, &tmp));
  GFX_LAUNCH(k_place_upper, grid_for(mu, 256, ctx->sm_count * 16), 256, 0, ctx->stream, g->row,
             urow_d, ucol_d, rowid, mu, g->m, const_cast<int32_t*>(g->col));
  // the transpose: (v, u) pairs stably sorted by v
  GFX_CK(cub::DeviceRadixSort::SortPairs(tmp, tb_sort, key_in, key_out, rowid, val_out, mu, 0, bits,
                                         ctx->stream));
  count_launch();
  GFX_LAUNCH(k_place_lower, grid_for(mu, 256, ctx->sm_count * 16), 256, 0, ctx->stream, urow_d,
             key_out, val_out, n, mu, g->m, const_cast<int32_t*>(g->col));
  GFX_CK(cudaGetLastError());
  return GFX_OK;
}

}  // extern "C"
