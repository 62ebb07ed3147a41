// knng_build.cu -- K7 exact initial graph (graph_init; AL1 "brute force"):
// row v = the first k of all u != v in edge order.
//
// Tiled SIMT kernel: a block owns 64 rows (8 per warp, each row's top-k in warp registers),
// streams the whole store through shared memory in tiles of 64 vectors and evaluates every
// (row, column) pair with the single-thread canonical distance (so the keys are bit-identical
// to the search path's warp evaluator).
#include <stdlib.h>

#include <algorithm>

#include "knng_common.cuh"
#include "knng_internal.h"

namespace knng {

// Rows [row0, row0+nrows) against columns [col0, col0+ncols) (u != v), optionally seeded with a
// sorted candidate row per output row (seed[r*k ..], -1 padded): out[r*k ..] = top-k.
// graph_init: rows = cols = the whole store; intra-batch all-pairs (K3, A5): rows = the batch (or a
// rank's shard of it), cols = the batch, seed = the search results C_i.
template <int M>
__global__ void __launch_bounds__(256) k_tile_topk(const uint8_t *__restrict__ vec, size_t stride, int nchunks,
                                                   int64_t row0, int64_t nrows, int64_t col0, int64_t ncols, int k,
                                                   const int32_t *seed_ids, const uint32_t *seed_keys,
                                                   int32_t *out_ids, uint32_t *out_keys) {
  extern __shared__ uint4 sm[];
  const int spad = nchunks + 1;                 // 16 B of padding per row: conflict-free LDS.128
  uint4 *srow = sm;
  uint4 *scol = sm + 64 * spad;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t r0 = (int64_t)blockIdx.x * 64;  // local row of this block
  // column split y of gridDim.y (partial top-k per split; merged by k_merge_partials)
  {
    const int64_t per = ((ncols + gridDim.y - 1) / gridDim.y + 63) / 64 * 64;
    const int64_t c_lo = (int64_t)blockIdx.y * per;
    const int64_t c_hi = c_lo + per < ncols ? c_lo + per : ncols;
    col0 += c_lo;
    ncols = c_hi > c_lo ? c_hi - c_lo : 0;
    out_ids += (size_t)blockIdx.y * nrows * k;
    out_keys += (size_t)blockIdx.y * nrows * k;
  }
  for (int i = threadIdx.x; i < 64 * nchunks; i += 256) {
    const int r = i / nchunks, c = i % nchunks;
    srow[r * spad + c] = (r0 + r < nrows) ? ldg16(vec + (size_t)(row0 + r0 + r) * stride + (size_t)c * 16)
                                          : make_uint4(0, 0, 0, 0);
  }
  WarpTopK<M> top[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    top[t].init(k);
    const int64_t rl = r0 + warp * 8 + t;
    if (seed_ids && rl < nrows) {
      const int32_t sid = lane < k ? seed_ids[(size_t)rl * k + lane] : -1;
      const uint32_t sk = lane < k ? seed_keys[(size_t)rl * k + lane] : 0u;
      top[t].insert(sid >= 0, sk, sid);
    }
  }
  for (int64_t c0 = 0; c0 < ncols; c0 += 64) {
    __syncthreads();
    for (int i = threadIdx.x; i < 64 * nchunks; i += 256) {
      const int r = i / nchunks, c = i % nchunks;
      scol[r * spad + c] = (c0 + r < ncols) ? ldg16(vec + (size_t)(col0 + c0 + r) * stride + (size_t)c * 16)
                                            : make_uint4(0, 0, 0, 0);
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int rl = warp * 8 + t;
      const int64_t row = row0 + r0 + rl;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int cl = lane + 32 * h;
        const int64_t col = col0 + c0 + cl;
        const bool valid = r0 + rl < nrows && c0 + cl < ncols && col != row;
        const uint32_t key = valid ? thread_dist<M>(srow + rl * spad, scol + cl * spad, nchunks) : 0u;
        top[t].insert(valid, key, (int32_t)col);
      }
    }
  }
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    const int64_t rl = r0 + warp * 8 + t;
    if (rl < nrows && lane < k) {
      out_ids[(size_t)rl * k + lane] = lane < top[t].cnt ? top[t].id : -1;
      out_keys[(size_t)rl * k + lane] = lane < top[t].cnt ? top[t].key : 0u;
    }
  }
}

// top-k over the seed row and the ny partial rows [ny][nrows][k] of the column splits
template <int M>
__global__ void k_merge_partials(int64_t nrows, int k, int ny, const int32_t *seed_ids, const uint32_t *seed_keys,
                                 const int32_t *pi, const uint32_t *pk, int32_t *out_ids, uint32_t *out_keys) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= nrows) return;
  WarpTopK<M> top;
  top.init(k);
  if (seed_ids) {
    const int32_t sid = lane < k ? seed_ids[(size_t)r * k + lane] : -1;
    top.insert(sid >= 0, lane < k ? seed_keys[(size_t)r * k + lane] : 0u, sid);
  }
  for (int y = 0; y < ny; ++y) {
    const size_t o = ((size_t)y * nrows + r) * k;
    const int32_t id = lane < k ? pi[o + lane] : -1;
    top.insert(id >= 0, lane < k ? pk[o + lane] : 0u, id);
  }
  if (lane < k) {
    out_ids[(size_t)r * k + lane] = lane < top.cnt ? top.id : -1;
    out_keys[(size_t)r * k + lane] = lane < top.cnt ? top.key : 0u;
  }
}

cudaError_t launch_tile_topk(const VecGeom &g, const uint8_t *vec, int64_t row0, int64_t nrows, int64_t col0,
                             int64_t ncols, int k, const int32_t *seed_ids, const uint32_t *seed_keys, int32_t *out_ids,
                             uint32_t *out_keys, DenseScratch *ws, cudaStream_t s) {
  if (nrows <= 0) return cudaSuccess;
  // u8 rows: the tcgen05 kind::i8 form (knng_tc.cu); two column halves per split, merged below
  const char *tce = getenv("KNNG_TC");
  const bool tc_u8 = g.metric == M_U8 && g.nchunks <= 16 && k <= 32;
  const bool tc_f32 = g.metric == M_F32 && g.nchunks <= 24 && k <= 32;   // operands fit smem up to d = 96
  if ((tc_u8 || tc_f32) && !(tce && atoi(tce) == 0)) {
    const int64_t bx = (nrows + 127) / 128, tn = tc_u8 ? 256 : 64;
    int64_t ny = bx >= 148 ? 1 : std::min<int64_t>((148 + bx - 1) / bx, std::max<int64_t>(1, (ncols + tn - 1) / tn));
    if (cudaError_t e = ws->part.ensure((size_t)2 * ny * nrows * k * 8)) return e;
    int32_t *pi = (int32_t *)ws->part.p;
    uint32_t *pk = (uint32_t *)((char *)ws->part.p + (size_t)2 * ny * nrows * k * 4);
    cudaError_t e =
        tc_u8 ? launch_tc_topk_u8(g, vec, row0, nrows, col0, ncols, k, seed_ids, seed_keys, ny, pi, pk, &ws->norm, s)
              : launch_tc_topk_f32(g, vec, row0, nrows, col0, ncols, k, seed_ids, seed_keys, ny, pi, pk, &ws->norm, s);
    if (e != cudaSuccess) return e;
    if (tc_u8)
      k_merge_partials<M_U8><<<(unsigned)((nrows + 3) / 4), 128, 0, s>>>(nrows, k, (int)(2 * ny), seed_ids, seed_keys,
                                                                          pi, pk, out_ids, out_keys);
    else
      k_merge_partials<M_F32><<<(unsigned)((nrows + 3) / 4), 128, 0, s>>>(nrows, k, (int)(2 * ny), seed_ids,
                                                                           seed_keys, pi, pk, out_ids, out_keys);
    return cudaGetLastError();
  }
  const size_t smem = (size_t)128 * (g.nchunks + 1) * 16;
  if (smem > 220 * 1024) return cudaErrorInvalidValue;
  const int64_t bx = (nrows + 63) / 64;
  // split the columns when the row blocks alone cannot fill the GPU (intra-batch all-pairs)
  int64_t ny = 1;
  if (bx < 2 * 148) ny = std::min<int64_t>((2 * 148 + bx - 1) / bx, std::max<int64_t>(1, ncols / 64));
  if (seed_ids && ny == 1) ny = 2;   // seeds are merged by k_merge_partials
  int32_t *pi = out_ids;
  uint32_t *pk = out_keys;
  if (ny > 1) {
    if (cudaError_t e = ws->part.ensure((size_t)ny * nrows * k * 8)) return e;
    pi = (int32_t *)ws->part.p;
    pk = (uint32_t *)((char *)ws->part.p + (size_t)ny * nrows * k * 4);
  }
  const dim3 grid((unsigned)bx, (unsigned)ny);
  cudaError_t e;
  if (g.metric == M_U8) {
    e = cudaFuncSetAttribute(k_tile_topk<M_U8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_tile_topk<M_U8><<<grid, 256, smem, s>>>(vec, g.stride, g.nchunks, row0, nrows, col0, ncols, k, nullptr, nullptr,
                                              pi, pk);
  } else {
    e = cudaFuncSetAttribute(k_tile_topk<M_F32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_tile_topk<M_F32><<<grid, 256, smem, s>>>(vec, g.stride, g.nchunks, row0, nrows, col0, ncols, k, nullptr,
                                               nullptr, pi, pk);
  }
  if (ny > 1) {
    const unsigned mb = (unsigned)((nrows + 3) / 4);
    if (g.metric == M_U8)
      k_merge_partials<M_U8><<<mb, 128, 0, s>>>(nrows, k, (int)ny, seed_ids, seed_keys, pi, pk, out_ids, out_keys);
    else
      k_merge_partials<M_F32><<<mb, 128, 0, s>>>(nrows, k, (int)ny, seed_ids, seed_keys, pi, pk, out_ids, out_keys);
  }
  return cudaGetLastError();
}

// Jaccard sets and strings: warp per row, lanes over all columns (single-thread pair keys: sorted-list
// intersection / str_key with the row as owner).
template <int M>
__global__ void __launch_bounds__(128) k_exact_build_csr(StoreView st, int64_t n, int k, int32_t *ids, uint32_t *keys) {
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
  if (row >= n) return;
  WarpTopK<M> top;
  top.init(k);
  if constexpr (str_metric(M)) {   // strings: the row's string as the warp's query (2-gram / character tables)
    __shared__ uint32_t qscr[4 * QSCR];
    __shared__ __align__(16) uint8_t jwp[M == M_JW ? 4 * 32 * JW_PTR : 16];
    const int wib = threadIdx.x >> 5;
    StrQuery<M> Q;
    if constexpr (M == M_JW) Q.ptr = jwp + (wib * 32 + lane) * JW_PTR;
    Q.load(st, row, qscr + wib * QSCR);
    for (int64_t c0 = 0; c0 < n; c0 += 32) {
      const int64_t col = c0 + lane;
      const bool valid = col < n && col != row;
      const uint32_t key = valid ? Q.key(st, (int32_t)col) : 0u;
      top.insert(valid, key, (int32_t)col);
    }
  } else {
    for (int64_t c0 = 0; c0 < n; c0 += 32) {
      const int64_t col = c0 + lane;
      const bool valid = col < n && col != row;
      const uint32_t key = valid ? pair_key<M>(st, row, col) : 0u;
      top.insert(valid, key, (int32_t)col);
    }
  }
  if (lane < k) {
    ids[(size_t)row * k + lane] = lane < top.cnt ? top.id : -1;
    keys[(size_t)row * k + lane] = lane < top.cnt ? top.key : 0u;
  }
}

cudaError_t launch_exact_build(const VecGeom &g, const StoreView &st, int64_t n, int k, int32_t *ids, uint32_t *keys,
                               DenseScratch *ws, cudaStream_t s) {
  if (csr_metric(g.metric)) {
    const unsigned nb = (unsigned)((n + 3) / 4);
    if (g.metric == M_JAC) k_exact_build_csr<M_JAC><<<nb, 128, 0, s>>>(st, n, k, ids, keys);
    else if (g.metric == M_JW) k_exact_build_csr<M_JW><<<nb, 128, 0, s>>>(st, n, k, ids, keys);
    else k_exact_build_csr<M_COS><<<nb, 128, 0, s>>>(st, n, k, ids, keys);
    return cudaGetLastError();
  }
  return launch_tile_topk(g, st.vec, 0, n, 0, n, k, nullptr, nullptr, ids, keys, ws, s);
}

}  // namespace knng
