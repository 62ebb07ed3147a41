// knng_build.cu -- K7 exact initial graph (graph_init; AL1 "brute force"):
// row v = the first k of all u != v in edge order.
//
// Tiled SIMT kernel: a block owns 64 rows (8 per warp, each row's top-k in warp registers),
// streams the whole store through shared memory in tiles of 64 vectors and evaluates every
// (row, column) pair with the single-thread canonical distance (so the keys are bit-identical
// to the search path's warp evaluator).
#include "knng_common.cuh"
#include "knng_internal.h"

namespace knng {

template <int M>
__global__ void __launch_bounds__(256) k_exact_build(const uint8_t *__restrict__ vec, size_t stride, int nchunks,
                                                     int64_t n, int k, int32_t *ids, uint32_t *keys) {
  extern __shared__ uint4 sm[];
  const int spad = nchunks + 1;                 // 16 B of padding per row: conflict-free LDS.128
  uint4 *srow = sm;
  uint4 *scol = sm + 64 * spad;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t r0 = (int64_t)blockIdx.x * 64;
  for (int i = threadIdx.x; i < 64 * nchunks; i += 256) {
    const int r = i / nchunks, c = i % nchunks;
    srow[r * spad + c] = (r0 + r < n) ? ldg16(vec + (size_t)(r0 + r) * stride + (size_t)c * 16) : make_uint4(0, 0, 0, 0);
  }
  WarpTopK<M> top[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) top[t].init(k);
  for (int64_t c0 = 0; c0 < n; c0 += 64) {
    __syncthreads();
    for (int i = threadIdx.x; i < 64 * nchunks; i += 256) {
      const int r = i / nchunks, c = i % nchunks;
      scol[r * spad + c] = (c0 + r < n) ? ldg16(vec + (size_t)(c0 + r) * stride + (size_t)c * 16) : make_uint4(0, 0, 0, 0);
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int rl = warp * 8 + t;
      const int64_t row = r0 + rl;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int cl = lane + 32 * h;
        const int64_t col = c0 + cl;
        const bool valid = row < n && col < n && col != row;
        const uint32_t key = valid ? thread_dist<M>(srow + rl * spad, scol + cl * spad, nchunks) : 0u;
        top[t].insert(valid, key, (int32_t)col);
      }
    }
  }
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    const int64_t row = r0 + warp * 8 + t;
    if (row < n && lane < k) {
      ids[(size_t)row * k + lane] = lane < top[t].cnt ? top[t].id : -1;
      keys[(size_t)row * k + lane] = lane < top[t].cnt ? top[t].key : 0u;
    }
  }
}

// Jaccard sets: warp per row, lanes over all columns (single-thread sorted-list intersection).
__global__ void __launch_bounds__(128) k_exact_build_sets(StoreView st, int64_t n, int k, int32_t *ids, uint32_t *keys) {
  const int lane = threadIdx.x & 31;
  const int64_t row = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
  if (row >= n) return;
  WarpTopK<M_JAC> top;
  top.init(k);
  for (int64_t c0 = 0; c0 < n; c0 += 32) {
    const int64_t col = c0 + lane;
    const bool valid = col < n && col != row;
    const uint32_t key = valid ? pair_key<M_JAC>(st, row, col) : 0u;
    top.insert(valid, key, (int32_t)col);
  }
  if (lane < k) {
    ids[(size_t)row * k + lane] = lane < top.cnt ? top.id : -1;
    keys[(size_t)row * k + lane] = lane < top.cnt ? top.key : 0u;
  }
}

cudaError_t launch_exact_build(const VecGeom &g, const StoreView &st, int64_t n, int k, int32_t *ids, uint32_t *keys,
                               cudaStream_t s) {
  if (g.metric == M_JAC) {
    k_exact_build_sets<<<(unsigned)((n + 3) / 4), 128, 0, s>>>(st, n, k, ids, keys);
    return cudaGetLastError();
  }
  const uint8_t *vec = st.vec;
  const size_t smem = (size_t)128 * (g.nchunks + 1) * 16;
  if (smem > 220 * 1024) return cudaErrorInvalidValue;
  const unsigned blocks = (unsigned)((n + 63) / 64);
  cudaError_t e;
  if (g.metric == M_U8) {
    e = cudaFuncSetAttribute(k_exact_build<M_U8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_exact_build<M_U8><<<blocks, 256, smem, s>>>(vec, g.stride, g.nchunks, n, k, ids, keys);
  } else {
    e = cudaFuncSetAttribute(k_exact_build<M_F32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_exact_build<M_F32><<<blocks, 256, smem, s>>>(vec, g.stride, g.nchunks, n, k, ids, keys);
  }
  return cudaGetLastError();
}

}  // namespace knng
