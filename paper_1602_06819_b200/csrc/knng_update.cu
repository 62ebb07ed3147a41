// knng_update.cu -- the batch update of graph_insert_batch:
//   K3 intra-batch all-pairs + new rows     (new row = top-k(C_i u peers), Q15)
//   K4 update ball + proposals              (Alg. 2, over the snapshot, Q12-Q14)
//   K5 proposal bucketing + per-node merge  (row_v = top-k(row_v u proposals); Q17)
//   K6 placement at the nearest medoid      (Alg. 5)
#include "knng_common.cuh"
#include "knng_internal.h"
#include "knng_update_one.cuh"

namespace knng {

// ---------------------------------------------------------------------------
// K3: warp per new point i; lanes take peers j = lane + 32t (thread-level canonical distance).
// ---------------------------------------------------------------------------
template <int M>
__global__ void __launch_bounds__(128) k_allpairs(StoreView st, int64_t n_t, int64_t B, int64_t q_lo, int64_t nq,
                                                  int k, const int32_t *Ci, const uint32_t *Ck, int32_t *oi,
                                                  uint32_t *ok) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= nq) return;
  const int64_t i = q_lo + r;
  WarpTopK<M> top;
  top.init(k);
  {
    const int32_t cid = lane < k ? Ci[r * k + lane] : -1;
    const uint32_t ck = lane < k ? Ck[r * k + lane] : 0u;
    top.insert(cid >= 0, ck, cid);
  }
  if constexpr (str_metric(M)) {   // strings: the row's string as the warp's query (2-gram / character tables)
    __shared__ uint32_t qscr[4 * QSCR];
    __shared__ __align__(16) uint8_t jwp[M == M_JW ? 4 * 32 * JW_PTR : 16];
    const int wib = threadIdx.x >> 5;
    StrQuery<M> Q;
    if constexpr (M == M_JW) Q.ptr = jwp + (wib * 32 + lane) * JW_PTR;
    Q.load(st, n_t + i, qscr + wib * QSCR);
    for (int64_t j0 = 0; j0 < B; j0 += 32) {
      const int64_t j = j0 + lane;
      const bool valid = j < B && j != i;
      const uint32_t key = valid ? Q.key(st, (int32_t)(n_t + j)) : 0u;
      top.insert(valid, key, (int32_t)(n_t + j));
    }
  } else {
    for (int64_t j0 = 0; j0 < B; j0 += 32) {
      const int64_t j = j0 + lane;
      const bool valid = j < B && j != i;
      uint32_t key = 0;
      if (valid) key = pair_key<M>(st, n_t + i, n_t + j);
      top.insert(valid, key, (int32_t)(n_t + j));
    }
  }
  if (lane < k) {
    oi[(size_t)r * k + lane] = lane < top.cnt ? top.id : -1;
    ok[(size_t)r * k + lane] = lane < top.cnt ? top.key : 0u;
  }
}

cudaError_t launch_tile_topk(const VecGeom &g, const uint8_t *vec, int64_t row0, int64_t nrows, int64_t col0,
                             int64_t ncols, int k, const int32_t *seed_ids, const uint32_t *seed_keys, int32_t *out_ids,
                             uint32_t *out_keys, DenseScratch *ws, cudaStream_t s);

// A5: new rows of batch queries [q_lo, q_lo+nq): top-k(C_i u {(D(x_i, x_j), n_t+j) : j != i}).
// Ci/Ck and the outputs are indexed by the local row (query - q_lo).
cudaError_t launch_allpairs(const VecGeom &g, const StoreView &st, int64_t n_t, int64_t B, int64_t q_lo, int64_t nq,
                            int k, const int32_t *Ci, const uint32_t *Ck, int32_t *oi, uint32_t *ok, DenseScratch *ws,
                            cudaStream_t s) {
  if (nq <= 0) return cudaSuccess;
  if (!csr_metric(g.metric))   // vectors: the smem-tiled kernel of the exact build, seeded with C_i
    return launch_tile_topk(g, st.vec, n_t + q_lo, nq, n_t, B, k, Ci, Ck, oi, ok, ws, s);
  const unsigned nb = (unsigned)((nq + 3) / 4);
  if (g.metric == M_JAC) k_allpairs<M_JAC><<<nb, 128, 0, s>>>(st, n_t, B, q_lo, nq, k, Ci, Ck, oi, ok);
  else if (g.metric == M_JW) k_allpairs<M_JW><<<nb, 128, 0, s>>>(st, n_t, B, q_lo, nq, k, Ci, Ck, oi, ok);
  else k_allpairs<M_COS><<<nb, 128, 0, s>>>(st, n_t, B, q_lo, nq, k, Ci, Ck, oi, ok);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// K4: update ball.  Warp per new point; BFS levels with a per-slot hash set (dedup, Q12);
// each level's nodes are evaluated 32 at a time with the warp evaluator; a node v proposes the
// new point when (D, id_x) precedes row_v[k-1] (Q14).
// ---------------------------------------------------------------------------

template <int M, int L, int CPL>
__global__ void __launch_bounds__(128) k_ball(BallArgs a) {
  __shared__ int s_n[4];
  __shared__ uint32_t qscr[csr_metric(M) ? 4 * QSCR : 1];
  __shared__ __align__(16) uint8_t jwp[M == M_JW ? 4 * 32 * JW_PTR : 16];   // JW character pointers per lane
  extern __shared__ int32_t bsm[];   // small balls: [4][hcap] hash + [4][ballmax] list in shared memory
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t gw = (int64_t)blockIdx.x * 4 + wib, nw = (int64_t)gridDim.x * 4;
  int32_t *hash = a.smem_ball ? bsm + wib * a.hcap : a.hash + gw * a.hcap;
  int32_t *list = a.smem_ball ? bsm + 4 * a.hcap + wib * a.ballmax : a.list + gw * a.ballmax;
  const int k = a.k;
  unsigned long long s_ball = 0, s_prop = 0;
  for (int64_t bl = gw; bl < a.nqb; bl += nw) {
    const int64_t b = a.q0 + bl;             // query of the batch; proposals are stored at slot bl
    for (int i = lane; i < a.hcap; i += 32) hash[i] = -1;
    if (lane == 0) s_n[wib] = 0;
    __syncwarp();
    typename QuerySel<M, L, CPL>::T Q;
    if constexpr (M == M_JW) Q.ptr = jwp + (wib * 32 + lane) * JW_PTR;
    Q.load(a.st, a.n_t + b, csr_metric(M) ? qscr + wib * QSCR : nullptr);
    const int32_t idx = (int32_t)(a.n_t + b);
    // L1 = the search result C(x)
    {
      const int32_t v = lane < k ? a.C[b * k + lane] : -1;
      const bool ins = v >= 0 && hash_insert(hash, a.hcap, v);
      const unsigned m = __ballot_sync(FULL, ins);
      if (ins) list[__popc(m & lanemask_lt())] = v;
      if (lane == 0) s_n[wib] = __popc(m);
      __syncwarp();
    }
    int lo = 0, hi = s_n[wib];
    int np = 0;
    int2 *props = a.props + (size_t)bl * a.ballmax;
    for (int d = 1; d <= a.depth; ++d) {
      for (int base = lo; base < hi; base += 32) {
        const int t = base + lane;
        const int32_t v = t < hi ? list[t] : -1;
        if (d < a.depth && v >= 0) {
          for (int e = 0; e < k; ++e) {
            const int32_t u = a.ids[(size_t)v * k + e];
            if (u >= 0 && hash_insert(hash, a.hcap, u)) {
              const int pos = atomicAdd(&s_n[wib], 1);
              if (pos < a.ballmax) list[pos] = u;
            }
          }
        }
        const int cnt = hi - base < 32 ? hi - base : 32;
        uint32_t key;
        if constexpr (str_metric(M)) key = Q.rkey(a.st, v);   // strings: v's own key of the new point (v's row)
        else key = Q.eval(a.st, v, cnt);
        bool prop = false;
        if (v >= 0) {
          const uint32_t kk = a.keys[(size_t)v * k + k - 1];
          const int32_t ik = a.ids[(size_t)v * k + k - 1];
          prop = precedes<M>(key, idx, kk, ik);
        }
        const unsigned pm = __ballot_sync(FULL, prop);
        if (prop) props[np + __popc(pm & lanemask_lt())] = make_int2(v, (int)key);
        np += __popc(pm);
      }
      __syncwarp();
      lo = hi;
      hi = s_n[wib] < a.ballmax ? s_n[wib] : a.ballmax;
      __syncwarp();
    }
    s_ball += (unsigned long long)lo;
    s_prop += np;
    if (lane == 0) a.prop_cnt[bl] = np;
    __syncwarp();
  }
  if (lane == 0) {
    atomicAdd(a.stats + 4, s_ball);
    atomicAdd(a.stats + 5, s_prop);
  }
}

// ---------------------------------------------------------------------------
// B = 1 (the paper's sequential algorithm, Alg. 1 + Alg. 2): the whole update of one insert in one warp.
// The new row is the search result C (no batch peers); the ball is collected over the snapshot rows
// first (levels with dedup, Q12-Q13), its nodes are evaluated, and then every proposal is applied in
// place -- each ball node's row has exactly one writer (the ball is a set), so no bucketing is needed.
// Shared memory: hash [hcap] + list [ballmax] + proposals [ballmax] (node, key).
// ---------------------------------------------------------------------------
template <int M, int L, int CPL>
__global__ void __launch_bounds__(32) k_update_one(BallArgs a, const uint32_t *Ckeys) {
  extern __shared__ int32_t usm[];
  __shared__ uint32_t qscr[csr_metric(M) ? QSCR : 1];
  __shared__ __align__(16) uint8_t jwp[M == M_JW ? 32 * JW_PTR : 16];
  __shared__ int s_n;
  update_one_warp<M, L, CPL>(a, a.C, Ckeys, usm, &s_n, csr_metric(M) ? qscr : nullptr, nullptr, nullptr, nullptr,
                             M == M_JW ? jwp : nullptr);
}

template <int M, int L, int CPL>
static cudaError_t run_update_one(const BallArgs &a, const uint32_t *Ckeys, cudaStream_t s) {
  const size_t smem = update_one_smem(a.hcap, a.ballmax);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_update_one<M, L, CPL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  k_update_one<M, L, CPL><<<1, 32, smem, s>>>(a, Ckeys);
  return cudaGetLastError();
}

template <int M, int L, int CPL>
static cudaError_t run_ball(const BallArgs &a, int64_t nslots, cudaStream_t s) {
  if (a.nqb == 0) return cudaSuccess;
  const int64_t blocks = nslots / 4;
  const size_t smem = a.smem_ball ? (size_t)4 * (a.hcap + a.ballmax) * 4 : 0;
  k_ball<M, L, CPL><<<(unsigned)blocks, 128, smem, s>>>(a);
  return cudaGetLastError();
}

#define KNNG_SHAPES(X, M) \
  X(M, 1, 1) X(M, 2, 1) X(M, 4, 1) X(M, 8, 1) X(M, 16, 1) X(M, 32, 1) X(M, 32, 2) X(M, 32, 4)
// fp32 rows of <= 32 chunks: 4 chunks per lane at most, partials in-lane (see VecQuery::reduce)
#define KNNG_SHAPES_F32(X) \
  X(M_F32, 1, 1) X(M_F32, 1, 2) X(M_F32, 1, 3) X(M_F32, 1, 4) X(M_F32, 2, 3) X(M_F32, 2, 4) X(M_F32, 4, 3) \
  X(M_F32, 4, 4) X(M_F32, 8, 3) X(M_F32, 8, 4) X(M_F32, 32, 2) X(M_F32, 32, 4)

cudaError_t launch_update_one(const VecGeom &g, const BallArgs &a, const uint32_t *Ckeys, cudaStream_t s) {
#define X(MM, LL, CC) \
  if (g.metric == MM && g.L == LL && g.CPL == CC) return run_update_one<MM, LL, CC>(a, Ckeys, s);
  KNNG_SHAPES(X, M_U8)
  KNNG_SHAPES_F32(X)
  X(M_JAC, 8, 1)
  X(M_JW, 8, 1)
  X(M_COS, 8, 1)
#undef X
  return cudaErrorInvalidValue;
}

cudaError_t launch_ball(const VecGeom &g, const BallArgs &a, int64_t nslots, cudaStream_t s) {
#define X(MM, LL, CC) \
  if (g.metric == MM && g.L == LL && g.CPL == CC) return run_ball<MM, LL, CC>(a, nslots, s);
  KNNG_SHAPES(X, M_U8)
  KNNG_SHAPES_F32(X)
  X(M_JAC, 8, 1)
  X(M_JW, 8, 1)
  X(M_COS, 8, 1)
#undef X
  return cudaErrorInvalidValue;
}

// ---------------------------------------------------------------------------
// K5: bucket the proposals by node (count, exclusive scan, scatter), then one thread per
// touched node merges its row with its proposals: row_v = top-k(row_v u proposals).  The merge
// owns each row (no atomics on rows); a top-k under a strict total order does not depend on
// the order the proposals arrive in, so the result equals the fixed (qid, key, node) order.
// ---------------------------------------------------------------------------
__global__ void k_prop_count(const int2 *props, const int32_t *prop_cnt, int ballmax, int64_t B, int32_t *ncnt) {
  const int64_t b = blockIdx.x;
  if (b >= B) return;
  const int n = prop_cnt[b];
  for (int j = threadIdx.x; j < n; j += blockDim.x) atomicAdd(ncnt + props[b * ballmax + j].x, 1);
}

__global__ void k_scan_block(const int32_t *in, int32_t *out, int32_t *blocksum, int64_t n) {
  __shared__ int32_t ws[32];
  const int64_t i = (int64_t)blockIdx.x * 1024 + threadIdx.x;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int32_t x = i < n ? in[i] : 0;
  int32_t v = x;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t y = __shfl_up_sync(FULL, v, o);
    if (lane >= o) v += y;
  }
  if (lane == 31) ws[w] = v;
  __syncthreads();
  if (w == 0) {
    int32_t s = ws[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(FULL, s, o);
      if (lane >= o) s += y;
    }
    ws[lane] = s;
  }
  __syncthreads();
  const int32_t pre = (w > 0 ? ws[w - 1] : 0) + v - x;   // exclusive
  if (i < n) out[i] = pre;
  if (threadIdx.x == 1023) blocksum[blockIdx.x] = ws[31];
}

__global__ void k_scan_sums(int32_t *blocksum, int64_t nb) {
  // single block: exclusive scan of nb block sums, 1024 at a time
  __shared__ int32_t ws[32];
  __shared__ int32_t carry;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < nb; base += 1024) {
    const int64_t i = base + threadIdx.x;
    const int32_t x = i < nb ? blocksum[i] : 0;
    int32_t v = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t y = __shfl_up_sync(FULL, v, o);
      if (lane >= o) v += y;
    }
    if (lane == 31) ws[w] = v;
    __syncthreads();
    if (w == 0) {
      int32_t s = ws[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(FULL, s, o);
        if (lane >= o) s += y;
      }
      ws[lane] = s;
    }
    __syncthreads();
    const int32_t c0 = carry;
    if (i < nb) blocksum[i] = c0 + (w > 0 ? ws[w - 1] : 0) + v - x;
    __syncthreads();
    if (threadIdx.x == 0) carry = c0 + ws[31];
    __syncthreads();
  }
}

__global__ void k_scan_add(int32_t *out, const int32_t *blocksum, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * 1024 + threadIdx.x;
  if (i < n) out[i] += blocksum[blockIdx.x];
}

cudaError_t exclusive_scan_i32(const int32_t *in, int32_t *out, int32_t *tmp, int64_t n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const int64_t nb = (n + 1023) / 1024;
  k_scan_block<<<(unsigned)nb, 1024, 0, s>>>(in, out, tmp, n);
  k_scan_sums<<<1, 1024, 0, s>>>(tmp, nb);
  k_scan_add<<<(unsigned)nb, 1024, 0, s>>>(out, tmp, n);
  return cudaGetLastError();
}

__global__ void k_prop_scatter(const int2 *props, const int32_t *prop_cnt, int ballmax, int64_t B, int64_t n_t,
                               const int32_t *noff, int32_t *nfill, int2 *sorted) {
  const int64_t b = blockIdx.x;
  if (b >= B) return;
  const int n = prop_cnt[b];
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    const int2 pr = props[b * ballmax + j];
    const int pos = noff[pr.x] + atomicAdd(nfill + pr.x, 1);
    sorted[pos] = make_int2(pr.y, (int)(n_t + b));   // (key, new id)
  }
}

template <int M>
__global__ void k_node_merge(int32_t *ids, uint32_t *keys, int k, int64_t n_t, int32_t *ncnt, int32_t *nfill,
                             const int32_t *noff, const int2 *sorted, int32_t *prow, int64_t member_cap,
                             const uint8_t *part_of, const int32_t *local_idx) {
  const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= n_t) return;
  const int c = ncnt[v];
  if (c == 0) return;
  int32_t ri[32];
  uint32_t rk[32];
  for (int e = 0; e < k; ++e) { ri[e] = ids[v * k + e]; rk[e] = keys[v * k + e]; }
  const int o = noff[v];
  for (int j = 0; j < c; ++j) {
    const int2 pr = sorted[o + j];
    const uint32_t key = (uint32_t)pr.x;
    const int32_t id = pr.y;
    if (!precedes<M>(key, id, rk[k - 1], ri[k - 1])) continue;
    int pos = k - 1;
    while (pos > 0 && precedes<M>(key, id, rk[pos - 1], ri[pos - 1])) {
      rk[pos] = rk[pos - 1];
      ri[pos] = ri[pos - 1];
      --pos;
    }
    rk[pos] = key;
    ri[pos] = id;
  }
  for (int e = 0; e < k; ++e) { ids[v * k + e] = ri[e]; keys[v * k + e] = rk[e]; }
  if (prow) {   // partitioned: keep the row's partition-local copy current (new ids are placed already)
    const uint8_t pv = part_of[v];
    int32_t *lr = prow + ((size_t)pv * member_cap + local_idx[v]) * k;
    for (int e = 0; e < k; ++e) {
      const int32_t u = ri[e];
      lr[e] = (u >= 0 && part_of[u] == pv) ? local_idx[u] : -1;
    }
  }
  ncnt[v] = 0;
  nfill[v] = 0;
}

cudaError_t launch_merge_props(int metric, int32_t *ids, uint32_t *keys, int k, int64_t n_t, int64_t B,
                               const int2 *props, const int32_t *prop_cnt, int ballmax, int32_t *ncnt,
                               int32_t *nfill, int32_t *noff, int32_t *scan_tmp, int2 *sorted, cudaStream_t s,
                               int *n_launch, int32_t *prow, int64_t member_cap, const uint8_t *part_of,
                               const int32_t *local_idx) {
  if (B == 0) return cudaSuccess;
  k_prop_count<<<(unsigned)B, 128, 0, s>>>(props, prop_cnt, ballmax, B, ncnt);
  const int64_t nb = (n_t + 1023) / 1024;
  k_scan_block<<<(unsigned)nb, 1024, 0, s>>>(ncnt, noff, scan_tmp, n_t);
  k_scan_sums<<<1, 1024, 0, s>>>(scan_tmp, nb);
  k_scan_add<<<(unsigned)nb, 1024, 0, s>>>(noff, scan_tmp, n_t);
  k_prop_scatter<<<(unsigned)B, 128, 0, s>>>(props, prop_cnt, ballmax, B, n_t, noff, nfill, sorted);
  const unsigned mb = (unsigned)((n_t + 255) / 256);
  if (metric == M_U8) k_node_merge<M_U8><<<mb, 256, 0, s>>>(ids, keys, k, n_t, ncnt, nfill, noff, sorted, prow, member_cap, part_of,
                                                          local_idx);
  else if (metric == M_F32) k_node_merge<M_F32><<<mb, 256, 0, s>>>(ids, keys, k, n_t, ncnt, nfill, noff, sorted, prow, member_cap, part_of,
                                                          local_idx);
  else if (metric == M_JW) k_node_merge<M_JW><<<mb, 256, 0, s>>>(ids, keys, k, n_t, ncnt, nfill, noff, sorted, prow, member_cap, part_of,
                                                          local_idx);
  else if (metric == M_COS) k_node_merge<M_COS><<<mb, 256, 0, s>>>(ids, keys, k, n_t, ncnt, nfill, noff, sorted, prow, member_cap, part_of,
                                                          local_idx);
  else k_node_merge<M_JAC><<<mb, 256, 0, s>>>(ids, keys, k, n_t, ncnt, nfill, noff, sorted, prow, member_cap, part_of,
                                                          local_idx);
  if (n_launch) *n_launch += 6;
  return cudaGetLastError();
}

// The partition-local store of nodes [first, first + count) (read by K1 on partitioned graphs): row v of
// partition p = part_of[v] at local index l = local_idx[v] holds the local index of each entry in p (-1
// across partitions, Q10); vector rows / token ranges are copied to the same (p, l) slot.
__global__ void k_local_rows(const int32_t *ids, int k, int64_t first, int64_t count, const uint8_t *part_of,
                             const int32_t *local_idx, int32_t *prow, int64_t cap) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count * k) return;
  const int64_t v = first + i / k;
  const int e = (int)(i % k);
  const int32_t u = ids[v * k + e];
  const uint8_t pv = part_of[v];
  prow[((size_t)pv * cap + local_idx[v]) * k + e] = (u >= 0 && part_of[u] == pv) ? local_idx[u] : -1;
}
__global__ void k_local_vecs(const uint8_t *vec, int nchunks, size_t stride, int64_t first, int64_t count,
                             const uint8_t *part_of, const int32_t *local_idx, uint8_t *pvec, int64_t cap) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count * nchunks) return;
  const int64_t v = first + i / nchunks;
  const int c = (int)(i % nchunks);
  const uint4 x = *(const uint4 *)(vec + (size_t)v * stride + 16 * c);
  *(uint4 *)(pvec + ((size_t)part_of[v] * cap + local_idx[v]) * stride + 16 * c) = x;
}
__global__ void k_local_sets(const uint64_t *off, int64_t first, int64_t count, const uint8_t *part_of,
                             const int32_t *local_idx, ulonglong2 *pset, int64_t cap) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const int64_t v = first + i;
  pset[(size_t)part_of[v] * cap + local_idx[v]] = make_ulonglong2(off[v], off[v + 1]);
}

cudaError_t launch_local_store(const StoreView &st, const int32_t *ids, int k, int64_t first, int64_t count,
                               const uint8_t *part_of, const int32_t *local_idx, const LocalStore &ls, cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  const int64_t nr = count * k;
  k_local_rows<<<(unsigned)((nr + 255) / 256), 256, 0, s>>>(ids, k, first, count, part_of, local_idx, ls.prow, ls.cap);
  if (ls.pvec) {
    const int64_t nv = count * st.nchunks;
    k_local_vecs<<<(unsigned)((nv + 255) / 256), 256, 0, s>>>(st.vec, st.nchunks, st.stride, first, count, part_of,
                                                              local_idx, ls.pvec, ls.cap);
  }
  if (ls.pset)
    k_local_sets<<<(unsigned)((count + 255) / 256), 256, 0, s>>>(st.off, first, count, part_of, local_idx, ls.pset,
                                                                 ls.cap);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// K6: nearest medoid (ties -> lowest p) and ordered append to the member lists.
// Single block: new ids are appended in batch order, so member lists stay ascending.
// ---------------------------------------------------------------------------
template <int M>
__global__ void k_place_target(StoreView st, int64_t n_t, int64_t B, int P, const int32_t *medoids, int32_t *target) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= B) return;
  int best = 0;
  uint32_t bk = 0;
  for (int p = 0; p < P; ++p) {
    const uint32_t kp = pair_key<M>(st, n_t + i, medoids[p]);
    if (p == 0 || closer<M>(kp, bk)) { best = p; bk = kp; }
  }
  target[i] = best;
}

__global__ void k_place_append(int64_t n_t, int64_t B, int P, const int32_t *target, int32_t *members,
                               int64_t member_cap, int64_t *member_cnt, uint8_t *part_of, int32_t *local_idx) {
  // one block of 1024 threads; per chunk of 1024 points, rank = # earlier points with the same target
  __shared__ int32_t tg[1024];
  __shared__ int64_t base[256];
  for (int p = threadIdx.x; p < P; p += blockDim.x) base[p] = member_cnt[p];
  __syncthreads();
  for (int64_t c0 = 0; c0 < B; c0 += 1024) {
    const int64_t i = c0 + threadIdx.x;
    const int t = i < B ? target[i] : -1;
    tg[threadIdx.x] = t;
    __syncthreads();
    if (t >= 0) {
      int r = 0;
      for (int j = 0; j < (int)threadIdx.x; ++j) r += tg[j] == t;
      const int64_t pos = base[t] + r;
      members[(size_t)t * member_cap + pos] = (int32_t)(n_t + i);
      part_of[n_t + i] = (uint8_t)t;
      local_idx[n_t + i] = (int32_t)pos;
    }
    __syncthreads();
    if (threadIdx.x < (unsigned)P) {
      int cnt = 0;
      for (int j = 0; j < 1024; ++j) cnt += tg[j] == (int)threadIdx.x;
      base[threadIdx.x] += cnt;
    }
    __syncthreads();
  }
  for (int p = threadIdx.x; p < P; p += blockDim.x) member_cnt[p] = base[p];
}

// key of query row i of qs against graph row j of st (two stores)
template <int M>
__device__ __forceinline__ uint32_t cross_key(const StoreView &qs, int64_t i, const StoreView &st, int64_t j) {
  if (M == M_JAC) {
    const uint64_t ai = qs.off[i], bj = st.off[j];
    return set_key(qs.tok + ai, (int)(qs.off[i + 1] - ai), st.tok + bj, (int)(st.off[j + 1] - bj));
  }
  return thread_dist<M>((const uint4 *)(qs.vec + (size_t)i * qs.stride), (const uint4 *)(st.vec + (size_t)j * st.stride),
                        st.nchunks);
}
template <int M>
__global__ void k_route_target(StoreView qs, int64_t qrow0, int64_t nq, StoreView st, int P, const int32_t *medoids,
                               int32_t *target) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nq) return;
  int best = 0;
  uint32_t bk = 0;
  for (int p = 0; p < P; ++p) {
    const uint32_t kp = cross_key<M>(qs, qrow0 + i, st, medoids[p]);
    if (p == 0 || closer<M>(kp, bk)) { best = p; bk = kp; }
  }
  target[i] = best;
}
cudaError_t launch_route_target(const VecGeom &g, const StoreView &qs, int64_t qrow0, int64_t nq, const StoreView &st,
                                int P, const int32_t *medoids, int32_t *target, cudaStream_t s) {
  if (nq == 0) return cudaSuccess;
  const unsigned blocks = (unsigned)((nq + 127) / 128);
  if (g.metric == M_U8) k_route_target<M_U8><<<blocks, 128, 0, s>>>(qs, qrow0, nq, st, P, medoids, target);
  else if (g.metric == M_F32) k_route_target<M_F32><<<blocks, 128, 0, s>>>(qs, qrow0, nq, st, P, medoids, target);
  else k_route_target<M_JAC><<<blocks, 128, 0, s>>>(qs, qrow0, nq, st, P, medoids, target);
  return cudaGetLastError();
}

cudaError_t launch_place(const VecGeom &g, const StoreView &st, int64_t n_t, int64_t B, int P, const int32_t *medoids,
                         int32_t *members, int64_t member_cap, int64_t *member_cnt, uint8_t *part_of,
                         int32_t *local_idx, int32_t *target, cudaStream_t s) {
  if (B == 0) return cudaSuccess;
  const unsigned blocks = (unsigned)((B + 127) / 128);
  if (g.metric == M_U8) k_place_target<M_U8><<<blocks, 128, 0, s>>>(st, n_t, B, P, medoids, target);
  else if (g.metric == M_F32) k_place_target<M_F32><<<blocks, 128, 0, s>>>(st, n_t, B, P, medoids, target);
  else k_place_target<M_JAC><<<blocks, 128, 0, s>>>(st, n_t, B, P, medoids, target);
  k_place_append<<<1, 1024, 0, s>>>(n_t, B, P, target, members, member_cap, member_cnt, part_of, local_idx);
  return cudaGetLastError();
}

}  // namespace knng
