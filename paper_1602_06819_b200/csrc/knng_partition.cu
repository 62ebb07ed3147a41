// knng_partition.cu -- K8 balanced k-medoids of the graph (Alg. 4; readings
// Q21-Q23) and the partition state used by Alg. 3 / Alg. 5.
//
// One iteration, all on the device:
//   assign  : keys D(node, medoid_p) for every node (thread per node), then the capacity-
//             constrained greedy pass in ascending node id (c = 1): a single warp,
//             lane l owning clusters l, l+32, ...; each node goes to the eligible cluster with the
//             largest similarity * (1 - |C|/capacity), compared exactly by cross-multiplication,
//             ties -> smaller size -> smaller medoid id.
//   update  : per-cluster ascending member lists (scan), the cluster-induced undirected adjacency
//             (CSR), and the hop sums of the candidate medoids by a bit-parallel multi-source BFS:
//             64 candidates of every cluster advance together, one bit each ("shortest
//             path ... Dijkstra" on unit weights); unreachable members cost |C|.
// The accept / stop rule of Q23 is host control flow over device-computed costs.
#include <math.h>
#include <string.h>

#include <algorithm>

#include "knng_common.cuh"
#include "knng_handle.h"

namespace knng {

cudaError_t exclusive_scan_i32(const int32_t *in, int32_t *out, int32_t *tmp, int64_t n, cudaStream_t s);

__global__ void k_init_medoids(uint64_t seed, int64_t n, int P, int32_t *med) {
  if (threadIdx.x || blockIdx.x) return;
  const uint64_t h3 = rng_prefix(seed, 0xFFFFFFFFull, 0);   // stream (seed, 0xFFFFFFFF, 0, j)
  int got = 0;
  uint64_t j = 0;
  while (got < P) {
    const int32_t c = (int32_t)rng_index(h3, j++, (uint64_t)n);
    bool dup = false;
    for (int i = 0; i < got; ++i) dup |= med[i] == c;
    if (!dup) med[got++] = c;
  }
}

template <int M>
__global__ void k_medoid_keys(StoreView st, int64_t n, int P, const int32_t *med, uint32_t *D) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int p = 0; p < P; ++p) D[(size_t)i * P + p] = pair_key<M>(st, i, med[p]);
}

// assign comparison: cluster a (key ka, size sa) strictly above b (P:188 score sim * w)
template <int M>
__device__ __forceinline__ bool assign_better(uint32_t ka, int64_t sa, uint32_t kb, int64_t sb, int64_t cap) {
  if (M == M_U8) return (uint64_t)(cap - sa) * (1ull + kb) > (uint64_t)(cap - sb) * (1ull + ka);
  if (M == M_F32) {
    const double l = __dmul_rn((double)(cap - sa), __dadd_rn(1.0, (double)__uint_as_float(kb)));
    const double r = __dmul_rn((double)(cap - sb), __dadd_rn(1.0, (double)__uint_as_float(ka)));
    return l > r;
  }
  return (uint64_t)(ka >> 16) * (uint64_t)(cap - sa) * (uint64_t)(kb & 0xFFFFu) >
         (uint64_t)(kb >> 16) * (uint64_t)(cap - sb) * (uint64_t)(ka & 0xFFFFu);
}

template <int M>
__device__ __forceinline__ bool cand_beats(bool va, uint32_t ka, int64_t sa, int32_t ma, bool vb, uint32_t kb,
                                           int64_t sb, int32_t mb, int64_t cap) {
  if (!vb) return va;
  if (!va) return false;
  if (assign_better<M>(ka, sa, kb, sb, cap)) return true;
  if (assign_better<M>(kb, sb, ka, sa, cap)) return false;
  if (sa != sb) return sa < sb;
  return ma < mb;
}

template <int M>
__global__ void __launch_bounds__(32) k_greedy_assign(const uint32_t *D, int64_t n, int P, const int32_t *med,
                                                      int64_t cap, uint8_t *part, int64_t *sizes_out) {
  const int lane = threadIdx.x;
  const int TP = (P + 31) / 32;
  int64_t sz[8];
  int32_t mid[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    sz[t] = 0;
    const int p = lane + 32 * t;
    mid[t] = (t < TP && p < P) ? med[p] : 0x7FFFFFFF;
  }
  uint32_t nk[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    const int p = lane + 32 * t;
    nk[t] = (t < TP && p < P && n > 0) ? D[p] : 0u;
  }
  for (int64_t i = 0; i < n; ++i) {
    uint32_t ck[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) ck[t] = nk[t];
    if (i + 1 < n) {   // prefetch the next node's keys
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const int p = lane + 32 * t;
        if (t < TP && p < P) nk[t] = D[(size_t)(i + 1) * P + p];
      }
    }
    // lane-local best
    bool bv = false;
    uint32_t bk = 0;
    int64_t bs = 0;
    int32_t bm = 0x7FFFFFFF;
    int bp = -1;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const int p = lane + 32 * t;
      const bool v = t < TP && p < P && sz[t] < cap;   // full clusters are ineligible
      if (cand_beats<M>(v, ck[t], sz[t], mid[t], bv, bk, bs, bm, cap)) {
        bv = v; bk = ck[t]; bs = sz[t]; bm = mid[t]; bp = p;
      }
    }
    // warp arg-best (strict total order -> reduction order is irrelevant)
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      const bool ov = __shfl_xor_sync(FULL, bv, o);
      const uint32_t okk = __shfl_xor_sync(FULL, bk, o);
      const int64_t os = __shfl_xor_sync(FULL, bs, o);
      const int32_t om = __shfl_xor_sync(FULL, bm, o);
      const int op = __shfl_xor_sync(FULL, bp, o);
      if (cand_beats<M>(ov, okk, os, om, bv, bk, bs, bm, cap)) { bv = ov; bk = okk; bs = os; bm = om; bp = op; }
    }
#pragma unroll
    for (int t = 0; t < 8; ++t)
      if (lane + 32 * t == bp) ++sz[t];
    if (lane == 0) part[i] = (uint8_t)bp;
  }
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    const int p = lane + 32 * t;
    if (t < TP && p < P) sizes_out[p] = sz[t];
  }
}

__global__ void k_flag_eq(const uint8_t *part, int64_t n, int p, int32_t *flag) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) flag[i] = part[i] == p;
}
__global__ void k_place_members(const uint8_t *part, int64_t n, int p, const int32_t *scan, int32_t *local_idx,
                                int32_t *members, int64_t member_cap) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && part[i] == p) {
    local_idx[i] = scan[i];
    members[(size_t)p * member_cap + scan[i]] = (int32_t)i;
  }
}

// undirected cluster-induced adjacency over cluster-major positions pos(i) = base[part i] + local i
__global__ void k_adj_degree(const int32_t *ids, int k, int64_t n, const uint8_t *part, const int32_t *local_idx,
                             const int64_t *base, int32_t *deg) {
  const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= n) return;
  const int pu = part[u];
  const int64_t su = base[pu] + local_idx[u];
  for (int e = 0; e < k; ++e) {
    const int32_t v = ids[u * k + e];
    if (v < 0 || part[v] != pu) continue;
    atomicAdd(deg + su, 1);
    atomicAdd(deg + base[pu] + local_idx[v], 1);
  }
}
__global__ void k_adj_fill(const int32_t *ids, int k, int64_t n, const uint8_t *part, const int32_t *local_idx,
                           const int64_t *base, const int32_t *off, int32_t *fill, int32_t *adj) {
  const int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= n) return;
  const int pu = part[u];
  const int64_t su = base[pu] + local_idx[u];
  for (int e = 0; e < k; ++e) {
    const int32_t v = ids[u * k + e];
    if (v < 0 || part[v] != pu) continue;
    const int64_t sv = base[pu] + local_idx[v];
    adj[off[su] + atomicAdd(fill + su, 1)] = (int32_t)sv;
    adj[off[sv] + atomicAdd(fill + sv, 1)] = (int32_t)su;
  }
}
__global__ void k_cluster_of(const int64_t *base, int P, int64_t n, uint8_t *cl) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  int p = 0;
  while (p + 1 < P && base[p + 1] <= s) ++p;
  cl[s] = (uint8_t)p;
}

// candidates (Q22): all members if |C| <= exact_limit, else {current medoid if member} u draws
__global__ void k_candidates(const int64_t *sizes, const int32_t *med, const uint8_t *part, const int32_t *local_idx,
                             int P, int64_t exact_limit, int ncand, uint64_t seed, uint64_t tag, int64_t iter,
                             int32_t *cand, int32_t *ncand_out, int candcap) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  const int64_t sz = sizes[p];
  int32_t *c = cand + (size_t)p * candcap;
  int cnt = 0;
  if (sz == 0) {
  } else if (sz <= exact_limit) {
    for (int64_t i = 0; i < sz; ++i) c[cnt++] = (int32_t)i;
  } else {
    if (part[med[p]] == p) c[cnt++] = local_idx[med[p]];
    const uint64_t h3 = rng_prefix(seed, tag, (uint64_t)(iter * P + p));   // stream (seed, tag, iter P + p, j)
    for (int j = 0; j < ncand - 1; ++j) c[cnt++] = (int32_t)rng_index(h3, (uint64_t)j, (uint64_t)sz);
  }
  ncand_out[p] = cnt;
}

__global__ void k_bfs_init(int64_t n, unsigned long long *vis, unsigned long long *fr) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s < n) { vis[s] = 0; fr[s] = 0; }
}
__global__ void k_bfs_seed(const int64_t *base, int P, const int32_t *cand, const int32_t *ncand, int candcap, int b,
                           unsigned long long *vis, unsigned long long *fr, unsigned long long *reach) {
  const int p = blockIdx.x;
  const int j = threadIdx.x;   // 64 threads
  const int ci = b * 64 + j;
  if (ci < ncand[p]) {
    const int64_t s = base[p] + cand[(size_t)p * candcap + ci];
    atomicOr(vis + s, 1ull << j);
    atomicOr(fr + s, 1ull << j);
    reach[p * 64 + j] = 1;
  } else {
    reach[p * 64 + j] = 0;
  }
}
__global__ void k_bfs_level(int64_t n, const int32_t *off, const int32_t *adj, const uint8_t *cl,
                            unsigned long long *vis, const unsigned long long *fr, unsigned long long *nx,
                            unsigned long long *hop, unsigned long long *reach, unsigned long long level, int *any) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  unsigned long long nw = 0;
  int p = -1;
  if (s < n) {
    unsigned long long acc = 0;
    for (int e = off[s]; e < off[s + 1]; ++e) acc |= fr[adj[e]];
    nw = acc & ~vis[s];
    vis[s] |= nw;
    nx[s] = nw;
    p = cl[s];
  }
  const unsigned act = __ballot_sync(FULL, nw != 0);
  if (!act) return;
  if (lane == 0) *any = 1;
  const int p0 = __shfl_sync(FULL, p, __ffs(act) - 1);
  const bool uni = __all_sync(FULL, nw == 0 || p == p0);
  if (uni) {
    for (int j = 0; j < 64; ++j) {
      const int c = __popc(__ballot_sync(FULL, (nw >> j) & 1ull));
      if (c && lane == 0) {
        atomicAdd(hop + p0 * 64 + j, level * (unsigned long long)c);
        atomicAdd(reach + p0 * 64 + j, (unsigned long long)c);
      }
    }
  } else {
    for (int j = 0; j < 64; ++j)
      if ((nw >> j) & 1ull) {
        atomicAdd(hop + p * 64 + j, level);
        atomicAdd(reach + p * 64 + j, 1ull);
      }
  }
}
// fold one batch of 64 candidates into the per-cluster best (min hop sum, ties -> smaller id)
__global__ void k_bfs_pick(int P, const int64_t *sizes, const int32_t *cand, const int32_t *ncand, int candcap,
                           int b, const int32_t *members, int64_t member_cap, const unsigned long long *hop,
                           const unsigned long long *reach, unsigned long long *best_sum, int32_t *best_id) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  const int64_t sz = sizes[p];
  for (int j = 0; j < 64; ++j) {
    const int ci = b * 64 + j;
    if (ci >= ncand[p]) break;
    const unsigned long long s = hop[p * 64 + j] + (unsigned long long)(sz - (int64_t)reach[p * 64 + j]) * sz;
    const int32_t id = members[(size_t)p * member_cap + cand[(size_t)p * candcap + ci]];
    if (best_id[p] < 0 || s < best_sum[p] || (s == best_sum[p] && id < best_id[p])) {
      best_sum[p] = s;
      best_id[p] = id;
    }
  }
}

}  // namespace knng

using namespace knng;

// (re)build members / local_idx / member_cnt from part_of for nodes 0..n-1
static int build_members(knng_graph *g, int32_t *flag, int32_t *scan, int32_t *tmp) {
  const int64_t n = g->n;
  const unsigned nb = (unsigned)((n + 255) / 256);
  std::vector<int64_t> cnt(g->P);
  for (int p = 0; p < g->P; ++p) {
    k_flag_eq<<<nb, 256, 0, g->stream>>>(g->part_of, n, p, flag);
    CK(exclusive_scan_i32(flag, scan, tmp, n, g->stream));
    k_place_members<<<nb, 256, 0, g->stream>>>(g->part_of, n, p, scan, g->local_idx, g->members, g->cap);
    int32_t last[2];
    CK(cudaMemcpyAsync(&last[0], scan + n - 1, 4, cudaMemcpyDeviceToHost, g->stream));
    CK(cudaMemcpyAsync(&last[1], flag + n - 1, 4, cudaMemcpyDeviceToHost, g->stream));
    CK(cudaStreamSynchronize(g->stream));
    cnt[p] = (int64_t)last[0] + last[1];
  }
  CK(cudaMemcpyAsync(g->member_cnt, cnt.data(), sizeof(int64_t) * g->P, cudaMemcpyHostToDevice, g->stream));
  CK(cudaStreamSynchronize(g->stream));
  return 0;
}

// the partition-local store K1 reads (rows, and vectors or token ranges, at (p, local index)), for the
// installed partition of nodes 0..n-1
static int build_local_store(knng_graph *g) {
  if (g->local_P != g->P) {
    if (g->prow) cudaFree(g->prow);
    if (g->pvec) cudaFree(g->pvec);
    if (g->pset) cudaFree(g->pset);
    g->prow = nullptr; g->pvec = nullptr; g->pset = nullptr;
    g->local_P = 0;
    const size_t rows = (size_t)g->P * g->cap;
    CK(cudaMalloc((void **)&g->prow, rows * g->k * 4));
    if (g->metric == KNNG_JACCARD_U32SET) CK(cudaMalloc((void **)&g->pset, rows * sizeof(ulonglong2)));
    else CK(cudaMalloc((void **)&g->pvec, rows * g->geom.stride));
    g->local_P = g->P;
  }
  CK(launch_local_store(graph_store_view(g), g->ids, g->k, 0, g->n, g->part_of, g->local_idx, graph_local_store(g),
                        g->stream));
  CK(cudaStreamSynchronize(g->stream));
  return 0;
}

// Device workspace of Alg. 4 (sized for n nodes, P clusters, degree k).
struct PartWs {
  DBuf wD, wpart, wacc, wflag, wscan, wtmp, wdeg, woff, wfill, wadj, wcl, wvis, wfr, wnx, wcand, wnc, whop, wreach,
      wbs, wbi, wsz, wbase, wany, wmed;
  int candcap = 0;
  cudaError_t ensure(int64_t n, int P, int k, int candcap_) {
    candcap = candcap_;
    cudaError_t e = cudaSuccess;
    auto E = [&](DBuf &b, size_t bytes) { if (e == cudaSuccess) e = b.ensure(bytes); };
    E(wD, (size_t)n * P * 4);
    E(wpart, (size_t)n);
    E(wacc, (size_t)n);
    E(wflag, (size_t)(n + 1) * 4);
    E(wscan, (size_t)(n + 1) * 4);
    E(wtmp, (size_t)((n + 1) / 1024 + 2) * 4);
    E(wdeg, (size_t)(n + 1) * 4);
    E(woff, (size_t)(n + 1) * 4);
    E(wfill, (size_t)(n + 1) * 4);
    E(wadj, (size_t)2 * n * k * 4 + 4);
    E(wcl, (size_t)n);
    E(wvis, (size_t)n * 8);
    E(wfr, (size_t)n * 8);
    E(wnx, (size_t)n * 8);
    E(wcand, (size_t)P * candcap * 4);
    E(wnc, (size_t)P * 4);
    E(whop, (size_t)P * 64 * 8);
    E(wreach, (size_t)P * 64 * 8);
    E(wbs, (size_t)P * 8);
    E(wbi, (size_t)P * 4);
    E(wsz, (size_t)P * 8);
    E(wbase, (size_t)(P + 1) * 8);
    E(wany, 8);
    E(wmed, (size_t)P * 4);
    return e;
  }
  ~PartWs() {
    DBuf *all[] = {&wD, &wpart, &wacc, &wflag, &wscan, &wtmp, &wdeg, &woff, &wfill, &wadj, &wcl, &wvis, &wfr, &wnx,
                   &wcand, &wnc, &whop, &wreach, &wbs, &wbi, &wsz, &wbase, &wany, &wmed};
    for (DBuf *b : all) b->release();
  }
};

// The update step of Alg. 4 on the current assignment g->part_of: member lists, the
// cluster-induced undirected adjacency, and per cluster the candidate (reading Q22: every member when
// |C| <= exact_limit, else the current medoid and ncand - 1 draws of stream (seed, tag, iter P + p, j))
// minimising the hop sum; unreachable members cost |C|, ties -> smaller id.  Empty clusters keep their
// medoid and add nothing to the cost.
static int medoid_update(knng_graph *g, int P, const std::vector<int32_t> &med, uint64_t seed, uint64_t tag,
                         int64_t iter, int64_t exact_limit, int ncand, PartWs &w, std::vector<int32_t> &newmed,
                         int64_t *cost_out) {
  const int64_t n = g->n;
  const int k = g->k;
  const int candcap = w.candcap;
  cudaStream_t s = g->stream;
  const unsigned nb = (unsigned)((n + 255) / 256);
  CK(cudaMemcpyAsync(w.wmed.p, med.data(), (size_t)P * 4, cudaMemcpyHostToDevice, s));
  g->P = P;
  if (int r = build_members(g, w.wflag.as<int32_t>(), w.wscan.as<int32_t>(), w.wtmp.as<int32_t>())) return r;
  std::vector<int64_t> sizes(P), base(P + 1, 0);
  CK(cudaMemcpyAsync(sizes.data(), g->member_cnt, (size_t)P * 8, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  for (int p = 0; p < P; ++p) base[p + 1] = base[p] + sizes[p];
  CK(cudaMemcpyAsync(w.wbase.p, base.data(), (size_t)(P + 1) * 8, cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(w.wsz.p, sizes.data(), (size_t)P * 8, cudaMemcpyHostToDevice, s));
  CK(cudaMemsetAsync(w.wdeg.p, 0, (size_t)(n + 1) * 4, s));
  CK(cudaMemsetAsync(w.wfill.p, 0, (size_t)(n + 1) * 4, s));
  k_adj_degree<<<nb, 256, 0, s>>>(g->ids, k, n, g->part_of, g->local_idx, w.wbase.as<int64_t>(), w.wdeg.as<int32_t>());
  CK(exclusive_scan_i32(w.wdeg.as<int32_t>(), w.woff.as<int32_t>(), w.wtmp.as<int32_t>(), n + 1, s));
  k_adj_fill<<<nb, 256, 0, s>>>(g->ids, k, n, g->part_of, g->local_idx, w.wbase.as<int64_t>(), w.woff.as<int32_t>(),
                                w.wfill.as<int32_t>(), w.wadj.as<int32_t>());
  k_cluster_of<<<nb, 256, 0, s>>>(w.wbase.as<int64_t>(), P, n, w.wcl.as<uint8_t>());
  k_candidates<<<(P + 63) / 64, 64, 0, s>>>(w.wsz.as<int64_t>(), w.wmed.as<int32_t>(), g->part_of, g->local_idx, P,
                                            exact_limit, ncand, seed, tag, iter, w.wcand.as<int32_t>(),
                                            w.wnc.as<int32_t>(), candcap);
  std::vector<int32_t> nc(P);
  CK(cudaMemcpyAsync(nc.data(), w.wnc.p, (size_t)P * 4, cudaMemcpyDeviceToHost, s));
  CK(cudaMemsetAsync(w.wbi.p, 0xFF, (size_t)P * 4, s));
  CK(cudaStreamSynchronize(s));
  int maxc = 0;
  for (int p = 0; p < P; ++p) maxc = std::max(maxc, nc[p]);
  for (int b = 0; b * 64 < maxc; ++b) {
    k_bfs_init<<<nb, 256, 0, s>>>(n, w.wvis.as<unsigned long long>(), w.wfr.as<unsigned long long>());
    CK(cudaMemsetAsync(w.whop.p, 0, (size_t)P * 64 * 8, s));
    k_bfs_seed<<<P, 64, 0, s>>>(w.wbase.as<int64_t>(), P, w.wcand.as<int32_t>(), w.wnc.as<int32_t>(), candcap, b,
                                w.wvis.as<unsigned long long>(), w.wfr.as<unsigned long long>(),
                                w.wreach.as<unsigned long long>());
    for (unsigned long long level = 1;; ++level) {
      CK(cudaMemsetAsync(w.wany.p, 0, 4, s));
      k_bfs_level<<<nb, 256, 0, s>>>(n, w.woff.as<int32_t>(), w.wadj.as<int32_t>(), w.wcl.as<uint8_t>(),
                                     w.wvis.as<unsigned long long>(), w.wfr.as<unsigned long long>(),
                                     w.wnx.as<unsigned long long>(), w.whop.as<unsigned long long>(),
                                     w.wreach.as<unsigned long long>(), level, w.wany.as<int>());
      int any = 0;
      CK(cudaMemcpyAsync(&any, w.wany.p, 4, cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      std::swap(w.wfr.p, w.wnx.p);
      std::swap(w.wfr.bytes, w.wnx.bytes);
      if (!any) break;
    }
    k_bfs_pick<<<(P + 63) / 64, 64, 0, s>>>(P, w.wsz.as<int64_t>(), w.wcand.as<int32_t>(), w.wnc.as<int32_t>(),
                                            candcap, b, g->members, g->cap, w.whop.as<unsigned long long>(),
                                            w.wreach.as<unsigned long long>(), w.wbs.as<unsigned long long>(),
                                            w.wbi.as<int32_t>());
  }
  std::vector<unsigned long long> bsum(P);
  newmed.assign(P, 0);
  CK(cudaMemcpyAsync(bsum.data(), w.wbs.p, (size_t)P * 8, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(newmed.data(), w.wbi.p, (size_t)P * 4, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  CK(cudaGetLastError());
  int64_t cost = 0;
  for (int p = 0; p < P; ++p) {
    if (sizes[p] == 0) { newmed[p] = med[p]; continue; }
    cost += (int64_t)bsum[p];
  }
  *cost_out = cost;
  return 0;
}

static void install_medoids(knng_graph *g, const std::vector<int32_t> &med) {
  cudaMemcpyAsync(g->medoids, med.data(), med.size() * 4, cudaMemcpyHostToDevice, g->stream);
  g->h_medoids = med;
  g->pool_bound = 0;        // the next search reads the partition sizes
  g->cnt_pending = false;
}

extern "C" int partition_kmedoids(knng_graph *g, int32_t P, double imbalance, int32_t max_iter, uint64_t seed,
                                  uint8_t *part_out, int32_t *medoids_out, int64_t *cost_out,
                                  const int32_t *init_medoids) {
  knng_err_slot().clear();
  if (!g) return fail(KNNG_ERR_INVALID_ARG, "partition_kmedoids: null graph");
  if (g->metric == KNNG_JARO_WINKLER || g->metric == KNNG_COSINE_2GRAM)
    return fail(KNNG_ERR_INVALID_ARG, "partition_kmedoids: string metrics run on unpartitioned graphs");
  if (P < 1 || P > 255) return fail(KNNG_ERR_INVALID_ARG, "partition_kmedoids: P=%d outside 1..255", P);
  if (!(imbalance >= 1.0)) return fail(KNNG_ERR_INVALID_ARG, "partition_kmedoids: imbalance < 1");
  if (max_iter < 1) return fail(KNNG_ERR_INVALID_ARG, "partition_kmedoids: max_iter < 1");
  if (!medoids_out) return fail(KNNG_ERR_INVALID_ARG, "partition_kmedoids: null medoids_out");
  const int64_t n = g->n;
  if (n < P) return fail(KNNG_ERR_INVALID_ARG, "partition_kmedoids: n < P");
  const int64_t cap = (int64_t)ceil((double)n * imbalance / (double)P);   // F4, ceil
  if (cap * P < n) return fail(KNNG_ERR_CAPACITY_INFEAS, "capacity %lld x %d < n", (long long)cap, P);
  for (int i = 0; init_medoids && i < P; ++i)
    if (init_medoids[i] < 0 || init_medoids[i] >= n) return fail(KNNG_ERR_INVALID_ARG, "bad init medoid");
  CK(cudaSetDevice(g->device));
  cudaStream_t s = g->stream;
  const int64_t exact_limit = 4096;
  const int ncand = 64;

  // partition state of the handle (member lists sized for the whole capacity)
  if (!g->part_of) {
    CK(cudaMalloc((void **)&g->part_of, (size_t)g->cap));
    CK(cudaMalloc((void **)&g->local_idx, (size_t)g->cap * 4));
  }
  if (g->members) cudaFree(g->members);
  if (g->member_cnt) cudaFree(g->member_cnt);
  if (g->medoids) cudaFree(g->medoids);
  g->members = nullptr; g->member_cnt = nullptr; g->medoids = nullptr;
  g->P = 0;
  CK(cudaMalloc((void **)&g->members, (size_t)P * g->cap * 4));
  CK(cudaMalloc((void **)&g->member_cnt, (size_t)P * 8));
  CK(cudaMalloc((void **)&g->medoids, (size_t)P * 4));

  PartWs w;
  CK(w.ensure(n, P, g->k, (int)std::max<int64_t>(exact_limit, ncand)));
  const unsigned nb = (unsigned)((n + 255) / 256);

  // initial medoids (Alg. 4 "Randomly pick k initial medoids")
  if (init_medoids) CK(cudaMemcpyAsync(g->medoids, init_medoids, (size_t)P * 4, cudaMemcpyHostToDevice, s));
  else k_init_medoids<<<1, 1, 0, s>>>(seed, n, P, g->medoids);

  std::vector<int32_t> med(P), newmed(P);
  CK(cudaMemcpyAsync(med.data(), g->medoids, (size_t)P * 4, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (cost_out)
    for (int i = 0; i <= max_iter; ++i) cost_out[i] = -1;
  int accepted = 0;
  int64_t prev_cost = -1;
  // the handle's part_of doubles as the working assignment; the accepted one is kept in wacc
  for (int it = 0; it < max_iter; ++it) {
    // ---------------- assign ----------------
    CK(cudaMemcpyAsync(w.wmed.p, med.data(), (size_t)P * 4, cudaMemcpyHostToDevice, s));
    const StoreView st = graph_store_view(g);
    if (g->metric == KNNG_L2SQ_U8) {
      k_medoid_keys<M_U8><<<nb, 256, 0, s>>>(st, n, P, w.wmed.as<int32_t>(), w.wD.as<uint32_t>());
      k_greedy_assign<M_U8><<<1, 32, 0, s>>>(w.wD.as<uint32_t>(), n, P, w.wmed.as<int32_t>(), cap, g->part_of,
                                             w.wsz.as<int64_t>());
    } else if (g->metric == KNNG_L2SQ_F32) {
      k_medoid_keys<M_F32><<<nb, 256, 0, s>>>(st, n, P, w.wmed.as<int32_t>(), w.wD.as<uint32_t>());
      k_greedy_assign<M_F32><<<1, 32, 0, s>>>(w.wD.as<uint32_t>(), n, P, w.wmed.as<int32_t>(), cap, g->part_of,
                                              w.wsz.as<int64_t>());
    } else {
      k_medoid_keys<M_JAC><<<nb, 256, 0, s>>>(st, n, P, w.wmed.as<int32_t>(), w.wD.as<uint32_t>());
      k_greedy_assign<M_JAC><<<1, 32, 0, s>>>(w.wD.as<uint32_t>(), n, P, w.wmed.as<int32_t>(), cap, g->part_of,
                                              w.wsz.as<int64_t>());
    }
    CK(cudaGetLastError());
    // ---------------- update: members, adjacency, hop sums ----------------
    int64_t cost = 0;
    if (int r = medoid_update(g, P, med, seed, 0xFFFFFFFEull, it, exact_limit, ncand, w, newmed, &cost)) return r;
    // Q23: keep the iteration only if the total hop sum does not rise
    if (it > 0 && cost > prev_cost) break;
    CK(cudaMemcpyAsync(w.wacc.p, g->part_of, (size_t)n, cudaMemcpyDeviceToDevice, s));
    if (cost_out) cost_out[accepted] = cost;
    ++accepted;
    prev_cost = cost;
    bool changed = false;
    for (int p = 0; p < P; ++p) changed |= newmed[p] != med[p];
    med = newmed;
    if (!changed) break;
  }
  // install the accepted partition
  CK(cudaMemcpyAsync(g->part_of, w.wacc.p, (size_t)n, cudaMemcpyDeviceToDevice, s));
  g->P = P;
  if (int r = build_members(g, w.wflag.as<int32_t>(), w.wscan.as<int32_t>(), w.wtmp.as<int32_t>())) return r;
  if (int r = build_local_store(g)) return r;
  install_medoids(g, med);
  memcpy(medoids_out, med.data(), (size_t)P * 4);
  if (part_out) CK(cudaMemcpyAsync(part_out, g->part_of, (size_t)n, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return accepted;
}

// Alg. 5's last step ("compute new medoids"; F5 P:1349-1353): the update step of Alg. 4 on
// the current partition -- nodes keep their partitions (placement already assigned the inserted ones),
// every medoid becomes its cluster's hop-sum minimiser over the current graph.  Candidate draws use
// stream (seed, 0xFFFFFFFD, epoch P + p, j).
extern "C" int graph_recompute_medoids(knng_graph *g, uint64_t seed, int64_t epoch, int32_t *medoids_out,
                                       int64_t *cost_out) {
  knng_err_slot().clear();
  if (!g) return fail(KNNG_ERR_INVALID_ARG, "graph_recompute_medoids: null graph");
  if (g->P == 0) return fail(KNNG_ERR_INVALID_ARG, "graph_recompute_medoids: the graph is not partitioned");
  if (g->pend_B) return fail(KNNG_ERR_INVALID_ARG, "graph_recompute_medoids: a staged batch is pending");
  if (epoch < 0) return fail(KNNG_ERR_INVALID_ARG, "graph_recompute_medoids: epoch < 0");
  CK(cudaSetDevice(g->device));
  const int P = g->P;
  PartWs w;
  CK(w.ensure(g->n, P, g->k, 4096));
  std::vector<int32_t> med = g->h_medoids, newmed;
  int64_t cost = 0;
  if (int r = medoid_update(g, P, med, seed, 0xFFFFFFFDull, epoch, 4096, 64, w, newmed, &cost)) return r;
  install_medoids(g, newmed);
  if (medoids_out) memcpy(medoids_out, newmed.data(), (size_t)P * 4);
  if (cost_out) *cost_out = cost;
  CK(cudaStreamSynchronize(g->stream));
  return KNNG_OK;
}
