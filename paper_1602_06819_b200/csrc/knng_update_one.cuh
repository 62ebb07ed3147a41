// knng_update_one.cuh -- the update of a single insert (B = 1: the paper's sequential Alg. 2,
// P:127-151) run by one warp: new row = C (the search's top-k), the update ball over the snapshot rows
// (levels 1..DEPTH, dedup by a shared hash, Q12), the proposals (Q14) and their application in place.
// Used by k_update_one (knng_update.cu) and by K1's fused B = 1 launch (knng_search.cu).
#pragma once
#include "knng_common.cuh"
#include "knng_internal.h"

namespace knng {

// open-addressing insert; true when u was not present
__device__ __forceinline__ bool hash_insert(int32_t *h, int hcap, int32_t u) {
  uint32_t x = (uint32_t)u * 0x9E3779B1u;
  int pos = (int)(x >> 7) & (hcap - 1);
  for (;;) {
    const int32_t old = atomicCAS(h + pos, -1, u);
    if (old == -1) return true;
    if (old == u) return false;
    pos = (pos + 1) & (hcap - 1);
  }
}

// shared scratch of update_one_warp: hash [hcap], list [ballmax (even)], props [ballmax] int2
__host__ __device__ __forceinline__ size_t update_one_smem(int hcap, int ballmax) {
  return (size_t)(hcap + ballmax + (ballmax & 1)) * 4 + (size_t)ballmax * 8;
}

// C / Ckeys: the new point's search result (k entries, -1 padded).  nb / np: the ball and proposal
// counts are returned there (the fused launch sums them), else added to stats[4], [5].  kt: keys of
// the new point against nodes 0..n_t-1 (the fused launch's table), else evaluated here.
template <int M, int L, int CPL>
__device__ __forceinline__ void update_one_warp(const BallArgs &a, const int32_t *C, const uint32_t *Ckeys,
                                                int32_t *usm, int *s_n, uint32_t *qscr, int *nb, int *npr,
                                                const uint32_t *kt = nullptr, uint8_t *jwp = nullptr,
                                                int32_t *sids = nullptr) {
  const int lane = threadIdx.x & 31;
  const int k = a.k;
  const int32_t *rows = sids ? sids : a.ids;   // the rows the update reads (the fused launch's shared copy)
  int32_t *hash = usm;
  int32_t *list = hash + a.hcap;
  int2 *props = (int2 *)(list + a.ballmax + (a.ballmax & 1));
  const int32_t idx = (int32_t)a.n_t;            // the new point's id
  // new row n_t = C (the top-k of the search; B = 1 has no batch peers)
  if (lane < k) {
    a.ids[(size_t)idx * k + lane] = C[lane];
    if (sids) sids[(size_t)idx * k + lane] = C[lane];
    a.keys[(size_t)idx * k + lane] = Ckeys[lane];
  }
  for (int i = lane; i < a.hcap; i += 32) hash[i] = -1;
  if (lane == 0) *s_n = 0;
  __syncwarp();
  typename QuerySel<M, L, CPL>::T Q;
  if constexpr (M == M_JW) Q.ptr = jwp ? jwp + lane * JW_PTR : nullptr;
  if (!kt || str_metric(M)) Q.load(a.st, a.n_t, qscr);
  {
    const int32_t v = lane < k ? C[lane] : -1;
    const bool ins = v >= 0 && hash_insert(hash, a.hcap, v);
    const unsigned m = __ballot_sync(FULL, ins);
    if (ins) list[__popc(m & lanemask_lt())] = v;
    if (lane == 0) *s_n = __popc(m);
    __syncwarp();
  }
  // levels 1..DEPTH over the snapshot rows: collect the ball, evaluate, propose.  A level's rows are
  // read G = 32 / k at a time (lane = node g, entry e), four groups in flight before the inserts.
  const int G = 32 / k;
  const int gl = lane / k, ge = lane - gl * k;
  int lo = 0, hi = *(volatile int *)s_n, np = 0;
  for (int d = 1; d <= a.depth; ++d) {
    if (d < a.depth) {
      for (int gb = lo; gb < hi; gb += 4 * G) {
        int32_t u[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int t = gb + r * G + gl;
          u[r] = (gl < G && t < hi) ? rows[(size_t)list[t] * k + ge] : -1;
        }
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          if (u[r] >= 0 && u[r] != idx && hash_insert(hash, a.hcap, u[r])) {
            const int pos = atomicAdd(s_n, 1);
            if (pos < a.ballmax) list[pos] = u[r];
          }
        }
      }
    }
    for (int base = lo; base < hi; base += 32) {
      const int t = base + lane;
      const int32_t v = t < hi ? list[t] : -1;
      const int cnt = hi - base < 32 ? hi - base : 32;
      uint32_t key;
      if constexpr (str_metric(M)) key = Q.rkey(a.st, v);   // strings: v's own key of the new point (v's row)
      else key = kt ? (v >= 0 ? kt[v] : 0u) : Q.eval(a.st, v, cnt);   // kt: the fused launch's key table
      bool prop = false;
      if (v >= 0) prop = precedes<M>(key, idx, a.keys[(size_t)v * k + k - 1], rows[(size_t)v * k + k - 1]);
      const unsigned pm = __ballot_sync(FULL, prop);
      if (prop) props[np + __popc(pm & lanemask_lt())] = make_int2(v, (int)key);
      np += __popc(pm);
    }
    __syncwarp();
    lo = hi;
    const int sn = *(volatile int *)s_n;
    hi = sn < a.ballmax ? sn : a.ballmax;
    __syncwarp();
  }
  // apply (Q14): row_v = top-k(row_v u {(D, idx)}); G proposals at a time, k lanes each (distinct rows):
  // the row is read at once, the entry's position is a ballot, the tail shifts by one lane
  for (int j0 = 0; j0 < np; j0 += G) {
    const int j = j0 + gl;
    const bool act = gl < G && j < np;
    int32_t v = -1, ri = -1;
    uint32_t key = 0, rk = 0;
    if (act) {
      v = props[j].x;
      key = (uint32_t)props[j].y;
      ri = rows[(size_t)v * k + ge];
      rk = a.keys[(size_t)v * k + ge];
    }
    const bool before = act && precedes<M>(rk, ri, key, idx);   // entry e stays ahead of the new one
    const unsigned grp = (k == 32 ? FULL : ((1u << k) - 1u)) << (gl * k);
    const int pos = __popc(__ballot_sync(FULL, before) & grp);
    const uint32_t uk = __shfl_up_sync(FULL, rk, 1);
    const int32_t ui = __shfl_up_sync(FULL, ri, 1);
    if (act && ge >= pos) {
      a.keys[(size_t)v * k + ge] = ge == pos ? key : uk;
      a.ids[(size_t)v * k + ge] = ge == pos ? idx : ui;
      if (sids) sids[(size_t)v * k + ge] = ge == pos ? idx : ui;
    }
  }
  if (nb) {
    *nb = lo;
    *npr = np;
  } else if (lane == 0) {
    atomicAdd(a.stats + 4, (unsigned long long)lo);
    atomicAdd(a.stats + 5, (unsigned long long)np);
  }
}

}  // namespace knng
