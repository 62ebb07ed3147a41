// knng_search.cu -- K1 iGNNS search (section 3) and K2 partition merge (Alg. 3,
// P:166-178).
//
// One warp per (query, partition) task.  The search is a dependent pointer chase, so the
// commit order is the paper's sequential order (every evaluation, top-k insert, visited mark
// and move happens exactly as in the algorithm); the warp's 32 lanes work speculatively:
//   * walk step: the k neighbours of `cur` are gathered and evaluated together (16-byte
//     vector loads), then the scan "first neighbour that improves" is resolved with a
//     ballot; only the fresh evaluations up to that neighbour are committed (budget).
//   * restart: a window of 32 RNG draws (Q4) is held in lanes; redraws of evaluated nodes are
//     free; the next G fresh draws are evaluated together and their keys cached in registers,
//     so a run of skipped starts costs one round trip per G starts.
// Visited / expanded sets are bitmaps over the pool-local index, in shared memory when the pool
// is small enough, else in a per-warp-slot global workspace.
#include "knng_common.cuh"
#include "knng_internal.h"

namespace knng {

template <int M, int L, int CPL>
__global__ void __launch_bounds__(128) k_search(SearchArgs a) {
  extern __shared__ uint32_t smem_bits[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int wpb = blockDim.x >> 5;
  const int64_t gw = (int64_t)blockIdx.x * wpb + wib, nw = (int64_t)gridDim.x * wpb;
  const int Pn = a.P > 0 ? a.P : 1;
  const int64_t T = a.nq * Pn;
  uint32_t *bits = a.smem_bits ? smem_bits + (size_t)wib * a.bits_words : a.gbits + gw * a.bits_words;
  const int k = a.k;
  unsigned long long s_evals = 0, s_starts = 0, s_skip = 0, s_exp = 0;

  for (int64_t task = gw; task < T; task += nw) {
    const int64_t b = task / Pn;
    const int p = (int)(task % Pn);
    const int64_t m = a.P > 0 ? a.member_cnt[p] : a.n_t;
    const int32_t *pool = a.P > 0 ? a.members + (size_t)p * a.member_cap : nullptr;
    const int64_t words = (m + 31) >> 5;
    uint32_t *ev = bits, *ex = bits + words;
    for (int64_t w = lane; w < 2 * words; w += 32) bits[w] = 0;
    __syncwarp();

    // budget (Q6) -- never more than the pool (Q7)
    int64_t budget = (int64_t)floor((double)m / a.speedup);
    const int64_t lo = m < a.kr ? m : a.kr;
    if (budget < lo) budget = lo;
    if (budget > m) budget = m;

    VecQuery<M, L, CPL> Q;
    Q.load(a.qbase + (size_t)b * a.stride, a.nchunks);
    WarpTopK<M> top;
    top.init(a.kr);
    const uint64_t h3 = rng_prefix(a.seed, (uint64_t)(a.pid_base + b), (uint64_t)p);

    int64_t c = 0, jbase = 0;
    int32_t wnode = -1;
    uint32_t wkey = 0, wl = 0;
    bool whave = false;
    int wpos = 32;

    while (c < budget) {
      // ------------------------------ restart ------------------------------
      if (wpos >= 32) {
        const int64_t j = jbase + lane;
        if (a.starts) {
          wnode = j < a.nstarts ? a.starts[j] : -1;
        } else {
          const uint64_t idx = rng_index(h3, (uint64_t)j, (uint64_t)m);
          wnode = pool ? pool[idx] : (int32_t)idx;
        }
        wl = wnode >= 0 ? (a.P > 0 ? (uint32_t)a.local_idx[wnode] : (uint32_t)wnode) : 0u;
        jbase += 32;
        whave = false;
        wpos = 0;
      }
      const unsigned active = FULL << wpos;
      const unsigned invm = __ballot_sync(FULL, wnode < 0) & active;
      const unsigned lim = invm ? ((1u << (__ffs(invm) - 1)) - 1u) : FULL;
      const bool evb = wnode >= 0 ? bit_get(ev, wl) : true;
      const unsigned same = __match_any_sync(FULL, wnode) & active;
      const bool fresh = lane >= wpos && !evb && (__ffs(same) - 1) == lane;   // redraws are free (Q4)
      const unsigned fm = __ballot_sync(FULL, fresh) & active & lim;
      if (fm == 0) {
        if (invm) break;          // injected start sequence exhausted
        wpos = 32;
        continue;
      }
      // evaluate the next G fresh draws that have no cached key
      unsigned hm = __ballot_sync(FULL, whave);
      const unsigned need = first_bits(fm, a.G) & ~hm;
      if (need) {
        const int nn = __popc(need);
        const int src = lane < nn ? (int)__fns(need, 0, lane + 1) : 0;
        const int32_t cid = __shfl_sync(FULL, wnode, src);
        const uint32_t kk = Q.eval(a.vec, a.stride, a.nchunks, lane < nn ? cid : -1, nn);
        const int rank = __popc(need & lanemask_lt());
        const uint32_t mine = __shfl_sync(FULL, kk, rank & 31);
        if ((need >> lane) & 1u) { wkey = mine; whave = true; }
        hm |= need;
      }
      // committable: fresh draws in order up to the first one without a key
      const unsigned miss = fm & ~hm;
      unsigned cm = miss ? (fm & ((1u << (__ffs(miss) - 1)) - 1u)) : fm;
      if ((int64_t)__popc(cm) > budget - c) cm = first_bits(cm, (int)(budget - c));
      const bool inc = (cm >> lane) & 1u;
      // s_max before each draw: best of top-k and of the earlier committed draws
      uint32_t run = wkey;
      bool rv = inc;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t ok_ = __shfl_up_sync(FULL, run, o);
        const bool ov = __shfl_up_sync(FULL, rv, o);
        if (lane >= o && ov) {
          if (!rv || closer<M>(ok_, run)) run = ok_;
          rv = true;
        }
      }
      uint32_t bk = __shfl_up_sync(FULL, run, 1);
      bool bv = __shfl_up_sync(FULL, rv, 1) && lane > 0;
      if (top.cnt > 0) {
        const uint32_t tb = top.best();
        bk = (bv && closer<M>(bk, tb)) ? bk : tb;
        bv = true;
      }
      // first start never skipped (Q3): it is the only draw with no best before it
      const bool acc = inc && (!bv || !skip_start<M>(wkey, bk, a.e_num, a.e_den));
      const unsigned am = __ballot_sync(FULL, acc);
      const int al = am ? __ffs(am) - 1 : -1;
      const unsigned commit = am ? (cm & (al == 31 ? FULL : ((2u << al) - 1u))) : cm;
      const bool cmt = (commit >> lane) & 1u;
      if (cmt) bit_set(ev, wl);
      top.insert(cmt, wkey, wnode);          // Q5: skipped starts enter the top-k too
      const int ncm = __popc(commit);
      c += ncm;
      s_starts += ncm;
      s_skip += ncm - (am ? 1 : 0);
      __syncwarp();
      // budget reached: stop, unless a start was accepted -- then, as in the sequential
      // algorithm, its walk begins and ends at the first fresh evaluation it needs
      if (c >= budget && !am) break;
      if (!am) {
        wpos = miss ? (__ffs(miss) - 1) : 32;
        continue;
      }
      wpos = al + 1;

      // ------------------- hill climbing, eager first improvement -------------------
      int32_t cur = __shfl_sync(FULL, wnode, al);
      uint32_t kcur = __shfl_sync(FULL, wkey, al);
      uint32_t curl = __shfl_sync(FULL, wl, al);
      bool stop = false;
      for (;;) {
        if (lane == 0) bit_set(ex, curl);
        ++s_exp;
        const int32_t v = lane < k ? a.rows[(size_t)cur * k + lane] : -1;
        const bool inpool = v >= 0 && (a.P == 0 || a.part_of[v] == p);   // Q10
        const uint32_t lv = inpool ? (a.P > 0 ? (uint32_t)a.local_idx[v] : (uint32_t)v) : 0u;
        __syncwarp();
        const bool evb2 = inpool ? bit_get(ev, lv) : true;
        const bool exb2 = inpool ? bit_get(ex, lv) : false;
        const uint32_t key = Q.eval(a.vec, a.stride, a.nchunks, inpool ? v : -1, k);
        const bool imp = inpool && closer<M>(key, kcur);
        const unsigned im = __ballot_sync(FULL, imp);
        const int fi = im ? __ffs(im) - 1 : 31;
        const unsigned range = fi == 31 ? FULL : ((2u << fi) - 1u);
        unsigned fm2 = __ballot_sync(FULL, inpool && !evb2) & range;
        bool hit2 = false;
        if ((int64_t)__popc(fm2) > budget - c) { fm2 = first_bits(fm2, (int)(budget - c)); hit2 = true; }
        const bool cm2 = (fm2 >> lane) & 1u;
        if (cm2) bit_set(ev, lv);
        top.insert(cm2, key, v);
        c += __popc(fm2);
        __syncwarp();
        if (hit2) { stop = true; break; }    // the over-budget evaluation is not performed
        if (!im) break;                      // local maximum -> restart
        cur = __shfl_sync(FULL, v, fi);
        kcur = __shfl_sync(FULL, key, fi);
        curl = __shfl_sync(FULL, lv, fi);
        if (__shfl_sync(FULL, exb2, fi)) break;   // Q9: moving onto an expanded node restarts
      }
      if (stop) break;
    }
    s_evals += c;
    if (lane < a.kr) {
      const size_t o = ((size_t)b * Pn + p) * a.kr + lane;
      a.out_ids[o] = lane < top.cnt ? top.id : -1;
      a.out_keys[o] = lane < top.cnt ? top.key : 0u;
    }
    __syncwarp();
  }
  if (lane == 0) {
    atomicAdd(a.stats + 0, s_evals);
    atomicAdd(a.stats + 1, s_starts);
    atomicAdd(a.stats + 2, s_skip);
    atomicAdd(a.stats + 3, s_exp);
  }
}

// K2: keep the k_r best of the P*k_r per-partition candidates (Alg. 3 "Keep k most similar").
template <int M>
__global__ void k_merge_parts(const int32_t *ci, const uint32_t *ck, int64_t nq, int P, int kr,
                              int32_t *oi, uint32_t *ok) {
  const int lane = threadIdx.x & 31;
  const int64_t q = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (q >= nq) return;
  WarpTopK<M> top;
  top.init(kr);
  for (int p = 0; p < P; ++p) {
    const size_t o = ((size_t)q * P + p) * kr;
    const int32_t id = lane < kr ? ci[o + lane] : -1;
    const uint32_t key = lane < kr ? ck[o + lane] : 0u;
    top.insert(id >= 0, key, id);
  }
  if (lane < kr) {
    oi[(size_t)q * kr + lane] = lane < top.cnt ? top.id : -1;
    ok[(size_t)q * kr + lane] = lane < top.cnt ? top.key : 0u;
  }
}

// ---------------------------------------------------------------------------
template <int M, int L, int CPL>
static cudaError_t run_search(const SearchArgs &a0, cudaStream_t s) {
  SearchArgs a = a0;
  const int Pn = a.P > 0 ? a.P : 1;
  const int64_t T = a.nq * Pn;
  if (T == 0) return cudaSuccess;
  const int wpb = 4;
  size_t smem = 0;
  if (a.smem_bits) smem = (size_t)wpb * a.bits_words * 4;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_search<M, L, CPL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  int64_t blocks = (T + wpb - 1) / wpb;
  if (!a.smem_bits) {
    const int64_t cap = (int64_t)a.bits_words > 0 ? 148 * 16 : blocks;
    if (blocks > cap) blocks = cap;
  }
  k_search<M, L, CPL><<<(unsigned)blocks, wpb * 32, smem, s>>>(a);
  return cudaGetLastError();
}

#define KNNG_SHAPES(X, M) \
  X(M, 1, 1) X(M, 2, 1) X(M, 4, 1) X(M, 8, 1) X(M, 16, 1) X(M, 32, 1) X(M, 32, 2) X(M, 32, 4)

cudaError_t launch_search(const VecGeom &g, const SearchArgs &a, cudaStream_t s, int *n_launch) {
  if (n_launch) ++*n_launch;
#define X(MM, LL, CC) \
  if (g.metric == MM && g.L == LL && g.CPL == CC) return run_search<MM, LL, CC>(a, s);
  KNNG_SHAPES(X, M_U8)
  KNNG_SHAPES(X, M_F32)
#undef X
  return cudaErrorInvalidValue;
}

cudaError_t launch_merge_parts(int metric, const int32_t *ci, const uint32_t *ck, int64_t nq, int P, int kr,
                               int32_t *oi, uint32_t *ok, cudaStream_t s) {
  if (nq == 0) return cudaSuccess;
  const unsigned blocks = (unsigned)((nq + 3) / 4);
  if (metric == M_U8) k_merge_parts<M_U8><<<blocks, 128, 0, s>>>(ci, ck, nq, P, kr, oi, ok);
  else if (metric == M_F32) k_merge_parts<M_F32><<<blocks, 128, 0, s>>>(ci, ck, nq, P, kr, oi, ok);
  else k_merge_parts<M_JAC><<<blocks, 128, 0, s>>>(ci, ck, nq, P, kr, oi, ok);
  return cudaGetLastError();
}

}  // namespace knng
