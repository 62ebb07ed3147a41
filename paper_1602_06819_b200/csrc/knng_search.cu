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
#include <stdio.h>
#include <stdlib.h>

#include "knng_common.cuh"
#include "knng_internal.h"

namespace knng {

constexpr int RING_CHUNKS = 8;    // smem ring of 8 x 32 precomputed draws per CTA
constexpr int FASTC = 4;          // chunks the consumer's skip-only fast path commits at once

struct RingHdr {
  int seq[RING_CHUNKS];   // seq[s] = c + 1 once chunk c is in slot s
  int consumed;           // chunks < consumed are free
  int done;               // consumer finished the task
};

// Producer warp(s): speculative evaluation of the random starts.  The draw sequence of a search
// is fixed by the counter RNG (Q4) and the key of a draw is a pure function of (query, node), so
// producers evaluate draws ahead of the consumer, 32 per chunk, into the CTA's smem ring.
// Nothing here touches a counter, the visited sets or the top-k.
template <class QT>
__device__ __forceinline__ void produce(const SearchArgs &a, const QT &Q, volatile RingHdr *hdr,
                                        int2 *ring, int pw, int nprod, int64_t nch, uint64_t h3, int64_t m,
                                        const int32_t *pool) {
  const int lane = threadIdx.x & 31;
  long long p_wait = 0, p_work = 0;
  // chunks c and c + nprod are produced together (both sets of loads in flight)
  for (int64_t c = pw; c < nch; c += 2 * nprod) {
    const int64_t c2 = c + nprod;
    const bool two = c2 < nch;
    const int64_t clast = two ? c2 : c;
    const long long t0 = a.prof ? clock64() : 0;
    while (clast - hdr->consumed >= RING_CHUNKS && !hdr->done) __nanosleep(32);
    const long long t1 = a.prof ? clock64() : 0;
    p_wait += t1 - t0;
    if (hdr->done) break;
    const uint64_t ia = rng_index(h3, (uint64_t)(c * 32 + lane), (uint64_t)m);
    const int32_t na = pool ? pool[ia] : (int32_t)ia;
    int32_t nb = -1;
    if (two) {
      const uint64_t ib = rng_index(h3, (uint64_t)(c2 * 32 + lane), (uint64_t)m);
      nb = pool ? pool[ib] : (int32_t)ib;
    }
    uint32_t ka, kb;
    Q.eval2(a.st, na, nb, ka, kb);
    // repeats of a node inside a window are resolved by the consumer (the atomicOr that flips the
    // node's visited bit decides which draw evaluates it)
    volatile int *ra = (volatile int *)(ring + (c % RING_CHUNKS) * 32 + lane);
    ra[0] = na;
    ra[1] = (int)ka;
    if (two) {
      volatile int *rb = (volatile int *)(ring + (c2 % RING_CHUNKS) * 32 + lane);
      rb[0] = nb;
      rb[1] = (int)kb;
    }
    __threadfence_block();
    __syncwarp();
    if (lane == 0) {
      hdr->seq[c % RING_CHUNKS] = (int)(c + 1);
      if (two) hdr->seq[c2 % RING_CHUNKS] = (int)(c2 + 1);
    }
    if (a.prof) p_work += clock64() - t1;
  }
  if (a.prof && lane == 0) {
    atomicAdd(a.prof + 3, (unsigned long long)p_work);
    atomicAdd(a.prof + 4, (unsigned long long)p_wait);
  }
}

// K1: one CTA per (query, partition) task: warp 0 runs the search in the paper's sequential
// order, warps 1.. produce its random-start keys ahead of it.
template <int M, int L, int CPL>
__global__ void __launch_bounds__(64, 8) k_search(SearchArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  volatile RingHdr *hdr = (volatile RingHdr *)smem;
  int2 *ring = (int2 *)(smem + 128);
  int32_t *rowbuf = (int32_t *)(smem + 128 + RING_CHUNKS * 32 * 8);          // [k][k]
  int32_t *rowbuf2 = rowbuf + a.k * a.k;                                      // [32][k]
  uint32_t *qscr = (uint32_t *)(rowbuf2 + 32 * a.k);                          // [2][QMAX] (sets)
  uint32_t *sbits = qscr + (M == M_JAC ? 2 * QMAX : 0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nprod = (blockDim.x >> 5) - 1;
  const int Pn = a.part_cnt;
  const int64_t T = a.nq * Pn;
  uint32_t *bits = a.smem_bits ? sbits : a.gbits + (int64_t)blockIdx.x * a.bits_words;
  const int k = a.k;
  const float rk = 1.0f / (float)k;
  unsigned long long s_evals = 0, s_starts = 0, s_skip = 0, s_exp = 0;

  for (int64_t task = blockIdx.x; task < T; task += gridDim.x) {
    const int64_t b = task / Pn;
    const int pl = (int)(task % Pn);          // output slot
    const int p = a.part_lo + pl;             // partition searched
    const int64_t m = a.P > 0 ? a.member_cnt[p] : a.n_t;
    const int32_t *pool = a.P > 0 ? a.members + (size_t)p * a.member_cap : nullptr;
    const int64_t words = (m + 31) >> 5;
    uint32_t *ev = bits, *ex = bits + words;
    __syncthreads();
    for (int64_t w = threadIdx.x; w < 2 * words; w += blockDim.x) bits[w] = 0;
    if (threadIdx.x < RING_CHUNKS) hdr->seq[threadIdx.x] = 0;
    if (threadIdx.x == 0) { hdr->consumed = 0; hdr->done = 0; }
    __syncthreads();

    // budget (Q6) -- never more than the pool (Q7)
    int64_t budget = (int64_t)floor((double)m / a.speedup);
    const int64_t lo = m < a.kr ? m : a.kr;
    if (budget < lo) budget = lo;
    if (budget > m) budget = m;
    // chunks the producers may evaluate: they run until the consumer is done (redraws push the
    // consumed draws past the budget), capped for degenerate cases (speedup ~ 1)
    const int64_t nch = a.starts ? 0 : (8 * budget + 31) / 32 + 8;

    typename QuerySel<M, L, CPL>::T Q;
    Q.load(a.qs, a.qrow0 + b, M == M_JAC ? qscr + (warp < 2 ? warp : 1) * QMAX : nullptr);
    const uint64_t h3 = rng_prefix(a.seed, (uint64_t)(a.pid_base + b), (uint64_t)p);
    if (warp > 0) {
      if (budget > 0) {
        if (M == M_U8 && a.st.nchunks <= 8 && a.qs.nchunks <= 8) {
          // u8 rows of <= 128 B: 4 lanes x 2 chunks per candidate (2 shuffle levels), measured the
          // fastest layout for 32-draw chunks (scripts/micro/eval_micro.cu)
          VecQuery<M_U8, 4, 2> PQ;
          PQ.load(a.qs, a.qrow0 + b, nullptr);
          produce(a, PQ, hdr, ring, warp - 1, nprod, nch, h3, m, pool);
        } else {
          produce(a, Q, hdr, ring, warp - 1, nprod, nch, h3, m, pool);
        }
      }
      continue;
    }

    // ================================ consumer ================================
    WarpTopK<M> top;
    top.init(a.kr);
    int64_t c = 0, jbase = 0;
    int32_t wnode = -1;
    uint32_t wkey = 0, wl = 0;
    bool whave = false, wpf = false;
    SkipThr<M> thr;              // skip rule prepared against the current best key
    uint32_t thr_key = 0;
    bool thr_ok = false;
    int wpos = 32;

    const long long tc0 = a.prof ? clock64() : 0;
    long long p_wait = 0, p_walk = 0, p_win = 0;
    while (c < budget) {
      // ------------------------------ restart ------------------------------
      if (wpos >= 32) {
        // ---- fast path: FASTC whole produced chunks in which no draw can be accepted.  Against the
        // current s_max every draw is skipped (so none is a new best and the threshold cannot move);
        // each unevaluated node among them is evaluated once (the atomicOr that flips its bit) and
        // skipped, exactly as the sequential loop would do draw by draw; the budget is not reached.
        const int64_t ch0 = jbase / 32;
        if (top.cnt > 0 && nprod > 0 && ch0 + FASTC <= nch && c + 32 * FASTC <= budget) {
          const long long tw = a.prof ? clock64() : 0;
          for (int t = 0; t < FASTC; ++t) {
            const int slot = (int)((ch0 + t) % RING_CHUNKS);
            while (hdr->seq[slot] != (int)(ch0 + t + 1)) __nanosleep(20);
          }
          if (a.prof) p_wait += clock64() - tw;
          __threadfence_block();
          if (!thr_ok || thr_key != top.key_at0) {
            thr.set(top.key_at0, a.e_num, a.e_den);
            thr_key = top.key_at0;
            thr_ok = true;
          }
          int32_t fnode[FASTC];
          uint32_t fkey[FASTC];
          bool pass = false;
#pragma unroll
          for (int t = 0; t < FASTC; ++t) {
            const volatile int *rs = (const volatile int *)(ring + ((ch0 + t) % RING_CHUNKS) * 32 + lane);
            fnode[t] = rs[0];
            fkey[t] = (uint32_t)rs[1];
            pass |= !thr.skip(fkey[t]);
          }
          if (!__any_sync(FULL, pass)) {
            bool fr[FASTC];
#pragma unroll
            for (int t = 0; t < FASTC; ++t) {
              const uint32_t li = a.P > 0 ? (uint32_t)a.local_idx[fnode[t]] : (uint32_t)fnode[t];
              const uint32_t bit = 1u << (li & 31);
              fr[t] = !(atomicOr(ev + (li >> 5), bit) & bit);
            }
            __syncwarp();
            int nf = 0;
#pragma unroll
            for (int t = 0; t < FASTC; ++t) {
              top.insert(fr[t], fkey[t], fnode[t]);     // Q5: skipped starts enter the top-k
              nf += __popc(__ballot_sync(FULL, fr[t]));
            }
            c += nf;
            s_starts += nf;
            s_skip += nf;
            p_win += FASTC;
            __syncwarp();
            if (lane == 0) hdr->consumed = (int)(ch0 + FASTC);
            jbase += 32 * FASTC;
            continue;
          }
        }
        const int64_t j = jbase + lane;
        const int64_t ch = jbase / 32;
        if (ch < nch && nprod > 0) {                 // produced ahead into the ring
          const int slot = (int)(ch % RING_CHUNKS);
          const long long tw = a.prof ? clock64() : 0;
          while (hdr->seq[slot] != (int)(ch + 1)) __nanosleep(20);
          if (a.prof) p_wait += clock64() - tw;
          ++p_win;
          __threadfence_block();
          const volatile int *rs = (const volatile int *)(ring + slot * 32 + lane);
          wnode = rs[0];
          wkey = (uint32_t)rs[1];
          whave = true;
          __syncwarp();
          if (lane == 0) hdr->consumed = (int)(ch + 1);
        } else {
          if (a.starts) {
            wnode = j < a.nstarts ? a.starts[j] : -1;
          } else {
            const uint64_t idx = rng_index(h3, (uint64_t)j, (uint64_t)m);
            wnode = pool ? pool[idx] : (int32_t)idx;
          }
          whave = false;
        }
        wl = wnode >= 0 ? (a.P > 0 ? (uint32_t)a.local_idx[wnode] : (uint32_t)wnode) : 0u;
        jbase += 32;
        wpos = 0;
        // prefetch the rows of the draws that could still be accepted: the skip threshold only
        // tightens as s_max improves, so "passes against the current best" is a superset
        wpf = false;
        if (whave && wnode >= 0) {
          if (top.cnt > 0 && (!thr_ok || thr_key != top.key_at0)) {
            thr.set(top.key_at0, a.e_num, a.e_den);
            thr_key = top.key_at0;
            thr_ok = true;
          }
          wpf = top.cnt == 0 ? lane == 0 : !thr.skip(wkey);
          if (__ballot_sync(FULL, wpf)) {
            cp_async_wait_all();      // older copies into rowbuf2 must land first
            if (wpf)
              for (int e = 0; e < k; ++e) cp_async4(rowbuf2 + lane * k + e, a.rows + (size_t)wnode * k + e);
          }
        }
      }
      const unsigned active = FULL << wpos;
      const unsigned invm = __ballot_sync(FULL, wnode < 0) & active;
      const unsigned lim = invm ? ((1u << (__ffs(invm) - 1)) - 1u) : FULL;
      const bool evb = wnode >= 0 ? bit_get(ev, wl) : true;
      // Redraws of evaluated nodes are free (Q4).  A node drawn twice inside the window looks fresh
      // in both lanes: the later lane can never be accepted when the earlier one is skipped (same key,
      // tighter s_max), and the commit's atomicOr lets only the first evaluation count.
      const bool fresh = lane >= wpos && !evb;
      const unsigned fm = __ballot_sync(FULL, fresh) & active & lim;
      if (fm == 0) {
        if (invm) break;          // injected start sequence exhausted
        wpos = 32;
        continue;
      }
      // evaluate the next G fresh draws that have no key yet (beyond the produced range)
      unsigned hm = __ballot_sync(FULL, whave);
      const unsigned nokey = fm & ~hm;
      if (nokey) {
        const unsigned need = first_bits(nokey, a.G);
        const int nn = __popc(need);
        const int src = lane < nn ? (int)__fns(need, 0, lane + 1) : 0;
        const int32_t cid = __shfl_sync(FULL, wnode, src);
        const uint32_t kk = Q.eval(a.st, lane < nn ? cid : -1, nn);
        const int rank = __popc(need & lanemask_lt());
        const uint32_t mine = __shfl_sync(FULL, kk, rank & 31);
        if ((need >> lane) & 1u) { wkey = mine; whave = true; }
        hm |= need;
      }
      // committable: fresh draws in order up to the first one without a key
      const unsigned miss = fm & ~hm;
      const unsigned cmfull = miss ? (fm & ((1u << (__ffs(miss) - 1)) - 1u)) : fm;
      unsigned cm = cmfull;
      if ((int64_t)__popc(cm) > budget - c) cm = first_bits(cm, (int)(budget - c));
      const bool inc = (cm >> lane) & 1u;
      unsigned am;
      if (top.cnt > 0 && (!thr_ok || thr_key != top.key_at0)) {
        thr.set(top.key_at0, a.e_num, a.e_den);
        thr_key = top.key_at0;
        thr_ok = true;
      }
      if (top.cnt > 0 && __ballot_sync(FULL, inc && !thr.skip(wkey)) == 0) {
        am = 0;   // every committable draw is skipped even against the current s_max
      } else {
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
      am = __ballot_sync(FULL, acc);
      }
      const int al = am ? __ffs(am) - 1 : -1;
      const unsigned commit = am ? (cm & (al == 31 ? FULL : ((2u << al) - 1u))) : cm;
      const bool cmt = (commit >> lane) & 1u;
      bool newly = false;
      if (cmt) {
        const uint32_t bit = 1u << (wl & 31);
        newly = !(atomicOr(ev + (wl >> 5), bit) & bit);
      }
      top.insert(newly, wkey, wnode);        // Q5: skipped starts enter the top-k too
      const int ncm = __popc(__ballot_sync(FULL, newly));
      c += ncm;
      s_starts += ncm;
      s_skip += ncm - (am ? 1 : 0);
      __syncwarp();
      // budget reached: stop, unless a start was accepted -- then, as in the sequential
      // algorithm, its walk begins and ends at the first fresh evaluation it needs
      if (c >= budget && !am) break;
      if (!am) {
        const unsigned rest = cmfull & ~commit;   // truncated by the budget (repeats inside): resume there
        wpos = rest ? (__ffs(rest) - 1) : (miss ? (__ffs(miss) - 1) : 32);
        continue;
      }
      wpos = al + 1;

      // ------------------- hill climbing, eager first improvement -------------------
      const long long tk0 = a.prof ? clock64() : 0;
      int32_t cur = __shfl_sync(FULL, wnode, al);
      uint32_t kcur = __shfl_sync(FULL, wkey, al);
      uint32_t curl = __shfl_sync(FULL, wl, al);
      int pf = -1;                 // row of cur prefetched into rowbuf[pf*k ..] by the last step
      int pf2 = al;                // ... or into rowbuf2[pf2*k ..] when the window was loaded
      if (!__shfl_sync(FULL, wpf, al)) pf2 = -1;
      bool stop = false;
      for (;;) {
        if (lane == 0) bit_set(ex, curl);
        ++s_exp;
        int32_t v = -1;
        if (pf >= 0 || pf2 >= 0) {
          cp_async_wait_all();
          __syncwarp();
        }
        if (lane < k)
          v = pf >= 0 ? rowbuf[pf * k + lane] : (pf2 >= 0 ? rowbuf2[pf2 * k + lane] : a.rows[(size_t)cur * k + lane]);
        pf2 = -1;
        const bool inpool = v >= 0 && (a.P == 0 || a.part_of[v] == p);   // Q10
        const uint32_t lv = inpool ? (a.P > 0 ? (uint32_t)a.local_idx[v] : (uint32_t)v) : 0u;
        __syncwarp();
        // prefetch the rows of the in-pool neighbours: the next cur is one of them
        for (int base = 0; base < k * k; base += 32) {
          const int idx = base + lane;
          const int t = __float2int_rz(__fmul_rn(__int2float_rn(idx) + 0.5f, rk));   // idx / k
          const int32_t vt = __shfl_sync(FULL, inpool ? v : -1, t < 32 ? t : 31);
          if (idx < k * k && vt >= 0) cp_async4(rowbuf + idx, a.rows + (size_t)vt * k + (idx - t * k));
        }
        const bool evb2 = inpool ? bit_get(ev, lv) : true;
        const bool exb2 = inpool ? bit_get(ex, lv) : false;
        const uint32_t key = Q.eval(a.st, inpool ? v : -1, k);
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
        pf = fi;
        if (__shfl_sync(FULL, exb2, fi)) break;   // Q9: moving onto an expanded node restarts
      }
      if (a.prof) p_walk += clock64() - tk0;
      if (stop) break;
    }
    if (a.prof && lane == 0) {
      atomicAdd(a.prof + 0, (unsigned long long)(clock64() - tc0));
      atomicAdd(a.prof + 1, (unsigned long long)p_wait);
      atomicAdd(a.prof + 2, (unsigned long long)p_walk);
      atomicAdd(a.prof + 5, (unsigned long long)p_win);
    }
    if (lane == 0) hdr->done = 1;
    s_evals += c;
    if (lane < a.kr) {
      const size_t o = ((size_t)b * Pn + pl) * a.kr + lane;
      a.out_ids[o] = lane < top.cnt ? top.id : -1;
      a.out_keys[o] = lane < top.cnt ? top.key : 0u;
    }
    __syncwarp();
  }
  if (lane == 0 && warp == 0) {
    atomicAdd(a.stats + 0, s_evals);
    atomicAdd(a.stats + 1, s_starts);
    atomicAdd(a.stats + 2, s_skip);
    atomicAdd(a.stats + 3, s_exp);
  }
}

// K2: keep the k_r best of the P*k_r per-partition candidates (Alg. 3 "Keep k most similar",
// P:176).  Input is rank-major [world][nq][P/world][kr] (world = 1: [nq][P][kr]), the layout an
// all-gather of the per-rank candidate buffers produces.
template <int M>
__global__ void k_merge_parts(const int32_t *ci, const uint32_t *ck, int64_t nq, int P, int world, int kr,
                              int32_t *oi, uint32_t *ok) {
  const int lane = threadIdx.x & 31;
  const int64_t q = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (q >= nq) return;
  const int Pown = P / world;
  WarpTopK<M> top;
  top.init(kr);
  for (int p = 0; p < P; ++p) {
    const int r = p / Pown, j = p % Pown;
    const size_t o = (((size_t)r * nq + q) * Pown + j) * kr;
    const int32_t id = lane < kr ? ci[o + lane] : -1;
    const uint32_t key = lane < kr ? ck[o + lane] : 0u;
    top.insert(id >= 0, key, id);
  }
  if (lane < kr) {
    oi[(size_t)q * kr + lane] = lane < top.cnt ? top.id : -1;
    ok[(size_t)q * kr + lane] = lane < top.cnt ? top.key : 0u;
  }
}

template <int M, int L, int CPL>
static cudaError_t run_search(const SearchArgs &a, cudaStream_t s) {
  const int Pn = a.part_cnt;
  const int64_t T = a.nq * Pn;
  if (T == 0) return cudaSuccess;
  // consumer + producer (a second producer did not pay: measured on C2/C3)
  const int warps = a.starts ? 1 : 2;
  size_t smem = 128 + RING_CHUNKS * 32 * 8 + (size_t)(a.k * a.k + 32 * a.k) * 4 + (M == M_JAC ? 2 * QMAX * 4 : 0);
  if (a.smem_bits) smem += (size_t)a.bits_words * 4;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_search<M, L, CPL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  int64_t blocks = T;
  if (!a.smem_bits && blocks > a.gslots) blocks = a.gslots;
  if (getenv("KNNG_PROFILE")) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_search<M, L, CPL>, warps * 32, smem);
    fprintf(stderr, "KNNG_PROFILE k_search: %lld CTAs, %d per SM resident (%zu B smem each)\n", (long long)blocks,
            per_sm, smem);
  }
  k_search<M, L, CPL><<<(unsigned)blocks, warps * 32, smem, s>>>(a);
  return cudaGetLastError();
}

#define KNNG_SHAPES(X, M) \
  X(M, 1, 1) X(M, 2, 1) X(M, 4, 1) X(M, 8, 1) X(M, 16, 1) X(M, 32, 1) X(M, 32, 2) X(M, 32, 4)
// fp32 rows of <= 32 chunks: 4 chunks per lane at most, partials in-lane (see VecQuery::reduce)
#define KNNG_SHAPES_F32(X) \
  X(M_F32, 1, 1) X(M_F32, 1, 2) X(M_F32, 1, 3) X(M_F32, 1, 4) X(M_F32, 2, 3) X(M_F32, 2, 4) X(M_F32, 4, 3) \
  X(M_F32, 4, 4) X(M_F32, 8, 3) X(M_F32, 8, 4) X(M_F32, 32, 2) X(M_F32, 32, 4)

cudaError_t launch_search(const VecGeom &g, const SearchArgs &a, cudaStream_t s, int *n_launch) {
  if (n_launch) ++*n_launch;
#define X(MM, LL, CC) \
  if (g.metric == MM && g.L == LL && g.CPL == CC) return run_search<MM, LL, CC>(a, s);
  KNNG_SHAPES(X, M_U8)
  KNNG_SHAPES_F32(X)
  X(M_JAC, 8, 1)
#undef X
  return cudaErrorInvalidValue;
}

cudaError_t launch_merge_parts(int metric, const int32_t *ci, const uint32_t *ck, int64_t nq, int P, int world, int kr,
                               int32_t *oi, uint32_t *ok, cudaStream_t s) {
  if (nq == 0) return cudaSuccess;
  const unsigned blocks = (unsigned)((nq + 3) / 4);
  if (metric == M_U8) k_merge_parts<M_U8><<<blocks, 128, 0, s>>>(ci, ck, nq, P, world, kr, oi, ok);
  else if (metric == M_F32) k_merge_parts<M_F32><<<blocks, 128, 0, s>>>(ci, ck, nq, P, world, kr, oi, ok);
  else k_merge_parts<M_JAC><<<blocks, 128, 0, s>>>(ci, ck, nq, P, world, kr, oi, ok);
  return cudaGetLastError();
}

}  // namespace knng
