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

// Cycle counters of KNNG_PROFILE=1 exist only in builds with -DKNNG_PROFILE_COUNTERS (their state
// costs the consumer registers): KP(p) is false at compile time otherwise.
#ifdef KNNG_PROFILE_COUNTERS
#define KP(p) ((p) != nullptr)
#else
#define KP(p) false
#endif

namespace knng {

constexpr int FASTC = 2;          // chunks the consumer's skip-only fast path commits at once (<= ring)
constexpr int HDR_BYTES = 128;

struct RingHdr {
  int consumed;           // chunks < consumed are free
  int done;               // consumer finished the task
  int next_task;          // dynamic task scheduler: the CTA's next task
  int published;          // debug: last chunk a producer published
  int pstate;             // debug: producer state
};

// Producer warp(s): speculative evaluation of the random starts.  The draw sequence of a search
// is fixed by the counter RNG (Q4) and the key of a draw is a pure function of (query, node), so
// producers evaluate draws ahead of the consumer, 32 per chunk, into the CTA's smem ring.
// Nothing here touches a counter, the visited sets or the top-k.
//
// The rows of the drawn nodes are gathered into shared memory with 16-byte cp.async copies
// (no registers held by loads in flight), S chunks deep; the keys are computed from shared
// memory.  Producer pw owns chunks pw, pw + nprod, ...; local iteration i <-> chunk pw + i*nprod.
struct ProdCtx {
  volatile RingHdr *hdr;
  unsigned long long *ring;   // [ring][32][2]: (tag << 32 | node), (tag << 32 | key), tag = chunk + 1
  int ring_n;                 // ring chunks (power of 2)
  uint8_t *stg;       // this producer's S x 32 rows (pitch bytes each)
  int32_t *meta;      // this producer's S x 32 x 4 ints (node, rb, re, -)
  int pitch;
  int pw, nprod;
  int64_t nch;
  uint64_t h3;
  int64_t m;
  const int32_t *pool;
};

// draw i of this lane: (node id, pool index).  The pool index is the node's partition-local index
// (members_p is ascending in local index), which is what the ring carries: the consumer's visited
// bitmap needs it, and the node id only when the draw may enter the top-k or start a walk.
__device__ __forceinline__ int2 draw_node(const ProdCtx &x, int64_t i) {
  const int64_t c = x.pw + i * x.nprod;
  const uint64_t idx = rng_index(x.h3, (uint64_t)(c * 32 + (threadIdx.x & 31)), (uint64_t)x.m);
  return make_int2(x.pool ? x.pool[idx] : (int32_t)idx, (int32_t)idx);
}

// publish chunk (local iteration i) to the ring; false when the consumer has finished
__device__ __forceinline__ bool publish(const ProdCtx &x, int64_t i, int32_t node, uint32_t key, long long &p_wait,
                                        bool prof) {
  const int lane = threadIdx.x & 31;
  const int64_t c = x.pw + i * x.nprod;
  const long long t0 = prof ? clock64() : 0;
  int dn = 0;
  if (lane == 0)
    while (c - x.hdr->consumed >= x.ring_n && !(dn = x.hdr->done)) __nanosleep(32);
  dn = __shfl_sync(FULL, dn, 0);
  if (prof) p_wait += clock64() - t0;
  if (dn) return false;
  // Each entry word carries its chunk's tag next to the datum: an aligned 64-bit shared store is
  // single-copy atomic, so the consumer sees a whole (tag, datum) pair and needs no fence or barrier.
  const unsigned long long tag = (unsigned long long)(unsigned)(c + 1) << 32;
  volatile unsigned long long *e = x.ring + ((c & (x.ring_n - 1)) * 32 + lane) * 2;
  e[0] = tag | (uint32_t)node;
  e[1] = tag | key;
#ifdef KNNG_DEBUG_WAIT
  if (lane == 0) x.hdr->published = (int)c;
#endif
  return true;
}

// consumer: wait until chunk ch is in its slot and read this lane's (node, key)
__device__ __forceinline__ void ring_get(const unsigned long long *ring, int ring_n, volatile RingHdr *hdr, int64_t ch,
                                         int32_t &node, uint32_t &key) {
  const unsigned tag = (unsigned)(ch + 1);
  const volatile unsigned long long *e = ring + ((ch & (ring_n - 1)) * 32 + (threadIdx.x & 31)) * 2;
  unsigned long long w0, w1;
#ifdef KNNG_DEBUG_WAIT
  long long n = 0;
#endif
  for (;;) {
    w0 = e[0];
    w1 = e[1];
    if (__all_sync(FULL, (unsigned)(w0 >> 32) == tag && (unsigned)(w1 >> 32) == tag)) break;
#ifdef KNNG_DEBUG_WAIT
    if (++n == (1ll << 22) && (threadIdx.x & 31) == 0)
      printf("KNNG stuck wait: block %d chunk %lld consumed %d done %d published %d pstate %d\n", blockIdx.x,
             (long long)ch, hdr->consumed, hdr->done, hdr->published, hdr->pstate);
#endif
    __nanosleep(16);
  }
  node = (int32_t)(uint32_t)w0;
  key = (uint32_t)w1;
}

// Expanded set of the consumer warp (warp-uniform state): a shared open-addressing hash of
// pool-local ids (+1; 0 = empty), filled to 3/4 at most; beyond that the global bitmap gex takes
// the further entries (zeroed by the warp when first needed) and lookups consult both.
constexpr int EXCAP = 512;
__device__ __forceinline__ bool ex_has(const int32_t *exh, bool ovf, const uint32_t *gex, uint32_t lv) {
  uint32_t h = (lv * 0x9E3779B1u) >> (32 - 9);
  for (;;) {
    const int32_t e = exh[h];
    if (e == 0) break;
    if (e == (int32_t)(lv + 1)) return true;
    h = (h + 1) & (EXCAP - 1);
  }
  return ovf ? bit_get(gex, lv) : false;
}
__device__ __forceinline__ void ex_insert(int32_t *exh, int &cnt, bool &ovf, uint32_t *gex, int64_t words, uint32_t lv) {
  const int lane = threadIdx.x & 31;
  if (!ovf && cnt >= EXCAP * 3 / 4) {
    for (int64_t w = lane; w < words; w += 32) gex[w] = 0;
    __threadfence_block();
    __syncwarp();      // every lane's zeroing lands before lane 0 sets the first bit
    ovf = true;
  }
  if (ovf) {
    if (lane == 0) bit_set(gex, lv);
  } else {
    if (lane == 0) {
      uint32_t h = (lv * 0x9E3779B1u) >> (32 - 9);
      while (exh[h] != 0 && exh[h] != (int32_t)(lv + 1)) h = (h + 1) & (EXCAP - 1);
      exh[h] = (int32_t)(lv + 1);
    }
    ++cnt;
  }
  __syncwarp();
}

__device__ __forceinline__ bool consumer_done(const ProdCtx &x) {
  int dn = (threadIdx.x & 31) == 0 ? x.hdr->done : 0;
  return __shfl_sync(FULL, dn, 0) != 0;
}

// Evaluators of a staged chunk (32 rows at stage + j * pitch): key of candidate j in lane j.
// Warp form: L lanes per row (VecQuery::eval_smem).
template <class QT>
struct EvalWarp {
  static constexpr int NCH = 0;   // chunks per row known at run time only
  const QT &Q;
  __device__ __forceinline__ uint32_t key(const uint8_t *sb, int pitch, int nck) const {
    return Q.eval_smem(sb, pitch, nck);
  }
};
// Lane form: one lane per row, the whole distance in-lane (no shuffles; NCH independent chunk
// chains), the query's chunks broadcast from shared memory.  F32 keeps the canonical tree (Q24):
// with NCH <= 32 partial i is chunk i alone (f4_leaf from +0), partials >= NCH are +0, and the
// levels o = 16..1 add partial i + o into partial i -- the xor butterfly's values.
template <int M, int NCH_>
struct EvalLane {
  static constexpr int NCH = NCH_;
  const uint8_t *qsm;   // the query's NCH chunks (shared)
  __device__ __forceinline__ uint32_t key(const uint8_t *sb, int pitch, int) const {
    const uint8_t *row = sb + (threadIdx.x & 31) * pitch;
    if (M == M_U8) {   // exact integer sum: four independent accumulators (short dependency chains)
      uint32_t acc[4] = {0, 0, 0, 0};
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        const uint4 q = *(const uint4 *)(qsm + 16 * c), r = *(const uint4 *)(row + 16 * c);
        uint32_t d;
        d = __vabsdiffu4(q.x, r.x); acc[0] = __dp4a(d, d, acc[0]);
        d = __vabsdiffu4(q.y, r.y); acc[1] = __dp4a(d, d, acc[1]);
        d = __vabsdiffu4(q.z, r.z); acc[2] = __dp4a(d, d, acc[2]);
        d = __vabsdiffu4(q.w, r.w); acc[3] = __dp4a(d, d, acc[3]);
      }
      return (acc[0] + acc[1]) + (acc[2] + acc[3]);
    } else {
      static_assert(NCH <= 32, "lane form: one chunk per partial");
      float p[32];
#pragma unroll
      for (int i = 0; i < 32; ++i)
        p[i] = i < NCH ? f4_leaf(0.0f, *(const uint4 *)(qsm + 16 * i), *(const uint4 *)(row + 16 * i)) : 0.0f;
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1)
#pragma unroll
        for (int i = 0; i < o; ++i) p[i] = __fadd_rn(p[i], p[i + o]);
      return __float_as_uint(p[0]);
    }
  }
};

// vectors: lane's copies within a stage are the 16-byte chunks e = lane + 32 j (j < nchunks) of the
// 32 x nchunks stage, i.e. row e / nchunks, chunk e % nchunks (walked incrementally).
// S single-chunk stages in a ring: chunks i+1 .. i+S-1 are in flight while chunk i is evaluated.
template <int S, class EV>
__device__ __forceinline__ void produce_vec(const SearchArgs &a, const EV &ev, const ProdCtx &x) {
  const int lane = threadIdx.x & 31;
  const int nck = EV::NCH > 0 ? EV::NCH : a.st.nchunks;
  const uint8_t *base = a.st.vec;
  const size_t stride = a.st.stride;
  const int r0 = lane / nck, c0 = lane % nck, rs = 32 / nck, cs = 32 % nck;
  const int64_t ni = x.nch > x.pw ? (x.nch - x.pw + x.nprod - 1) / x.nprod : 0;
  const bool prof = KP(a.prof);
  long long p_wait = 0, p_work = 0;
  // compile-time widths: LR lanes per row, each copying chunks sl, sl + LR, ... of its row (immediate
  // offsets), 32 / LR rows per pass -- one shuffle and NCH / LR copies per pass
  constexpr int LR = EV::NCH >= 8 && EV::NCH % 8 == 0 ? 8 : (EV::NCH > 0 && EV::NCH <= 8 ? EV::NCH : 0);
  auto issue = [&](int st, int2 d) {
    x.meta[(st * 32 + lane) * 4] = d.y;   // published: the pool index
    uint8_t *dst = x.stg + st * 32 * x.pitch;
    if constexpr (LR > 0 && (32 % LR) == 0) {
      constexpr int RPP = 32 / LR, CPR = EV::NCH / LR;
      const int sl = lane % LR, rr = lane / LR;
#pragma unroll
      for (int p = 0; p < LR; ++p) {
        const int r = p * RPP + rr;
        const int32_t id = __shfl_sync(FULL, d.x, r);
        const uint8_t *src = base + (size_t)id * stride + sl * 16;
        uint8_t *drow = dst + r * x.pitch + sl * 16;
#pragma unroll
        for (int t = 0; t < CPR; ++t) cp_async16(drow + t * LR * 16, src + t * LR * 16);
      }
    } else {
      int r = r0, cc = c0;
#pragma unroll 8
      for (int j = 0; j < nck; ++j) {
        const int32_t id = __shfl_sync(FULL, d.x, r);
        cp_async16(dst + r * x.pitch + cc * 16, base + (size_t)id * stride + (size_t)cc * 16);
        cc += cs;
        r += rs;
        if (cc >= nck) { cc -= nck; ++r; }
      }
    }
  };
#pragma unroll
  for (int s = 0; s < S - 1; ++s) {
    if (s < ni) issue(s, draw_node(x, s));
    cp_async_commit();
  }
  int2 pn = S - 1 < ni ? draw_node(x, S - 1) : make_int2(0, 0);
  for (int64_t i = 0; i < ni; ++i) {
    const long long t0 = prof ? clock64() : 0;
    if (consumer_done(x)) break;
    const int64_t ii = i + S - 1;
    if (ii < ni) {
      issue((int)(ii % S), pn);
      if (ii + 1 < ni) pn = draw_node(x, ii + 1);   // (pool load) in flight during this evaluation
    }
    cp_async_commit();
    cp_async_wait<S - 1>();
    __syncwarp();
    const int st = (int)(i % S);
    const uint32_t key = ev.key(x.stg + st * 32 * x.pitch, x.pitch, nck);
    const int32_t node = x.meta[(st * 32 + lane) * 4];
    __syncwarp();
    if (prof) p_work += clock64() - t0;
    if (!publish(x, i, node, key, p_wait, prof)) break;
  }
  cp_async_wait<0>();
  __syncwarp();
  if (prof && lane == 0) {
    atomicAdd(a.prof + 3, (unsigned long long)p_work);
    atomicAdd(a.prof + 4, (unsigned long long)p_wait);
  }
}

// two stages measured fastest on every config (deeper pipelines cost CTAs per SM): the only one built
template <class EV>
__device__ __forceinline__ void produce_vec_s(const SearchArgs &a, const EV &ev, const ProdCtx &x) {
  produce_vec<2>(a, ev, x);
}

// the producer's evaluator: lane form for the configured row widths, else the warp form
template <int M, int L, int CPL>
__device__ __forceinline__ void produce_rows(const SearchArgs &a, const VecQuery<M, L, CPL> &Q, const ProdCtx &x,
                                             uint8_t *qsm, int64_t qrow) {
  const int lane = threadIdx.x & 31;
  const int nck = a.st.nchunks;
  const bool lane_form = a.lane_eval && ((M == M_U8 && (nck == 8 || nck == 2)) || (M == M_F32 && nck == 24));
  if (lane_form) {
    const uint8_t *qg = a.qs.vec + (size_t)qrow * a.qs.stride;
    for (int c = lane; c < nck; c += 32) *(uint4 *)(qsm + 16 * c) = ldg16(qg + 16 * c);
    __syncwarp();
    if constexpr (M == M_U8) {
      if (nck == 8) produce_vec_s(a, EvalLane<M_U8, 8>{qsm}, x);
      else produce_vec_s(a, EvalLane<M_U8, 2>{qsm}, x);
    } else if constexpr (M == M_F32) {
      produce_vec_s(a, EvalLane<M_F32, 24>{qsm}, x);
    }
    return;
  }
  if (M == M_U8 && nck <= 8 && a.qs.nchunks <= 8) {
    // u8 rows of <= 128 B: 4 lanes x 2 chunks per candidate (2 shuffle levels)
    VecQuery<M_U8, 4, 2> PQ;
    PQ.load(a.qs, qrow, nullptr);
    produce_vec_s(a, EvalWarp<VecQuery<M_U8, 4, 2>>{PQ}, x);
  } else {
    produce_vec_s(a, EvalWarp<VecQuery<M, L, CPL>>{Q}, x);
  }
}

// sets: lane j stages candidate j's token range (aligned 16-byte chunks, SLOTCH at most) in its own
// slot; longer sets are evaluated from global memory.  Two prefetch levels: the node of chunk
// i + S and the offsets of chunk i + S - 1 are loaded while chunk i is computed.
template <int S, int L>
__device__ __forceinline__ void produce_set(const SearchArgs &a, const SetQuery<L> &Q, const ProdCtx &x) {
  constexpr int SLOTCH = SetQuery<L>::SLOTCH;
  const int lane = threadIdx.x & 31;
  const uint32_t *tok = a.st.tok;
  const uint64_t *off = a.st.off;
  const int64_t ni = x.nch > x.pw ? (x.nch - x.pw + x.nprod - 1) / x.nprod : 0;
  const bool prof = KP(a.prof);
  long long p_wait = 0, p_work = 0;
  auto issue = [&](int st, int2 d, uint64_t b, uint64_t e) {
    const uint64_t a0 = b & ~3ull;
    const int rb = (int)(b - a0), re = (int)(e - a0);
    int4 *mt = (int4 *)(x.meta + (st * 32 + lane) * 4);
    *mt = make_int4(d.x, rb, re, d.y);
    const int nch = (re + 3) >> 2;
    if (nch <= SLOTCH) {
      uint8_t *dst = x.stg + (st * 32 + lane) * x.pitch;
      for (int j = 0; j < nch; ++j) cp_async16(dst + 16 * j, tok + a0 + 4 * j);
    }
  };
  // prologue
  int2 n1 = make_int2(0, 0);
  uint64_t b1 = 0, e1 = 0;
#pragma unroll
  for (int s = 0; s < S - 1; ++s) {
    if (s < ni) {
      const int2 nd = draw_node(x, s);
      issue(s, nd, off[nd.x], off[nd.x + 1]);
    }
    cp_async_commit();
  }
  if (S - 1 < ni) {
    n1 = draw_node(x, S - 1);
    b1 = off[n1.x];
    e1 = off[n1.x + 1];
  }
  int2 n2 = S < ni ? draw_node(x, S) : make_int2(0, 0);
  for (int64_t i = 0; i < ni; ++i) {
    const long long t0 = prof ? clock64() : 0;
    if (consumer_done(x)) break;
    const int64_t ii = i + S - 1;
    if (ii < ni) {
      issue((int)(ii % S), n1, b1, e1);
      if (ii + 1 < ni) {
        n1 = n2;
        b1 = off[n1.x];
        e1 = off[n1.x + 1];
        if (ii + 2 < ni) n2 = draw_node(x, ii + 2);
      }
    }
    cp_async_commit();
    cp_async_wait<S - 1>();
    __syncwarp();
    const int st = (int)(i % S);
    const int4 mt = *(const int4 *)(x.meta + (st * 32 + lane) * 4);
    uint32_t key;
    if (((mt.z + 3) >> 2) <= SLOTCH) {
      key = Q.eval_slot(x.stg + (st * 32 + lane) * x.pitch, mt.y, mt.z);
    } else {   // long set: straight from global memory
      const uint64_t b = off[mt.x];
      key = Q.eval_slot_global(tok + (b & ~3ull), mt.y, mt.z);
    }
    __syncwarp();
    if (prof) p_work += clock64() - t0;
    if (!publish(x, i, mt.w, key, p_wait, prof)) break;
  }
  cp_async_wait<0>();
  __syncwarp();
  if (prof && lane == 0) {
    atomicAdd(a.prof + 3, (unsigned long long)p_work);
    atomicAdd(a.prof + 4, (unsigned long long)p_wait);
  }
}

template <class QT>
__device__ __forceinline__ void set_bitmap(QT &, const uint32_t *) {}
template <int L>
__device__ __forceinline__ void set_bitmap(SetQuery<L> &Q, const uint32_t *bm) { Q.bm = bm; }
template <class QT>
__device__ __forceinline__ int query_len(const QT &) { return 0; }
template <int L>
__device__ __forceinline__ int query_len(const SetQuery<L> &Q) { return Q.qn; }
template <int M, int L, int CPL>
__device__ __forceinline__ void produce_any(const SearchArgs &a, const VecQuery<M, L, CPL> &Q, const ProdCtx &x,
                                            uint8_t *qsm, int64_t qrow) {
  produce_rows(a, Q, x, qsm, qrow);
}
template <int L>
__device__ __forceinline__ void produce_any(const SearchArgs &a, const SetQuery<L> &Q, const ProdCtx &x, uint8_t *,
                                            int64_t) {
  produce_set<2>(a, Q, x);
}

// K1: one CTA per (query, partition) task: warp 0 runs the search in the paper's sequential
// order, warps 1.. produce its random-start keys ahead of it.
// MB: launch-bound variant.  MB = 4 lets a CTA of up to 4 warps keep 128 registers per thread (8
// two-warp CTAs per SM); MB = 12 caps a two-warp CTA at 80 registers (12 per SM, some spills) for
// latency-bound task mixes that want more concurrent walks.
template <int M, int L, int CPL, int MB>
__global__ void __launch_bounds__(MB == 4 ? 128 : 64, MB) k_search(SearchArgs a) {   // MB 4: <= 128 regs; 10: <= 96
  extern __shared__ __align__(16) uint8_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nprod = (blockDim.x >> 5) - 1;
  const int k = a.k;
  volatile RingHdr *hdr = (volatile RingHdr *)smem;
  unsigned long long *ring = (unsigned long long *)(smem + HDR_BYTES);
  const int S = a.stages;
  uint8_t *stg = smem + HDR_BYTES + a.ring * 32 * 16;                         // [nprod][S][32] rows
  int32_t *meta = (int32_t *)(stg + (size_t)nprod * S * 32 * a.pitch);        // [nprod][S][32][4]
  uint8_t *qprod = (uint8_t *)(meta + nprod * S * 32 * 4);                   // [nprod][512 B] query copies
  int32_t *rowbuf = (int32_t *)(qprod + nprod * 512);                         // [k][k]
  int32_t *rowbuf2 = rowbuf + k * k;                                          // [32][k]
  // partitioned: the same rows' partition-local indices (lrows, -1 = other partition)
  const int lk = a.P > 0 ? k : 0;
  int32_t *lrowbuf = rowbuf2 + 32 * k;                                        // [k][k] (P > 0)
  int32_t *lrowbuf2 = lrowbuf + lk * k;                                       // [32][k] (P > 0)
  uint32_t *qscr = (uint32_t *)(lrowbuf2 + 32 * lk);                          // [2][QMAX] (sets)
  uint32_t *vbm = qscr + (M == M_JAC ? 2 * QMAX : 0);                        // [vwords] (sets)
  const int vwords = M == M_JAC ? a.st.vwords : 0;
  const uint32_t vw_lim = (uint32_t)a.st.vwords;   // (bounds for the Jaccard vocabulary bitmap)
  int32_t *exh = (int32_t *)(vbm + vwords);                                  // [EXCAP] expanded-set hash
  uint32_t *sbits = (uint32_t *)(exh + EXCAP);                               // [bits_words / 2] (smem bits)
  const int Pn = a.part_cnt;
  const int64_t T = a.nq * Pn;
  // per CTA slot in global memory: [evaluated words][expanded-overflow words]
  uint32_t *gslot = a.gbits + (int64_t)blockIdx.x * a.bits_words;
  const float rk = 1.0f / (float)k;
  unsigned long long s_evals = 0, s_starts = 0, s_skip = 0, s_exp = 0;
  int prev_qn = 0;                              // sets: tokens of the previous query (scratch 0)
  for (int w = threadIdx.x; w < vwords; w += blockDim.x) vbm[w] = 0;
  if (threadIdx.x == 0) hdr->next_task = (int)blockIdx.x;

  for (;;) {
    __syncthreads();                          // previous task finished by every warp
    const int64_t task = hdr->next_task;
    if (task >= T) break;
    const int64_t b = task / Pn;
    const int pl = (int)(task % Pn);          // output slot
    const int p = a.part_lo + pl;             // partition searched
    const int64_t m = a.P > 0 ? a.member_cnt[p] : a.n_t;
    const int32_t *pool = a.P > 0 ? a.members + (size_t)p * a.member_cap : nullptr;
    const int64_t words = (m + 31) >> 5;
    // evaluated set: bitmap over the pool (shared memory when it fits the plan, else L2/HBM);
    // expanded set: shared hash, overflowing into a global bitmap (cleared when first used)
    uint32_t *ev = a.smem_bits ? sbits : gslot;
    uint32_t *gex = gslot + words;
    for (int64_t w = threadIdx.x; w < words; w += blockDim.x) ev[w] = 0;
    for (int w = threadIdx.x; w < EXCAP; w += blockDim.x) exh[w] = 0;
    for (int w = threadIdx.x; w < a.ring * 32; w += blockDim.x)   // no stale tags from the last task
      ((uint4 *)ring)[w] = make_uint4(0, 0, 0, 0);
    if (threadIdx.x == 0) { hdr->consumed = 0; hdr->done = 0; }
    if (M == M_JAC && vwords > 0 && warp == 0)   // clear the previous query's vocabulary bits
      for (int i = lane; i < prev_qn; i += 32) {
        const uint32_t t = qscr[i];
        if ((t >> 5) < vw_lim) vbm[t >> 5] = 0;
      }
    __syncthreads();
    // dynamic task scheduling: the CTA's next task (read after the next top barrier)
    if (threadIdx.x == 0) hdr->next_task = (int)(gridDim.x + atomicAdd(a.task_ctr, 1ull));

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
    if (M == M_JAC && vwords > 0) {
      // vocabulary bitmap of the query: one bit test per candidate token (tokens beyond the store's
      // largest token cannot match and are left out)
      const int qn = query_len(Q);
      if (warp == 0 && qn <= QMAX) {
        for (int i = lane; i < qn; i += 32) {
          const uint32_t t = qscr[i];
          if ((t >> 5) < vw_lim) atomicOr(vbm + (t >> 5), 1u << (t & 31));
        }
        prev_qn = qn;
      } else if (warp == 0) {
        prev_qn = 0;
      }
      __syncthreads();
      if (qn <= QMAX) set_bitmap(Q, vbm);
    }
    const uint64_t h3 = rng_prefix(a.seed, (uint64_t)(a.pid_base + b), (uint64_t)p);
    if (warp > 0) {
      if (budget > 0 && nch > 0) {
        ProdCtx x;
        x.hdr = hdr;
        x.ring = ring;
        x.ring_n = a.ring;
        x.stg = stg + (size_t)(warp - 1) * S * 32 * a.pitch;
        x.meta = meta + (warp - 1) * S * 32 * 4;
        x.pitch = a.pitch;
        x.pw = warp - 1;
        x.nprod = nprod;
        x.nch = nch;
        x.h3 = h3;
        x.m = m;
        x.pool = pool;
        produce_any(a, Q, x, qprod + (warp - 1) * 512, a.qrow0 + b);
      }
      continue;
    }

    // ================================ consumer ================================
    WarpTopK<M> top;
    top.init(a.kr);
    int64_t c = 0, jbase = 0;
    int32_t wnode = -1;
    uint32_t wkey = 0, wl = 0;
    bool wvalid = false;
    bool whave = false, wpf = false;
    SkipThr<M> thr;              // skip rule prepared against the current best key
    uint32_t thr_key = 0;
    bool thr_ok = false;
    int wpos = 32;

    const long long tc0 = KP(a.prof) ? clock64() : 0;
    long long p_wait = 0, p_walk = 0, p_win = 0;
    int ex_cnt = 0;
    bool ex_ovf = false;
    while (c < budget) {
      // ------------------------------ restart ------------------------------
      if (wpos >= 32) {
        // ---- fast path: FASTC whole produced chunks in which no draw can be accepted.  Against the
        // current s_max every draw is skipped (so none is a new best and the threshold cannot move);
        // each unevaluated node among them is evaluated once (the atomicOr that flips its bit) and
        // skipped, exactly as the sequential loop would do draw by draw; the budget is not reached.
        const int64_t ch0 = jbase / 32;
        if (top.cnt > 0 && nprod > 0 && ch0 + FASTC <= nch && c + 32 * FASTC <= budget) {
          const long long tw = KP(a.prof) ? clock64() : 0;
          int32_t fnode[FASTC];
          uint32_t fkey[FASTC];
#pragma unroll
          for (int t = 0; t < FASTC; ++t) ring_get(ring, a.ring, hdr, ch0 + t, fnode[t], fkey[t]);
          if (KP(a.prof)) p_wait += clock64() - tw;
          if (!thr_ok || thr_key != top.key_at0) {
            thr.set(top.key_at0, a.e_num, a.e_den);
            thr_key = top.key_at0;
            thr_ok = true;
          }
          // the chunks before the first one holding a draw that passes the skip test go the fast way
          unsigned pm = 0;
#pragma unroll
          for (int t = 0; t < FASTC; ++t) pm |= __any_sync(FULL, !thr.skip(fkey[t])) ? (1u << t) : 0u;
          const int tp = pm ? __ffs(pm) - 1 : FASTC;
          if (tp > 0) {
            bool fr[FASTC];
#pragma unroll
            for (int t = 0; t < FASTC; ++t) {
              fr[t] = false;
              if (t < tp) {
                const uint32_t li = (uint32_t)fnode[t];   // the ring carries the pool index
                const uint32_t bit = 1u << (li & 31);
                fr[t] = !(atomicOr(ev + (li >> 5), bit) & bit);
              }
            }
            __syncwarp();
            int nf = 0;
#pragma unroll
            for (int t = 0; t < FASTC; ++t) {
              if (t < tp) {                             // (warp-uniform)
                int32_t nd = fnode[t];
                const bool ct = top.could_take(fkey[t]);
                if (pool && fr[t] && ct) nd = pool[nd]; // node id only when it may enter the top-k
                top.insert(fr[t], fkey[t], nd);         // Q5: skipped starts enter the top-k
                nf += __popc(__ballot_sync(FULL, fr[t]));
              }
            }
            c += nf;
            s_starts += nf;
            s_skip += nf;
            p_win += tp;
            __syncwarp();
            if (lane == 0) hdr->consumed = (int)(ch0 + tp);
            jbase += 32 * tp;
            continue;
          }
        }
        const int64_t j = jbase + lane;
        const int64_t ch = jbase / 32;
        if (ch < nch && nprod > 0) {                 // produced ahead into the ring
          const long long tw = KP(a.prof) ? clock64() : 0;
          uint32_t kk;
          int32_t pidx;
          ring_get(ring, a.ring, hdr, ch, pidx, kk);
          wkey = kk;
          wl = (uint32_t)pidx;
          wnode = pool ? -2 : pidx;                   // -2: valid, node id not looked up yet
          wvalid = true;
          if (KP(a.prof)) p_wait += clock64() - tw;
          ++p_win;
          whave = true;
          __syncwarp();
          if (lane == 0) hdr->consumed = (int)(ch + 1);
        } else {
          if (a.starts) {
            wnode = j < a.nstarts ? a.starts[j] : -1;
            wl = wnode >= 0 ? (a.P > 0 ? (uint32_t)a.local_idx[wnode] : (uint32_t)wnode) : 0u;
          } else {
            const uint64_t idx = rng_index(h3, (uint64_t)j, (uint64_t)m);
            wnode = pool ? pool[idx] : (int32_t)idx;
            wl = (uint32_t)idx;
          }
          wvalid = wnode >= 0;
          whave = false;
        }
        jbase += 32;
        wpos = 0;
        // prefetch the rows of the draws that could still be accepted: the skip threshold only
        // tightens as s_max improves, so "passes against the current best" is a superset
        wpf = false;
        if (whave && wvalid) {
          if (top.cnt > 0 && (!thr_ok || thr_key != top.key_at0)) {
            thr.set(top.key_at0, a.e_num, a.e_den);
            thr_key = top.key_at0;
            thr_ok = true;
          }
          wpf = top.cnt == 0 ? lane == 0 : !thr.skip(wkey);
          if (wpf && wnode == -2) wnode = pool[wl];
          if (!a.win_prefetch) wpf = false;
          if (__ballot_sync(FULL, wpf)) {
            cp_async_wait_all();      // older copies into rowbuf2 must land first
            if (wpf)
              for (int e = 0; e < k; ++e) {
                cp_async4(rowbuf2 + lane * k + e, a.rows + (size_t)wnode * k + e);
                if (a.P > 0) cp_async4(lrowbuf2 + lane * k + e, a.lrows + (size_t)wnode * k + e);
              }
          }
        }
      }
      const unsigned active = FULL << wpos;
      const unsigned invm = __ballot_sync(FULL, !wvalid) & active;
      const unsigned lim = invm ? ((1u << (__ffs(invm) - 1)) - 1u) : FULL;
      const bool evb = wvalid ? bit_get(ev, wl) : true;
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
      const bool ct = top.could_take(wkey);   // (warp-wide)
      if (newly && wnode == -2 && ct) wnode = pool[wl];
      if (am && lane == __ffs(am) - 1 && wnode == -2) wnode = pool[wl];   // the accepted start
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
      const long long tk0 = KP(a.prof) ? clock64() : 0;
      int32_t cur = __shfl_sync(FULL, wnode, al);
      uint32_t kcur = __shfl_sync(FULL, wkey, al);
      uint32_t curl = __shfl_sync(FULL, wl, al);
      int pf = -1;                 // row of cur prefetched into rowbuf[pf*k ..] by the last step
      int pf2 = al;                // ... or into rowbuf2[pf2*k ..] when the window was loaded
      if (!__shfl_sync(FULL, wpf, al)) pf2 = -1;
      bool stop = false;
      for (;;) {
        ex_insert(exh, ex_cnt, ex_ovf, gex, words, curl);
        ++s_exp;
        int32_t v = -1, vl = -1;
        if (pf >= 0 || pf2 >= 0) {
          cp_async_wait_all();
          __syncwarp();
        }
        if (lane < k) {
          v = pf >= 0 ? rowbuf[pf * k + lane] : (pf2 >= 0 ? rowbuf2[pf2 * k + lane] : a.rows[(size_t)cur * k + lane]);
          if (a.P > 0)
            vl = pf >= 0 ? lrowbuf[pf * k + lane]
                         : (pf2 >= 0 ? lrowbuf2[pf2 * k + lane] : a.lrows[(size_t)cur * k + lane]);
        }
        pf2 = -1;
        // Q10: neighbours in another partition are skipped (lrows holds -1 for them)
        const bool inpool = v >= 0 && (a.P == 0 || vl >= 0);
        const uint32_t lv = inpool ? (a.P > 0 ? (uint32_t)vl : (uint32_t)v) : 0u;
        __syncwarp();
        // prefetch the rows of the in-pool neighbours: the next cur is one of them
        if (a.walk_prefetch)
        for (int base = 0; base < k * k; base += 32) {
          const int idx = base + lane;
          const int t = __float2int_rz(__fmul_rn(__int2float_rn(idx) + 0.5f, rk));   // idx / k
          const int32_t vt = __shfl_sync(FULL, inpool ? v : -1, t < 32 ? t : 31);
          if (idx < k * k && vt >= 0) {
            cp_async4(rowbuf + idx, a.rows + (size_t)vt * k + (idx - t * k));
            if (a.P > 0) cp_async4(lrowbuf + idx, a.lrows + (size_t)vt * k + (idx - t * k));
          }
        }
        const bool evb2 = inpool ? bit_get(ev, lv) : true;
        const bool exb2 = (inpool && !a.ex_one) ? ex_has(exh, ex_ovf, gex, lv) : false;
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
        pf = a.walk_prefetch ? fi : -1;
        bool exq = exb2;
        if (a.ex_one) exq = lane == fi ? ex_has(exh, ex_ovf, gex, curl) : false;   // only the chosen neighbour
        if (__shfl_sync(FULL, exq, fi)) break;   // Q9: moving onto an expanded node restarts
      }
      if (KP(a.prof)) p_walk += clock64() - tk0;
      if (stop) break;
    }
    if (KP(a.prof) && lane == 0) {
      atomicAdd(a.prof + 0, (unsigned long long)(clock64() - tc0));
      if (a.task_cycles) a.task_cycles[task] = (unsigned long long)(clock64() - tc0);
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

// dynamic shared memory of one K1 CTA (the kernel's carve-up above)
size_t search_smem_bytes(const SearchArgs &a, bool sets) {
  const int nprod = a.starts ? 0 : a.nprod;
  size_t smem = HDR_BYTES + (size_t)a.ring * 32 * 16 + (size_t)nprod * (a.stages * 32 * (a.pitch + 16) + 512) +
                (size_t)(a.k * a.k + 32 * a.k) * 4 * (a.P > 0 ? 2 : 1) + (sets ? 2 * QMAX * 4 + (size_t)a.st.vwords * 4 : 0) +
                EXCAP * 4;
  if (a.smem_bits) smem += (size_t)(a.bits_words / 2) * 4;   // the evaluated bitmap
  return smem;
}

template <int M, int L, int CPL, int MB>
static cudaError_t run_search(const SearchArgs &a, cudaStream_t s) {
  const int Pn = a.part_cnt;
  const int64_t T = a.nq * Pn;
  if (T == 0) return cudaSuccess;
  // consumer + a.nprod producers (none when the starts are injected)
  const int nprod = a.starts ? 0 : a.nprod;
  const int warps = 1 + nprod;
  const size_t smem = search_smem_bytes(a, M == M_JAC);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_search<M, L, CPL, MB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  // persistent grid: the CTAs that fit at once (dynamic task scheduling balances the tail)
  int per_sm = 0;
  cudaError_t oe = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_search<M, L, CPL, MB>, warps * 32, smem);
  if (oe != cudaSuccess) return oe;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  int64_t blocks = T < (int64_t)per_sm * nsm ? T : (int64_t)per_sm * nsm;
  if (blocks > a.gslots) blocks = a.gslots;
  cudaError_t me = cudaMemsetAsync(a.task_ctr, 0, sizeof(unsigned long long), s);
  if (me != cudaSuccess) return me;
  if (getenv("KNNG_PROFILE"))
    fprintf(stderr, "KNNG_PROFILE k_search: %lld CTAs, %d per SM resident (%zu B smem each)\n", (long long)blocks,
            per_sm, smem);
  k_search<M, L, CPL, MB><<<(unsigned)blocks, warps * 32, smem, s>>>(a);
  return cudaGetLastError();
}

#define KNNG_SHAPES(X, M) \
  X(M, 1, 1) X(M, 2, 1) X(M, 4, 1) X(M, 8, 1) X(M, 16, 1) X(M, 32, 1) X(M, 32, 2) X(M, 32, 4)
// fp32 rows of <= 32 chunks: 4 chunks per lane at most, partials in-lane (see VecQuery::reduce)
#define KNNG_SHAPES_F32(X) \
  X(M_F32, 1, 1) X(M_F32, 1, 2) X(M_F32, 1, 3) X(M_F32, 1, 4) X(M_F32, 2, 3) X(M_F32, 2, 4) X(M_F32, 4, 3) \
  X(M_F32, 4, 4) X(M_F32, 8, 3) X(M_F32, 8, 4) X(M_F32, 32, 2) X(M_F32, 32, 4)

// the 96-register variant (10 two-warp CTAs per SM) for the u8 d=128 and Jaccard shapes (C1, C3, C4)
#define LEAN_OK(MM, LL, CC) (((MM) == M_U8 && (LL) == 8 && (CC) == 1) || (MM) == M_JAC)
cudaError_t launch_search(const VecGeom &g, const SearchArgs &a, cudaStream_t s, int *n_launch) {
  if (n_launch) ++*n_launch;
#define X(MM, LL, CC) \
  if (g.metric == MM && g.L == LL && g.CPL == CC) {                                         \
    if constexpr (LEAN_OK(MM, LL, CC))                                                       \
      if (a.lean && !a.starts && a.nprod == 1) return run_search<MM, LL, CC, 10>(a, s);      \
    return run_search<MM, LL, CC, 4>(a, s);                                                  \
  }
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
