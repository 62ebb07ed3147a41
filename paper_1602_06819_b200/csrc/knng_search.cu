// knng_search.cu -- K1 iGNNS search (section 3) and K2 partition merge (Alg. 3,
// P:166-178).
//
// One CTA runs one (query, partition) task at a time: warp 0 is the CONSUMER, which takes every
// decision of the search in the paper's sequential order (draw, redraw, evaluate, skip, accept,
// walk, budget); warp 1 is the PRODUCER, which evaluates the random starts ahead of it.  The draw
// sequence of a task is a pure function of the counter RNG (reading Q4) and the key of a draw a
// pure function of (query, node), so the producer can run ahead, 32 draws per chunk:
//   * gather: the 32 drawn rows are staged in shared memory with 16-byte cp.async copies;
//   * evaluate: one row per lane from shared memory (or the warp evaluator);
//   * repeat flag: whether the draw's pool node was already drawn EARLIER in the sequence -- a
//     test-and-set on the task's draw bitmap D (lowest lane first inside a chunk), whose latency is
//     hidden behind the next chunk's gather;
//   * publish: (pool index, key, node id, repeat) into a ring of chunks in shared memory.
// A draw is a free redraw (Q4) iff it repeats an earlier draw, or its node was evaluated by a walk
// -- and the consumer keeps the nodes its walks evaluated (W) and expanded (X) in a hash table in
// SHARED memory.  So deciding which draws are fresh needs no global-memory round trip: the restart
// loop of the consumer runs from shared memory alone.  The walk's neighbours consult W and the
// bitmap E of the consumed fresh draws (fire-and-forget reductions when a draw is committed), read
// together with the neighbours' vectors -- one round trip per walk step with the next rows
// prefetched.  Everything the consumer commits -- evaluations, top-k inserts, counters -- happens
// in the sequential algorithm's order, so results and counters are identical to the oracle's.
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>

#include "knng_common.cuh"
#include "knng_internal.h"

// Cycle counters (builds with -DKNNG_PROFILE_COUNTERS, KNNG_PROFILE=1 at run time): summed per task into
// SearchArgs::prof[0..9] = consumer, consumer ring wait, walks, producer gather wait, producer ring-full
// wait, windows, walk steps, tasks whose hash overflowed, fast-path chunks, produced chunks.
#ifdef KNNG_PROFILE_COUNTERS
#define KPROF(...) __VA_ARGS__
#else
#define KPROF(...)
#endif

namespace knng {

constexpr int FASTC = 2;          // chunks the consumer's skip-only fast path commits at once (<= ring)
constexpr int HDR_BYTES = 128;
constexpr int WPF = 8;            // window prefetch slots (rows of draws that may be accepted)
constexpr uint32_t HW = 1u, HX = 2u;   // hash entry flags: evaluated by a walk / expanded

struct RingHdr {
  int consumed;           // consumer -> producer: chunks < consumed are free
  int done;               // consumer finished the task
  int next_task;          // dynamic task scheduler: the CTA's next task
  int pad;
};

// explicit state spaces (a generic volatile access compiles to LD.E.STRONG.SYS, a generic atomic to ATOM.E)
__device__ __forceinline__ int lds_volatile(const int *p) {
  int v;
  asm volatile("ld.volatile.shared.b32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ void sts_volatile(int *p, int v) {
  asm volatile("st.volatile.shared.b32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
// bit-plane words of the task: shared (gs = false) or global (gs = true); warp-uniform choice
__device__ __forceinline__ void plane_red_or(uint32_t *p, uint32_t v, bool gs) {
  if (gs) asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
  else asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t plane_atom_or(uint32_t *p, uint32_t v, bool gs) {
  uint32_t o;
  if (gs) asm volatile("atom.relaxed.gpu.global.or.b32 %0, [%1], %2;" : "=r"(o) : "l"(p), "r"(v) : "memory");
  else asm volatile("atom.shared.or.b32 %0, [%1], %2;" : "=r"(o) : "r"(smem_u32(p)), "r"(v) : "memory");
  return o;
}
__device__ __forceinline__ uint32_t plane_ld(const uint32_t *p, bool gs) {
  uint32_t v;
  if (gs) asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  else asm volatile("ld.volatile.shared.b32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}

// asynchronous global -> shared copy of 4, 8 or 16 bytes (the row prefetches of the walk)
__device__ __forceinline__ void cp_async_n(void *smem_dst, const void *gsrc, int bytes) {
  const unsigned sa = smem_u32(smem_dst);
  if (bytes == 16) asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gsrc) : "memory");
  else if (bytes == 8) asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gsrc) : "memory");
  else asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(gsrc) : "memory");
}

// D/E bit planes of a task: word w holds the draw bits (D, producer) of pool nodes 16w..16w+15 in its
// low half and their consumed-evaluation bits (E, consumer) in its high half.
__device__ __forceinline__ uint32_t de_word(int32_t pidx) { return (uint32_t)pidx >> 4; }
__device__ __forceinline__ uint32_t d_bit(int32_t pidx) { return 1u << (pidx & 15); }
__device__ __forceinline__ uint32_t e_bit(int32_t pidx) { return 1u << (16 + (pidx & 15)); }

// ---- the consumer's hash of walk-evaluated (W) / expanded (X) pool nodes: entries (pidx << 2) | flags ----
__device__ __forceinline__ uint32_t h_slot(uint32_t pidx, int hb) { return (pidx * 0x9E3779B1u) >> (32 - hb); }
__device__ __forceinline__ uint32_t h_get(const uint32_t *H, int hb, int32_t pidx) {
  const uint32_t mask = (1u << hb) - 1u;
  uint32_t h = h_slot((uint32_t)pidx, hb);
  for (;;) {
    const uint32_t e = H[h];
    if (e == 0) return 0;
    if ((e >> 2) == (uint32_t)pidx) return e & 3u;
    h = (h + 1) & mask;
  }
}
// lane-concurrent insert (distinct or equal keys across lanes are both fine)
__device__ __forceinline__ void h_put(uint32_t *H, int hb, int32_t pidx, uint32_t fl) {
  const uint32_t mask = (1u << hb) - 1u, ent = ((uint32_t)pidx << 2) | fl;
  uint32_t h = h_slot((uint32_t)pidx, hb);
  for (;;) {
    uint32_t e = H[h];
    if (e == 0) {
      e = atomicCAS(H + h, 0u, ent);
      if (e == 0) return;
    }
    if ((e >> 2) == (uint32_t)pidx) {
      if ((e & fl) != fl) atomicOr(H + h, fl);
      return;
    }
    h = (h + 1) & mask;
  }
}

// ---------------------------------------------------------------------------------------------
// Producer
// ---------------------------------------------------------------------------------------------
struct ProdCtx {
  RingHdr *hdr;
  unsigned long long *ring;   // [ring][32][3] tagged words (see ring_put)
  int ring_n;                 // ring chunks (power of 2)
  uint8_t *stg;               // 2 x 32 staged rows (pitch bytes each)
  int4 *meta;                 // 2 x 32 {node, pidx, rb, re}
  int pitch;
  uint64_t h3;
  int64_t m;
  const int32_t *pool;
  const int32_t *starts;      // injected start sequence (unpartitioned only) or null
  int nstarts;
  uint32_t *de;               // D/E words of the task (shared or global)
  bool gde;                   // the D/E words are in global memory
  unsigned long long *prof;   // cycle counters or null
};

// draw j = 32 c + lane: (node id, pool index); pool index -1 past an injected sequence
__device__ __forceinline__ int2 draw_node(const ProdCtx &x, int64_t c) {
  const int64_t j = c * 32 + (threadIdx.x & 31);
  if (x.starts) {
    const int32_t nd = j < x.nstarts ? x.starts[j] : -1;
    return make_int2(nd, nd);
  }
  const uint64_t idx = rng_index(x.h3, (uint64_t)j, (uint64_t)x.m);
  return make_int2(x.pool ? x.pool[idx] : (int32_t)idx, (int32_t)idx);
}

// Test-and-set of the draw bitmap for a chunk's draws, in sequence order: inside the chunk the lowest
// lane of equal pool indices is the first occurrence (the others are repeats); across chunks the
// single producer issues chunk c's atomics after chunk c-1's.  Returns a word from which
// repeat_of() extracts the flag once the atomic has completed (used one iteration later).
__device__ __forceinline__ uint32_t draw_mark(const ProdCtx &x, int32_t pidx) {
  const unsigned grp = __match_any_sync(FULL, pidx);
  if (pidx < 0) return 0u;
  if (grp & lanemask_lt()) return 0xFFFFFFFFu;                  // an earlier lane drew the same node
#ifdef KNNG_HACK_NOATOM
  return x.gde ? plane_ld(x.de + de_word(pidx), true) : plane_atom_or(x.de + de_word(pidx), d_bit(pidx), x.gde);
#else
  return plane_atom_or(x.de + de_word(pidx), d_bit(pidx), x.gde);
#endif
}
__device__ __forceinline__ int repeat_of(uint32_t mark, int32_t pidx) {
  return pidx >= 0 ? (int)((mark & d_bit(pidx)) != 0) : 0;
}

// Ring entries: three 64-bit words per lane, each carrying its chunk's tag (chunk + 1) in the high half
// next to one datum -- (pidx | repeat << 31), key, node -- so that the consumer sees whole entries
// without a fence or flag: an aligned 64-bit shared store is single-copy atomic.  pidx 0x7FFFFFFF marks
// "no draw" (past the end of an injected start sequence).
constexpr uint32_t NO_DRAW = 0x7FFFFFFFu;
__device__ __forceinline__ void ring_put(unsigned long long *ring, int ring_n, int64_t c, int32_t pidx, int rep,
                                         uint32_t key, int32_t node) {
  const unsigned long long tag = (unsigned long long)(uint32_t)(c + 1) << 32;
  // plane-major slot: [3][32] words, so each plane's 32 lanes are one contiguous 256-byte row
  const unsigned sa = smem_u32(ring + (c & (ring_n - 1)) * 96 + (threadIdx.x & 31));
  const uint32_t w0 = pidx < 0 ? NO_DRAW : ((uint32_t)pidx | ((uint32_t)rep << 31));
  asm volatile("st.volatile.shared.b64 [%0], %1;" ::"r"(sa), "l"(tag | key) : "memory");
  asm volatile("st.volatile.shared.b64 [%0], %1;" ::"r"(sa + 256), "l"(tag | (uint32_t)node) : "memory");
  asm volatile("st.volatile.shared.b64 [%0], %1;" ::"r"(sa + 512), "l"(tag | w0) : "memory");
}
struct RingEnt {
  int32_t pidx;   // -1: no draw
  int rep;
  uint32_t key;
  int32_t node;
};
// consumer: wait until chunk ch is in its slot and read this lane's entry
__device__ __forceinline__ RingEnt ring_get(const unsigned long long *ring, int ring_n, int64_t ch) {
  const uint32_t tag = (uint32_t)(ch + 1);
  const unsigned sa = smem_u32(ring + (ch & (ring_n - 1)) * 96 + (threadIdx.x & 31));
  unsigned long long a, b, c;
  for (;;) {
    asm volatile("ld.volatile.shared.b64 %0, [%1];" : "=l"(a) : "r"(sa) : "memory");
    asm volatile("ld.volatile.shared.b64 %0, [%1];" : "=l"(b) : "r"(sa + 256) : "memory");
    asm volatile("ld.volatile.shared.b64 %0, [%1];" : "=l"(c) : "r"(sa + 512) : "memory");
    if (__all_sync(FULL, (uint32_t)(a >> 32) == tag && (uint32_t)(b >> 32) == tag && (uint32_t)(c >> 32) == tag)) break;
    __nanosleep(16);
  }
  RingEnt r;
  const uint32_t w0 = (uint32_t)c;
  r.pidx = w0 == NO_DRAW ? -1 : (int32_t)(w0 & 0x7FFFFFFFu);
  r.rep = (int)(w0 >> 31) & (w0 != NO_DRAW);
  r.key = (uint32_t)a;
  r.node = (int32_t)(uint32_t)b;
  return r;
}

// publish chunk c to the ring; false when the consumer has finished
__device__ __forceinline__ bool publish(const ProdCtx &x, int64_t c, int32_t pidx, int rep, uint32_t key,
                                        int32_t node) {
  const int lane = threadIdx.x & 31;
  int dn = 0;
  KPROF(const long long t0 = clock64();)
#ifdef KNNG_DEBUG_WAIT
  long long nw = 0;
  if (lane == 0)
    while (c - ((volatile RingHdr *)x.hdr)->consumed >= x.ring_n && !(dn = ((volatile RingHdr *)x.hdr)->done)) {
      __nanosleep(32);
      if (++nw == (1ll << 24))
        printf("KNNG stuck producer: block %d chunk %lld consumed %d\n", blockIdx.x, (long long)c,
               ((volatile RingHdr *)x.hdr)->consumed);
    }
#else
  // ring full: the consumer is behind (walking); back off so the waiting producer does not take issue
  // slots from the consumers of the SM
  if (lane == 0) {
    unsigned ns = 64;
    while (c - lds_volatile(&x.hdr->consumed) >= x.ring_n && !(dn = lds_volatile(&x.hdr->done))) {
      __nanosleep(ns);
      ns = ns < 1024 ? 2 * ns : 1024;
    }
  }
#endif
  dn = __shfl_sync(FULL, dn, 0);
  KPROF(if (x.prof && lane == 0) atomicAdd(x.prof + 4, (unsigned long long)(clock64() - t0));)
  if (dn) return false;
  KPROF(if (x.prof && lane == 0) atomicAdd(x.prof + 9, 1ull);)
  ring_put(x.ring, x.ring_n, c, pidx, rep, key, node);
  return true;
}

__device__ __forceinline__ bool consumer_done(const ProdCtx &x) {
  int dn = (threadIdx.x & 31) == 0 ? lds_volatile(&x.hdr->done) : 0;
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

// Vectors: two single-chunk stages; the gathers of chunk i+1 (and the draw bitmap atomics, and the
// pool loads of chunk i+2) are in flight while chunk i is evaluated and published.
template <class EV>
__device__ __forceinline__ void produce_vec(const SearchArgs &a, const EV &ev, const ProdCtx &x) {
  const int lane = threadIdx.x & 31;
  const int nck = EV::NCH > 0 ? EV::NCH : a.st.nchunks;
  const uint8_t *base = a.st.vec;
  const size_t stride = a.st.stride;
  const int r0 = lane / nck, c0 = lane % nck, rs = 32 / nck, cs = 32 % nck;
  // compile-time widths: LR lanes per row, each copying chunks sl, sl + LR, ... of its row (immediate
  // offsets), 32 / LR rows per pass -- one shuffle and NCH / LR copies per pass
  constexpr int LR = EV::NCH >= 8 && EV::NCH % 8 == 0 ? 8 : (EV::NCH > 0 && EV::NCH <= 8 ? EV::NCH : 0);
  auto issue = [&](int st, int2 d) {
    x.meta[st * 32 + lane] = make_int4(d.x, d.y, 0, 0);
    uint8_t *dst = x.stg + st * 32 * x.pitch;
    if constexpr (LR > 0 && (32 % LR) == 0) {
      constexpr int RPP = 32 / LR, CPR = EV::NCH / LR;
      const int sl = lane % LR, rr = lane / LR;
#pragma unroll
      for (int p = 0; p < LR; ++p) {
        const int r = p * RPP + rr;
        const int32_t id = __shfl_sync(FULL, d.x, r);
        if (id >= 0) {
          const uint8_t *src = base + (size_t)id * stride + sl * 16;
          uint8_t *drow = dst + r * x.pitch + sl * 16;
#pragma unroll
          for (int t = 0; t < CPR; ++t) cp_async16(drow + t * LR * 16, src + t * LR * 16);
        }
      }
    } else {
      int r = r0, cc = c0;
#pragma unroll 8
      for (int j = 0; j < nck; ++j) {
        const int32_t id = __shfl_sync(FULL, d.x, r);
        if (id >= 0) cp_async16(dst + r * x.pitch + cc * 16, base + (size_t)id * stride + (size_t)cc * 16);
        cc += cs;
        r += rs;
        if (cc >= nck) { cc -= nck; ++r; }
      }
    }
  };
  int2 d0 = draw_node(x, 0);
  issue(0, d0);
  uint32_t mk_cur = draw_mark(x, d0.y);
  cp_async_commit();
  int2 pn = draw_node(x, 1);
  for (int64_t i = 0;; ++i) {
    if (consumer_done(x)) break;
    issue((int)((i + 1) & 1), pn);
    const uint32_t mk_next = draw_mark(x, pn.y);
    pn = draw_node(x, i + 2);             // (pool load) in flight during this evaluation
    cp_async_commit();
    KPROF(const long long tw = clock64();)
    cp_async_wait<1>();
    __syncwarp();
    KPROF(if (x.prof && lane == 0) atomicAdd(x.prof + 3, (unsigned long long)(clock64() - tw));)
    const int st = (int)(i & 1);
    const int4 mt = x.meta[st * 32 + lane];
    // (the warp evaluator is warp-collective: every lane evaluates, invalid draws are masked after)
    const uint32_t kv = ev.key(x.stg + st * 32 * x.pitch, x.pitch, nck);
    const uint32_t key = mt.y >= 0 ? kv : 0u;
    __syncwarp();
    if (!publish(x, i, mt.y, repeat_of(mk_cur, mt.y), key, mt.x)) break;
    mk_cur = mk_next;
  }
  cp_async_wait<0>();
  __syncwarp();
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
      if (nck == 8) produce_vec(a, EvalLane<M_U8, 8>{qsm}, x);
      else produce_vec(a, EvalLane<M_U8, 2>{qsm}, x);
    } else if constexpr (M == M_F32) {
      produce_vec(a, EvalLane<M_F32, 24>{qsm}, x);
    }
    return;
  }
  if (M == M_U8 && nck <= 8 && a.qs.nchunks <= 8) {
    // u8 rows of <= 128 B: 4 lanes x 2 chunks per candidate (2 shuffle levels)
    VecQuery<M_U8, 4, 2> PQ;
    PQ.load(a.qs, qrow, nullptr);
    produce_vec(a, EvalWarp<VecQuery<M_U8, 4, 2>>{PQ}, x);
  } else {
    produce_vec(a, EvalWarp<VecQuery<M, L, CPL>>{Q}, x);
  }
}

// Sets: lane j stages candidate j's token range (aligned 16-byte chunks, SLOTCH at most) in its own
// slot; longer sets are evaluated from global memory.  Prefetch levels: the node of chunk i + 2 and
// the offsets of chunk i + 1 are loaded while chunk i is computed.
template <int L>
__device__ __forceinline__ void produce_set(const SearchArgs &a, const SetQuery<L> &Q, const ProdCtx &x) {
  constexpr int SLOTCH = SetQuery<L>::SLOTCH;
  const int lane = threadIdx.x & 31;
  const uint32_t *tok = a.st.tok;
  const uint64_t *off = a.st.off;
  auto issue = [&](int st, int2 d, uint64_t b, uint64_t e) {
    const uint64_t a0 = b & ~3ull;
    const int rb = (int)(b - a0), re = (int)(e - a0);
    x.meta[st * 32 + lane] = make_int4(d.x, d.y, rb, re);
    const int nch = d.y >= 0 ? (re + 3) >> 2 : 0;
    if (nch <= SLOTCH) {
      uint8_t *dst = x.stg + (st * 32 + lane) * x.pitch;
      for (int j = 0; j < nch; ++j) cp_async16(dst + 16 * j, tok + a0 + 4 * j);
    }
  };
  auto offs = [&](int2 d, uint64_t &b, uint64_t &e) {
    b = d.y >= 0 ? off[d.x] : 0;
    e = d.y >= 0 ? off[d.x + 1] : 0;
  };
  int2 d0 = draw_node(x, 0);
  uint64_t b0, e0;
  offs(d0, b0, e0);
  issue(0, d0, b0, e0);
  uint32_t mk_cur = draw_mark(x, d0.y);
  cp_async_commit();
  int2 n1 = draw_node(x, 1);
  uint64_t b1, e1;
  offs(n1, b1, e1);
  int2 n2 = draw_node(x, 2);
  for (int64_t i = 0;; ++i) {
    if (consumer_done(x)) break;
    issue((int)((i + 1) & 1), n1, b1, e1);
    const uint32_t mk_next = draw_mark(x, n1.y);
    n1 = n2;
    offs(n1, b1, e1);
    n2 = draw_node(x, i + 3);
    cp_async_commit();
    cp_async_wait<1>();
    __syncwarp();
    const int st = (int)(i & 1);
    const int4 mt = x.meta[st * 32 + lane];
    uint32_t key = 0;
    if (mt.y >= 0) {
      if (((mt.w + 3) >> 2) <= SLOTCH) {
        key = Q.eval_slot(x.stg + (st * 32 + lane) * x.pitch, mt.z, mt.w);
      } else {   // long set: straight from global memory
        const uint64_t b = off[mt.x];
        key = Q.eval_slot_global(tok + (b & ~3ull), mt.z, mt.w);
      }
    }
    __syncwarp();
    if (!publish(x, i, mt.y, repeat_of(mk_cur, mt.y), key, mt.x)) break;
    mk_cur = mk_next;
  }
  cp_async_wait<0>();
  __syncwarp();
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
  produce_set(a, Q, x);
}

// widths whose walk evaluates staged vectors one lane per neighbour (EvalLane shapes)
__host__ __device__ __forceinline__ bool walk_stage_ok(int metric, int nchunks) {
  return (metric == M_U8 && (nchunks == 8 || nchunks == 2)) || (metric == M_F32 && nchunks == 24);
}

// ---------------------------------------------------------------------------------------------
// K1: one CTA per (query, partition) task: warp 0 runs the search in the paper's sequential
// order, warp 1 produces its random-start keys ahead of it.
// MB: launch-bound variant.  MB = 8 keeps 128 registers per thread (8 two-warp CTAs per SM);
// MB = 10 caps a two-warp CTA at 96 registers for task mixes that want more concurrent walks.
// ---------------------------------------------------------------------------------------------
template <int M, int L, int CPL, int MB>
__global__ void __launch_bounds__(64, MB) k_search(SearchArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int k = a.k;
  RingHdr *hdr = (RingHdr *)smem;
  unsigned long long *ring = (unsigned long long *)(smem + HDR_BYTES);   // [ring][32][3] tagged words
  uint8_t *stg = smem + HDR_BYTES + a.ring * 32 * 24;                   // [2][32] rows
  int4 *meta = (int4 *)(stg + 2 * 32 * a.pitch);                        // [2][32]
  uint8_t *qprod = (uint8_t *)(meta + 2 * 32);                          // [512 B] query copy
  // rows the walk reads: ids int32[k] (unpartitioned) or lrows int2[k] = (id, local index) (P > 0),
  // RB bytes each, prefetched with cp.async of CU bytes
  const int RB = (a.P > 0 ? 8 : 4) * k;
  const int CU = (RB % 16 == 0) ? 16 : ((RB % 8 == 0) ? 8 : 4), NU = RB / CU;
  uint8_t *rowbuf = qprod + 512;                                        // [k] rows of cur's neighbours
  uint8_t *wbuf = rowbuf + ((k * RB + 15) & ~15);                       // [WPF] rows of possible starts
  // lane-form widths: the walk stages cur's neighbours' vectors too ([k] x pitch) and evaluates them
  // one lane per neighbour against the consumer's query copy qcons
  const bool wstage = M != M_JAC && walk_stage_ok(M, a.st.nchunks);
  uint8_t *qcons = wbuf + ((WPF * RB + 15) & ~15);                     // [512 B] (wstage)
  uint8_t *vbuf = qcons + (wstage ? 512 : 0);                           // [k][pitch] (wstage)
  uint32_t *pkey = (uint32_t *)(vbuf + (wstage ? k * a.pitch : 0));     // [32] pending walk evaluations
  int32_t *pid = (int32_t *)(pkey + 32);                                // [32]
  uint32_t *qscr = (uint32_t *)(pid + 32);                              // [2][QMAX] (sets)
  uint32_t *vbm = qscr + (M == M_JAC ? 2 * QMAX : 0);                   // [vwords] (sets)
  const int vwords = M == M_JAC ? a.st.vwords : 0;
  const uint32_t vw_lim = (uint32_t)a.st.vwords;
  uint32_t *H = vbm + vwords;                                           // [1 << hbits] W / X hash
  uint32_t *sbits = (uint32_t *)(((uintptr_t)(H + (1 << a.hbits)) + 15) & ~(uintptr_t)15);   // [de_words] (smem D/E)
  const int hb = a.hbits;
  const int hthr = (3 << hb) >> 2;                                      // fill limit of the hash
  const int Pn = a.part_cnt;
  const int64_t T = a.nq * Pn;
  // per CTA slot in global memory: [D/E words][expanded-overflow words]
  uint32_t *gslot = a.gbits + (int64_t)blockIdx.x * (a.de_words + a.x_words);
  unsigned long long s_evals = 0, s_starts = 0, s_skip = 0, s_exp = 0;
  int prev_qn = 0;                              // sets: tokens of the previous query (scratch 0)
  for (int w = threadIdx.x; w < vwords; w += blockDim.x) vbm[w] = 0;
  if (threadIdx.x == 0) hdr->next_task = (int)blockIdx.x;

  for (;;) {
    __syncthreads();                          // previous task finished by both warps
    const int64_t task = hdr->next_task;
    if (task >= T) break;
    const int64_t b = task / Pn;
    const int pl = (int)(task % Pn);          // output slot
    const int p = a.part_lo + pl;             // partition searched
    const int64_t m = a.P > 0 ? a.member_cnt[p] : a.n_t;
    const int32_t *pool = a.P > 0 ? a.members + (size_t)p * a.member_cap : nullptr;
    const int64_t dew = (m + 15) >> 4;
    uint32_t *de = a.smem_bits ? sbits : gslot;
    uint32_t *xg = gslot + a.de_words;
    for (int64_t w = threadIdx.x; w < (dew >> 2); w += blockDim.x) ((uint4 *)de)[w] = make_uint4(0, 0, 0, 0);
    for (int64_t w = (dew & ~3ll) + threadIdx.x; w < dew; w += blockDim.x) de[w] = 0;
    for (int w = threadIdx.x; w < (1 << hb); w += blockDim.x) H[w] = 0;
    for (int w = threadIdx.x; w < a.ring * 32 * 3; w += blockDim.x) ring[w] = 0;   // no stale tags
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

    typename QuerySel<M, L, CPL>::T Q;
    Q.load(a.qs, a.qrow0 + b, M == M_JAC ? qscr + warp * QMAX : nullptr);
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
      if (budget > 0) {
        ProdCtx x;
        x.hdr = hdr;
        x.ring = ring;
        x.ring_n = a.ring;
        x.stg = stg;
        x.meta = meta;
        x.pitch = a.pitch;
        x.h3 = h3;
        x.m = m;
        x.pool = pool;
        x.starts = a.starts;
        x.nstarts = a.nstarts;
        x.de = de;
        x.gde = !a.smem_bits;
        x.prof = a.prof;
        produce_any(a, Q, x, qprod, a.qrow0 + b);
      }
      continue;
    }

    // ================================ consumer ================================
    if (wstage) {
      const uint8_t *qg = a.qs.vec + (size_t)(a.qrow0 + b) * a.qs.stride;
      for (int cc = lane; cc < a.st.nchunks; cc += 32) *(uint4 *)(qcons + 16 * cc) = ldg16(qg + 16 * cc);
      __syncwarp();
    }
    WarpTopK<M> top;
    top.init(a.kr);
    int64_t c = 0, jbase = 0;
    int32_t wnode = -1, wl = -1;
    uint32_t wkey = 0;
    bool wrep = true;
    int wpos = 32, wslot = -1;                   // window lane state; wslot: its prefetch slot (-1: none)
    SkipThr<M> thr;                              // skip rule prepared against the current best key
    uint32_t thr_key = 0;
    bool thr_ok = false;
    int hcnt = 0;
    bool hovf = false;                           // the hash is full: walk evaluations go to E, expansions to xg
    const bool gde = !a.smem_bits;
    auto e_get = [&](int32_t pidx) -> bool {     // consumed evaluation bit (walk neighbours)
      return (plane_ld(de + de_word(pidx), gde) & e_bit(pidx)) != 0;
    };
    auto thr_update = [&]() {
      if (top.cnt > 0 && (!thr_ok || thr_key != top.key_at0)) {
        thr.set(top.key_at0, a.e_num, a.e_den);
        thr_key = top.key_at0;
        thr_ok = true;
      }
    };

    KPROF(const long long tc0 = clock64(); long long c_wait = 0, c_walk = 0; unsigned long long c_win = 0, c_steps = 0,
          c_fast = 0; long long c_ph[3] = {0, 0, 0};)
    while (c < budget) {
      // ------------------------------ restart ------------------------------
      if (wpos >= 32) {
        // ---- fast path: FASTC whole produced chunks in which no draw can be accepted.  Against the
        // current s_max every draw is skipped (so none is a new best and the threshold cannot move);
        // each fresh draw among them is evaluated once and skipped, exactly as the sequential loop
        // does draw by draw; the budget is not reached.
        const int64_t ch0 = jbase >> 5;
        if (top.cnt > 0 && c + 32 * FASTC <= budget) {
          KPROF(const long long tw = clock64();)
          RingEnt fe[FASTC];
#pragma unroll
          for (int t = 0; t < FASTC; ++t) fe[t] = ring_get(ring, a.ring, ch0 + t);
          KPROF(c_wait += clock64() - tw;)
          thr_update();
          // the chunks before the first one holding a draw that passes the skip test (or the end of an
          // injected sequence) go the fast way
          unsigned pm = 0;
#pragma unroll
          for (int t = 0; t < FASTC; ++t)
            pm |= __any_sync(FULL, fe[t].pidx < 0 || !thr.skip(fe[t].key)) ? (1u << t) : 0u;
          const int tp = pm ? __ffs(pm) - 1 : FASTC;
          if (tp > 0) {
            int nf = 0;
#pragma unroll
            for (int t = 0; t < FASTC; ++t) {
              if (t < tp) {                                   // (warp-uniform)
                const int32_t li = fe[t].pidx;
                bool fr = fe[t].rep == 0 && !(h_get(H, hb, li) & HW);
                if (hovf && fr) fr = !e_get(li);              // walk evaluations past the hash are in E
#ifndef KNNG_HACK_NOATOM
                if (fr) plane_red_or(de + de_word(li), e_bit(li), gde);
#endif
                top.insert(fr, fe[t].key, fe[t].node);        // Q5: skipped starts enter the top-k
                nf += __popc(__ballot_sync(FULL, fr));
              }
            }
            c += nf;
            s_starts += nf;
            s_skip += nf;
            __syncwarp();
            if (lane == 0) sts_volatile(&hdr->consumed, (int)(ch0 + tp));
            jbase += 32 * tp;
            KPROF(c_fast += tp;)
            continue;
          }
        }
        // ---- one chunk draw by draw ----
        const int64_t ch = jbase >> 5;
        KPROF(const long long tw = clock64();)
        const RingEnt e = ring_get(ring, a.ring, ch);
        KPROF(c_wait += clock64() - tw; ++c_win;)
        wl = e.pidx;
        wkey = e.key;
        wnode = e.node;
        wrep = e.rep != 0;
        __syncwarp();
        if (lane == 0) sts_volatile(&hdr->consumed, (int)(ch + 1));
        jbase += 32;
        wpos = 0;
        // prefetch the rows of the draws that could still be accepted: the skip threshold only
        // tightens as s_max improves, so "passes against the current best" is a superset
        wslot = -1;
        if (a.win_prefetch) {
          thr_update();
          const bool cand = wl >= 0 && !wrep && (top.cnt == 0 ? lane == 0 : !thr.skip(wkey));
          const unsigned cmk = __ballot_sync(FULL, cand);
          if (cmk) {
            const int r = __popc(cmk & lanemask_lt());
            if (cand && r < WPF) wslot = r;
            cp_async_wait_all();      // older copies into wbuf must land first
            __syncwarp();
            if (wslot >= 0) {
              const uint8_t *src = a.P > 0 ? (const uint8_t *)(a.lrows + (size_t)wnode * k)
                                           : (const uint8_t *)(a.rows + (size_t)wnode * k);
              for (int u = 0; u < NU; ++u) cp_async_n(wbuf + wslot * RB + u * CU, src + u * CU, CU);
            }
          }
        }
      }
      const unsigned active = FULL << wpos;
      const bool wvalid = wl >= 0;
      const unsigned invm = __ballot_sync(FULL, !wvalid) & active;
      const unsigned lim = invm ? ((1u << (__ffs(invm) - 1)) - 1u) : FULL;
      // Redraws are free (Q4): a draw repeating an earlier draw, or of a node a walk evaluated
      bool fresh = lane >= wpos && wvalid && !wrep && !(h_get(H, hb, wl) & HW);
      if (hovf && fresh) fresh = !e_get(wl);
      const unsigned fm = __ballot_sync(FULL, fresh) & active & lim;
      if (fm == 0) {
        if (invm) break;          // injected start sequence exhausted
        wpos = 32;
        continue;
      }
      unsigned cm = fm;
      if ((int64_t)__popc(cm) > budget - c) cm = first_bits(cm, (int)(budget - c));
      const bool inc = (cm >> lane) & 1u;
      unsigned am;
      thr_update();
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
#ifndef KNNG_HACK_NOATOM
      if (cmt) plane_red_or(de + de_word(wl), e_bit(wl), gde);
#endif
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
        if (invm) break;
        wpos = 32;
        continue;
      }
      wpos = al + 1;

      // ------------------- hill climbing, eager first improvement -------------------
      // One memory round trip per step: the rows and (for the lane-form widths) the vectors of cur's
      // in-pool neighbours are copied to shared memory together with their E bits; the next step reads
      // the chosen neighbour's row from there.  The walk's own evaluations go to the top-k in batches
      // (pbuf, flushed at the walk's end): the walk itself only compares against kcur.
      int32_t cur = __shfl_sync(FULL, wnode, al);
      uint32_t kcur = __shfl_sync(FULL, wkey, al);
      int32_t curl = __shfl_sync(FULL, wl, al);
      int rs = -1;                 // row of cur: rowbuf slot rs (prefetched by the last step), else
      int rw = __shfl_sync(FULL, wslot, al);   // wbuf slot rw (prefetched with the window), else global
      bool stop = false;
      int pn = 0;                  // pending walk evaluations in pbuf
      auto flush = [&]() {
        if (pn == 0) return;
        __syncwarp();
        const bool has = lane < pn;
        top.insert(has, has ? pkey[lane] : 0u, has ? pid[lane] : -1);
        pn = 0;
        __syncwarp();
      };
      KPROF(const long long tk0 = clock64();)
      if (rw >= 0) {               // the window's row copies must have landed
        cp_async_wait_all();
        __syncwarp();
      }
      for (;;) {
        KPROF(++c_steps; long long ts0 = clock64();)
        ++s_exp;
        int32_t v = -1, vl = -1;
        if (lane < k) {
          if (a.P > 0) {
            const int2 e2 = rs >= 0 ? ((const int2 *)(rowbuf + rs * RB))[lane]
                                    : (rw >= 0 ? ((const int2 *)(wbuf + rw * RB))[lane] : a.lrows[(size_t)cur * k + lane]);
            v = e2.x;
            vl = e2.y;
          } else {
            v = rs >= 0 ? ((const int32_t *)(rowbuf + rs * RB))[lane]
                        : (rw >= 0 ? ((const int32_t *)(wbuf + rw * RB))[lane] : a.rows[(size_t)cur * k + lane]);
          }
        }
        rw = -1;
        // Q10: neighbours in another partition are skipped (lrows holds -1 for them)
        const bool inpool = v >= 0 && (a.P == 0 || vl >= 0);
        const int32_t lv = inpool ? (a.P > 0 ? vl : v) : 0;
        __syncwarp();                          // rowbuf is read before the copies below overwrite it
        KPROF(__ballot_sync(FULL, inpool); long long ts1 = clock64(); c_ph[0] += ts1 - ts0;)
        // issue: rows (NU copies of CU bytes) and staged vectors (NCK copies of 16 bytes) of the in-pool
        // neighbours, their E bits and hash flags -- all in flight together
        const int per = NU + (wstage ? a.st.nchunks : 0);
        {
          const uint8_t *rsrc = a.P > 0 ? (const uint8_t *)a.lrows : (const uint8_t *)a.rows;
          for (int base = 0; base < k * per; base += 32) {
            const int idx = base + lane;
            const int t = idx / per;
            const int32_t vt = __shfl_sync(FULL, inpool ? v : -1, t < 32 ? t : 31);
            if (idx < k * per && vt >= 0) {
              const int u = idx - t * per;
              if (u < NU) cp_async_n(rowbuf + t * RB + u * CU, rsrc + (size_t)vt * RB + u * CU, CU);
              else cp_async16(vbuf + t * a.pitch + (u - NU) * 16, a.st.vec + (size_t)vt * a.st.stride + (u - NU) * 16);
            }
          }
        }
        // evaluated before?  W (this task's walks) or E (consumed fresh draws; walk evaluations past a full
        // hash)
        const bool eb = inpool ? e_get(lv) : true;
        const uint32_t hf = inpool ? h_get(H, hb, lv) : 0u;
        // cur is expanded (Q9 bookkeeping), while the copies are in flight
        if (!hovf) {
          if (lane == 0) h_put(H, hb, curl, HX);
          ++hcnt;
        } else if (lane == 0) {
          plane_red_or(xg + ((uint32_t)curl >> 5), 1u << (curl & 31), true);
        }
        uint32_t key;
        if constexpr (M == M_JAC) {
          key = Q.eval(a.st, inpool ? v : -1, k);
          cp_async_wait_all();
          __syncwarp();
        } else {
          cp_async_wait_all();
          __syncwarp();
          if (wstage) {   // lane t: neighbour t's whole distance from shared memory (lanes >= k read row 0)
            const uint8_t *vb = vbuf - (lane < k ? 0 : lane * a.pitch);
            if constexpr (M == M_U8) {
              key = a.st.nchunks == 8 ? EvalLane<M_U8, 8>{qcons}.key(vb, a.pitch, 8)
                                      : EvalLane<M_U8, 2>{qcons}.key(vb, a.pitch, 2);
            } else {
              key = EvalLane<M_F32, 24>{qcons}.key(vb, a.pitch, 24);
            }
          } else {
            key = Q.eval(a.st, inpool ? v : -1, k);
          }
        }
        const bool evb2 = (hf & HW) || eb;
        const bool imp = inpool && closer<M>(key, kcur);
        KPROF(__ballot_sync(FULL, imp); long long ts2 = clock64(); c_ph[1] += ts2 - ts1;)
        const unsigned im = __ballot_sync(FULL, imp);
        int fi = im ? __ffs(im) - 1 : 31;
        unsigned range = fi == 31 ? FULL : ((2u << fi) - 1u);
        if (a.full_scan) {
          // GNNS: every neighbour is evaluated; the walk moves to the most similar improving one
          // (the first in row order among equals): a warp arg-min under closer<M>
          range = FULL;
          uint32_t bk = key;
          int bl = imp ? lane : 32;
#pragma unroll
          for (int o = 16; o >= 1; o >>= 1) {
            const uint32_t ok2 = __shfl_xor_sync(FULL, bk, o);
            const int ol = __shfl_xor_sync(FULL, bl, o);
            if (ol < 32 && (bl == 32 || closer<M>(ok2, bk) || (!closer<M>(bk, ok2) && ol < bl))) {
              bk = ok2;
              bl = ol;
            }
          }
          fi = im ? bl : 31;
        }
        unsigned fm2 = __ballot_sync(FULL, inpool && !evb2) & range;
        bool hit2 = false;
        if ((int64_t)__popc(fm2) > budget - c) { fm2 = first_bits(fm2, (int)(budget - c)); hit2 = true; }
        const bool cm2 = (fm2 >> lane) & 1u;
        const int nf2 = __popc(fm2);
        if (!hovf && hcnt + nf2 > hthr) {   // the hash is full: overflow into E / xg from here on
          for (int64_t w = lane; w < ((m + 31) >> 5); w += 32) xg[w] = 0;
          __syncwarp();
          hovf = true;
        }
        if (cm2) {
          if (!hovf) h_put(H, hb, lv, HW);
          else plane_red_or(de + de_word(lv), e_bit(lv), gde);
        }
        hcnt += nf2;
        if (pn + nf2 > 32) flush();
        if (cm2) {
          const int q = pn + __popc(fm2 & lanemask_lt());
          pkey[q] = key;
          pid[q] = v;
        }
        pn += nf2;
        c += nf2;
        __syncwarp();
        KPROF(long long ts3 = clock64(); c_ph[2] += ts3 - ts2;)
        if (hit2) { stop = true; break; }    // the over-budget evaluation is not performed
        if (!im) break;                      // local maximum -> restart
        cur = __shfl_sync(FULL, v, fi);
        kcur = __shfl_sync(FULL, key, fi);
        curl = __shfl_sync(FULL, lv, fi);
        rs = fi;
        bool exq = lane == fi ? ((hf & HX) != 0 || (hovf && ((plane_ld(xg + ((uint32_t)curl >> 5), true) >> (curl & 31)) & 1u))) : false;
        if (__shfl_sync(FULL, exq, fi)) break;   // Q9: moving onto an expanded node restarts
      }
      flush();
      KPROF(c_walk += clock64() - tk0;)
      if (stop) break;
    }
    KPROF(if (a.prof && lane == 0) {
      atomicAdd(a.prof + 0, (unsigned long long)(clock64() - tc0));
      atomicAdd(a.prof + 1, (unsigned long long)c_wait);
      atomicAdd(a.prof + 2, (unsigned long long)c_walk);
      atomicAdd(a.prof + 5, c_win);
      atomicAdd(a.prof + 6, c_steps);
      atomicAdd(a.prof + 7, hovf ? 1ull : 0ull);
      atomicAdd(a.prof + 8, c_fast);
      atomicAdd(a.prof + 10, (unsigned long long)c_ph[0]);
      atomicAdd(a.prof + 11, (unsigned long long)c_ph[1]);
      atomicAdd(a.prof + 12, (unsigned long long)c_ph[2]);
    })
    if (lane == 0) sts_volatile(&hdr->done, 1);
    s_evals += c;
    if (lane < a.kr) {
      const size_t o = ((size_t)b * Pn + pl) * a.kr + lane;
      a.out_ids[o] = lane < top.cnt ? top.id : -1;
      a.out_keys[o] = lane < top.cnt ? top.key : 0u;
    }
    cp_async_wait_all();
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
  const size_t RB = (size_t)(a.P > 0 ? 8 : 4) * a.k;
  const bool wstage = !sets && walk_stage_ok(a.metric, a.st.nchunks);
  size_t smem = HDR_BYTES + (size_t)a.ring * 32 * 24 + (size_t)2 * 32 * (a.pitch + 16) + 512 +
                ((a.k * RB + 15) & ~(size_t)15) + ((WPF * RB + 15) & ~(size_t)15) +
                (wstage ? 512 + (size_t)a.k * a.pitch : 0) + 2 * 32 * 4 +
                (sets ? 2 * QMAX * 4 + (size_t)a.st.vwords * 4 : 0) + ((size_t)4 << a.hbits);
  if (a.smem_bits) smem += (size_t)a.de_words * 4 + 16;   // the D/E planes (16-byte aligned)
  return smem;
}

template <int M, int L, int CPL, int MB>
static cudaError_t run_search(const SearchArgs &a, cudaStream_t s) {
  const int Pn = a.part_cnt;
  const int64_t T = a.nq * Pn;
  if (T == 0) return cudaSuccess;
  const size_t smem = search_smem_bytes(a, M == M_JAC);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_search<M, L, CPL, MB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  // persistent grid: the CTAs that fit at once (dynamic task scheduling balances the tail)
  int per_sm = 0;
  cudaError_t oe = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_search<M, L, CPL, MB>, 64, smem);
  if (oe != cudaSuccess) return oe;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  int64_t blocks = T < (int64_t)per_sm * nsm ? T : (int64_t)per_sm * nsm;
  if (blocks > a.gslots) blocks = a.gslots;
  if (const char *e = getenv("KNNG_GRID")) blocks = std::max<int64_t>(1, std::min<int64_t>(blocks, atoll(e)));   // measurement
  cudaError_t me = cudaMemsetAsync(a.task_ctr, 0, sizeof(unsigned long long), s);
  if (me != cudaSuccess) return me;
  if (getenv("KNNG_PROFILE"))
    fprintf(stderr, "KNNG_PROFILE k_search: %lld CTAs, %d per SM resident (%zu B smem each, ring %d, hash %d, %s D/E)\n",
            (long long)blocks, per_sm, smem, a.ring, 1 << a.hbits, a.smem_bits ? "smem" : "global");
  k_search<M, L, CPL, MB><<<(unsigned)blocks, 64, smem, s>>>(a);
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
      if (a.lean) return run_search<MM, LL, CC, 10>(a, s);                                   \
    return run_search<MM, LL, CC, 8>(a, s);                                                  \
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
