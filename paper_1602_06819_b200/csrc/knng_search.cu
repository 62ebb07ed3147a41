// knng_search.cu -- K1 iGNNS search (section 3) and K2 partition merge (Alg. 3,
// P:166-178).
//
// One WARP runs one (query, partition) task at a time and takes every decision of the search in
// the paper's sequential order (draw, redraw, evaluate, skip, accept, walk, budget); a CTA holds
// WPC independent warps and the grid is persistent with a dynamic task counter.  The search is a
// latency chain (each random-start chunk and each walk step is one memory round trip), so the
// design keeps as many tasks in flight per SM as the registers allow (20 warps on sm_100a at 96
// registers) and gives each a small shared-memory footprint:
//   * restart draws (Q4) are taken 32 at a time ("chunk"): the drawn rows are gathered into the
//     warp's stage with 16-byte cp.async copies (8 lanes per 128-byte row: coalesced row segments),
//     together with the words of the task's evaluated bitmap E; the keys are computed one lane per
//     row from shared memory.  A draw is fresh iff its E bit is clear and no lower lane of the
//     chunk drew the same node; a chunk in which no fresh draw can be accepted (every key skipped
//     against the current s_max) is committed at once -- its fresh draws are counted, enter
//     the top-k (Q5) and set their E bits -- else it is resolved draw by draw.
//   * walk steps: the rows, vectors and E / X (expanded) bits of the current node's in-pool
//     neighbours are copied together (one round trip; the chosen neighbour's row is then already in
//     shared memory for the next step), the first improving neighbour is found with a ballot, and
//     the walk's evaluations reach the top-k in batches (the walk itself compares against kcur only).
// E and X live per warp slot in global memory (they are L2-resident for the pools of C1/C4 and
// stream for the 1M-node pools of C2/C3), zeroed when a task starts; only this warp reads or writes
// them, and its reductions are ordered before its later loads by the warp barriers between them.
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <map>
#include <mutex>

#include "knng_common.cuh"
#include "knng_internal.h"
#include "knng_update_one.cuh"

// Cycle counters (builds with -DKNNG_PROFILE_COUNTERS, KNNG_PROFILE=1 at run time): summed per task into
// SearchArgs::prof[0..12] = task, -, walks, -, -, windows, walk steps, -, fast chunks, chunks, walk
// phases (row, copies+keys, commit).
#ifdef KNNG_PROFILE_COUNTERS
#define KPROF(...) __VA_ARGS__
#else
#define KPROF(...)
#endif

namespace knng {

constexpr int WPC = 4;            // warps (independent tasks) per CTA
#ifndef KNNG_K1_MB
#define KNNG_K1_MB 6              // launch bound: >= 6 CTAs (24 warps) per SM -> <= 80 registers (measured best: 5 -> 96 and 8 -> 64 are slower)
#endif
constexpr int WPF = 4;            // window row prefetch slots (draws that may be accepted)

// explicit state spaces for the task's bit planes (global, gpu-scope: one warp reads and writes them)
__device__ __forceinline__ void g_red_or(uint32_t *p, uint32_t v) {
  asm volatile("red.relaxed.gpu.global.or.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t g_ld(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// asynchronous global -> shared copies to a 32-bit shared address (no generic-to-shared conversion)
__device__ __forceinline__ void cpa16(unsigned sa, const void *gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cpa_n(unsigned sa, const void *gsrc, int bytes) {
  if (bytes == 16) asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gsrc) : "memory");
  else if (bytes == 8) asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gsrc) : "memory");
  else asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(gsrc) : "memory");
}

// W filter of a dsk task (shared, WFLT_WORDS words): one bit per hashed pool index of the walk evaluations
constexpr int WFLT_WORDS = 1024;
__device__ __forceinline__ uint32_t wflt_h(int32_t i) { return ((uint32_t)i * 0x9E3779B1u) >> 17; }   // 15 bits
__device__ __forceinline__ bool wflt_test(const uint32_t *f, int32_t i) {
  const uint32_t h = wflt_h(i);
  return ((f[h >> 5] >> (h & 31)) & 1u) != 0;
}
__device__ __forceinline__ void wflt_set(uint32_t *f, int32_t i) {
  const uint32_t h = wflt_h(i);
  atomicOr(f + (h >> 5), 1u << (h & 31));
}
// E / X planes of a task: word w holds the evaluated bits (E) of pool nodes 16w..16w+15 in its low
// half and their expanded bits (X) in its high half.
__device__ __forceinline__ uint32_t pw(int32_t pidx) { return (uint32_t)pidx >> 4; }
__device__ __forceinline__ uint32_t e_bit(int32_t pidx) { return 1u << (pidx & 15); }
__device__ __forceinline__ uint32_t x_bit(int32_t pidx) { return 1u << (16 + (pidx & 15)); }

// widths whose keys are computed one lane per staged row (lane_key shapes)
__host__ __device__ __forceinline__ bool lane_eval_ok(int metric, int nchunks) {
  return (metric == M_U8 && (nchunks == 8 || nchunks == 2)) || (metric == M_F32 && nchunks == 24);
}

// Lane form: one lane per staged row, the whole distance in-lane (no shuffles; NCH independent chunk
// chains), the query's chunks broadcast from shared memory.  F32 keeps the canonical tree (Q24):
// with NCH <= 32 partial i is chunk i alone (f4_leaf from +0), partials >= NCH are +0, and the
// levels o = 16..1 add partial i + o into partial i -- the xor butterfly's values.
// Staged rows of the lane-form widths with nchunks % 8 == 0 are stored swizzled: chunk c of row r at
// position (c & ~7) | ((c ^ r) & 7), so that the 8 lanes of a quarter-warp reading chunk c of rows
// r..r+7 hit 8 different 16-byte bank groups (no padding needed).
__device__ __forceinline__ int swz_pos(int c, int r, bool swz) { return swz ? ((c & ~7) | ((c ^ r) & 7)) : c; }

template <int M, int NCH>
__device__ __forceinline__ uint32_t lane_key(const uint8_t *qsm, const uint8_t *row, int rr, bool swz) {
  if constexpr (M == M_U8) {   // exact integer sum: four independent accumulators
    uint32_t acc[4] = {0, 0, 0, 0};
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      const uint4 q = *(const uint4 *)(qsm + 16 * c), r = *(const uint4 *)(row + 16 * swz_pos(c, rr, swz));
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
      p[i] = i < NCH ? f4_leaf(0.0f, *(const uint4 *)(qsm + 16 * i), *(const uint4 *)(row + 16 * swz_pos(i, rr, swz))) : 0.0f;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1)
#pragma unroll
      for (int i = 0; i < o; ++i) p[i] = __fadd_rn(p[i], p[i + o]);
    return __float_as_uint(p[0]);
  }
}

// keys of rows staged at stage + r * pitch (lane r; lanes >= nrows read row 0 and are masked by the caller)
template <int M, int L, int CPL>
__device__ __forceinline__ uint32_t staged_keys(const typename QuerySel<M, L, CPL>::T &Q, const uint8_t *qsm,
                                                const uint8_t *stage, int pitch, int nck, int nrows, bool lane_form,
                                                bool swz) {
  const int lane = threadIdx.x & 31;
  if constexpr (csr_metric(M)) {
    return 0u;   // (sets and strings are evaluated per lane by the callers)
  } else {
    if (lane_form) {
      const int r = lane < nrows ? lane : 0;
      const uint8_t *row = stage + r * pitch;
      if constexpr (M == M_U8) return nck == 8 ? lane_key<M_U8, 8>(qsm, row, r, swz) : lane_key<M_U8, 2>(qsm, row, r, swz);
      else return lane_key<M_F32, 24>(qsm, row, r, swz);
    }
    return Q.eval_smem(stage, pitch, nck);   // warp form over 32 staged rows
  }
}

// shared memory of the fused B = 1 update (after the warps' regions): s_n, hash / list / props, query tokens
__host__ __device__ __forceinline__ size_t fuse_bytes(const SearchArgs &a, bool sets) {
  return a.fuse ? ((16 + update_one_smem(a.ub.hcap, a.ub.ballmax) + (sets ? QSCR * 4 : 0) + 15) & ~(size_t)15) : 0;
}

// Key matrix of a sequence of B inserts on a small graph (the KT launches): row i = the keys of point
// qrow0 + i against nodes 0 .. n0 + i - 1 (the pool its search and update will see); ld = n0 + B rounded
// to 4.  Thread per (i, v); exact keys (pair_key: the canonical forms of every metric).
template <int M>
__global__ void k_keymat(StoreView st, int64_t qrow0, int64_t n0, int64_t B, int64_t ld, uint32_t *out) {
  const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t i = blockIdx.y;
  if (i >= B || v >= n0 + i) return;
  out[(size_t)i * ld + v] = pair_key<M>(st, qrow0 + i, v);
}

cudaError_t launch_keymat(int metric, const StoreView &st, int64_t qrow0, int64_t n0, int64_t B, int64_t ld,
                          uint32_t *out, cudaStream_t s) {
  if (B <= 0) return cudaSuccess;
  const dim3 grid((unsigned)((n0 + B + 127) / 128), (unsigned)B);
  if (metric == M_U8) k_keymat<M_U8><<<grid, 128, 0, s>>>(st, qrow0, n0, B, ld, out);
  else if (metric == M_F32) k_keymat<M_F32><<<grid, 128, 0, s>>>(st, qrow0, n0, B, ld, out);
  else if (metric == M_JAC) k_keymat<M_JAC><<<grid, 128, 0, s>>>(st, qrow0, n0, B, ld, out);
  else if (metric == M_JW) k_keymat<M_JW><<<grid, 128, 0, s>>>(st, qrow0, n0, B, ld, out);
  else k_keymat<M_COS><<<grid, 128, 0, s>>>(st, qrow0, n0, B, ld, out);
  return cudaGetLastError();
}

// Rows of a lane-form width (NCK 16-byte chunks, compile time) gathered into stage slots: lane r
// holds the node id of slot r (-1: none), rows r < nrows.  LPR lanes share a row so that every copy
// instruction reads whole 128-byte segments; rows with NCK % 8 == 0 are stored swizzled (swz_pos).
template <int NCK>
__device__ __forceinline__ void gather_lf(unsigned sb, int pitch, const uint8_t *base, int32_t myid, int nrows) {
  constexpr int LPR = NCK < 8 ? NCK : 8;   // lanes per row
  constexpr int RPI = 32 / LPR;            // rows per pass
  constexpr int CPR = NCK / LPR;           // copies per lane and row
  constexpr bool SWZ = NCK % 8 == 0;
  const int lane = threadIdx.x & 31, sl = lane % LPR, rr = lane / LPR;
#pragma unroll
  for (int pp = 0; pp < 32 / RPI; ++pp) {
    if (pp * RPI >= nrows) break;   // warp-uniform
    const int r = pp * RPI + rr;
    const int32_t id = __shfl_sync(FULL, myid, r);
    if (r < nrows && id >= 0) {
      const uint8_t *src = base + (size_t)(uint32_t)id * (NCK * 16) + 16 * sl;
      const unsigned dst = sb + r * pitch;
#pragma unroll
      for (int j = 0; j < CPR; ++j) {
        const int t = sl + LPR * j;
        cpa16(dst + 16 * (SWZ ? ((t & ~7) | ((t ^ r) & 7)) : t), src + 16 * LPR * j);
      }
    }
  }
}

// The same rows gathered by the TMA engine: lane r issues ONE bulk copy of row r (cp.async.bulk, NCK * 16
// bytes, unswizzled at pitch NCK * 16 + 16: the pad keeps the lane-per-row key loads conflict-free) that
// completes on the warp's mbarrier; lane 0 arrives with the phase's byte count first.  The caller waits
// for the phase (bulk_wait) before reading the stage.
template <int NCK>
__device__ __forceinline__ void gather_bulk(unsigned sb, int pitch, const uint8_t *base, int32_t myid, int nrows,
                                            uint64_t *bar) {
  const int lane = threadIdx.x & 31;
  const bool v = lane < nrows && myid >= 0;
  const unsigned m = __ballot_sync(FULL, v);
  if (lane == 0) mbar_arrive_expect_tx(bar, (unsigned)__popc(m) * (NCK * 16));
  __syncwarp();
  if (v) bulk_g2s(sb + lane * pitch, base + (size_t)(uint32_t)myid * (NCK * 16), NCK * 16, smem_u32(bar));
}
__device__ __forceinline__ void bulk_wait(uint64_t *bar, uint32_t &phase) {
  mbar_wait(bar, phase);
  phase ^= 1u;
}

// ---------------------------------------------------------------------------------------------
// K1: MB = minimum CTAs per SM of the launch bounds (WPC warps each).  NCK > 0: a lane-form width
// (u8 d = 32 / 128, f32 d = 96) with its geometry known at compile time; PART = 1 / 0: partitioned /
// unpartitioned graph (-1: read from the arguments); BK = 1: lane-form rows gathered by bulk copies
// (one-stage plans).
// ---------------------------------------------------------------------------------------------
template <int M, int L, int CPL, int MB, int NCK, int PART, int KT, int BK>
__global__ void __launch_bounds__(32 * WPC, MB) k_search(SearchArgs a) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int k = a.k;
  constexpr bool LF = NCK > 0;                                             // one lane per staged row
  constexpr bool SWZ = LF && !BK && NCK % 8 == 0;
  const bool part = PART < 0 ? a.P > 0 : PART == 1;
  const int nck = csr_metric(M) ? 0 : (LF ? NCK : a.st.nchunks);
  const int pitch = LF ? (SWZ ? NCK * 16 : NCK * 16 + 16) : a.pitch;
  const int RB = 4 * k;                                                    // bytes of a walked row (local indices)
  const int slotch = (pitch - 16) >> 4;                                    // sets: 16-byte chunks of a lane's slot
  const bool row_pf = KT == 0 && a.row_pf != 0;                           // (KT: rows are loaded, keys looked up)
  const bool es = KT || a.e_smem != 0;                                     // E bitmap in shared memory
  const bool ns2 = !KT && !csr_metric(M) && es && a.ns2 != 0;                  // two chunk stages (needs es)
  const bool xs = es && (KT || a.x_smem != 0);                             // X bitmap in shared memory too
  // perm_e (global E words, permutation draws): draws set no E bits -- a walk neighbour's "drawn before" is
  // pi^-1(v) <= the last processed draw -- so the words hold the WALK evaluations W only, and a draw reads
  // its word only when the warp's shared filter of W (one bit per hashed pool index) says it may be in W
  const bool dsk = !es && a.perm_e != 0 && a.starts == nullptr;
  // ---- this warp's shared memory (a.wbytes each; search_warp_bytes) ----
  uint8_t *wsm = smem + (size_t)warp * a.wbytes;
  uint8_t *stage = wsm;                                                   // [32][pitch] draw rows / set slots
  uint8_t *wvec = stage;                                                   // [k][pitch] the walk's neighbour vectors
  uint8_t *rowbuf = stage + (ns2 ? 64 : 32) * pitch;                       // [k] rows of cur's neighbours (row_pf)
  uint8_t *wrow = rowbuf + (row_pf ? ((k * RB + 15) & ~15) : 0);           // [WPF] rows of possible starts
  uint8_t *qsm = wrow + ((WPF * RB + 15) & ~15);                           // [512 B] query (vectors)
  uint32_t *pkey = (uint32_t *)(qsm + 512);                                // [32] pending walk evaluations
  int32_t *pid = (int32_t *)(pkey + 32);                                   // [32]
  uint32_t *qscr = (uint32_t *)(pid + 32);                                // [QSCR] query tokens + table (sets)
  uint8_t *jwp = (uint8_t *)(qscr + (csr_metric(M) ? QSCR : 0));            // [32][JW_PTR] JW character pointers
  uint32_t *ebits = (uint32_t *)(jwp + (M == M_JW ? 32 * JW_PTR : 0));      // [e_bytes / 4] E bitmap (es)
  uint32_t *wflt = ebits;                                                  // [WFLT_WORDS] W filter (dsk; !es)
  long long *sched = (long long *)(smem + (size_t)WPC * a.wbytes);         // [WPC] next task per warp
  uint64_t *mbar = (uint64_t *)(sched + WPC) + warp;                       // (BK) the warp's bulk-copy barrier
  uint32_t bph = 0;                                                        // (BK) its phase
  if constexpr (BK != 0) {
    if (lane == 0) {
      mbar_init(mbar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
  }
  const int Pn = a.part_cnt;
  const int64_t T = a.nq * Pn;
  const int64_t gw = (int64_t)blockIdx.x * WPC + warp;                      // warp slot
  uint32_t *planes = a.gbits + gw * a.de_words;                            // E / X words of the task
  unsigned long long s_evals = 0, s_starts = 0, s_skip = 0, s_exp = 0;
  unsigned long long s_ball = 0, s_prop = 0;
  // fused launch: nseq sequential inserts (each a batch of one against the graph the previous one left:
  // the paper's Alg. 1 + 2 point after point); else one pass over the launch's tasks
  const int nseq = a.fuse ? a.nseq : 1;
  // KT launches with srows: the rows of every node the sequence can reach, in shared memory after the key
  // table (the walks and the update read them there; the update writes both copies)
  int32_t *srw = nullptr;
  // KT: two key-table buffers -- insert it reads buffer it & 1 while warps 1.. (idle: the launch has one
  // task) stage row it + 1 of the key matrix into the other
  uint8_t *ktbase = smem + (size_t)WPC * a.wbytes + 16 * WPC + fuse_bytes(a, csr_metric(M));
  const size_t ktb = (size_t)(((a.n_t + nseq) * 4 + 15) & ~15ll);
  auto stage_kt = [&](int r, int t0, int nth) {
    uint32_t *dst = (uint32_t *)(ktbase + (r & 1) * ktb);
    const uint32_t *src = a.ktm + (size_t)r * a.ktm_ld;
    const int64_t nn = a.n_t + r, n4 = nn >> 2;
#pragma unroll 4
    for (int64_t v = (int)threadIdx.x - t0; v < n4; v += nth) ((uint4 *)dst)[v] = ((const uint4 *)src)[v];
    for (int64_t v = (n4 << 2) + (int)threadIdx.x - t0; v < nn; v += nth) dst[v] = src[v];
  };
  if constexpr (KT != 0) {
    if (a.srows) {
      srw = (int32_t *)(ktbase + 2 * ktb);
      const int64_t nr4 = ((a.n_t + nseq) * k) >> 2;
      for (int64_t v = threadIdx.x; v < nr4; v += blockDim.x) ((int4 *)srw)[v] = ((const int4 *)a.rows)[v];
      for (int64_t v = (nr4 << 2) + threadIdx.x; v < (a.n_t + nseq) * k; v += blockDim.x) srw[v] = a.rows[v];
      __syncthreads();
    }
  }
  if constexpr (KT != 0) {
    stage_kt(0, 0, blockDim.x);
    __syncthreads();
  }
  for (int it = 0; it < nseq; ++it) {
  const int64_t n_t = a.n_t + it, qrow0 = a.qrow0 + it, pid_base = a.pid_base + it;
  int64_t task = gw;
  // KT (the fused B = 1 launch on a small graph): the keys of the query against every pool node are
  // computed up front by the whole CTA into a shared table; the search and the update then read keys
  // from it instead of gathering rows (same keys, same decisions, same counters).
  uint32_t *kt = nullptr;
  if constexpr (KT != 0) kt = (uint32_t *)(ktbase + (it & 1) * ktb);   // row `it` of the key matrix (staged)

  while (task < T) {
    const int64_t b = task / Pn;
    const int pl = (int)(task % Pn);          // output slot
    const int p = a.route ? a.route[b] : a.part_lo + pl;   // partition searched
    const int64_t m = part ? a.member_cnt[p] : n_t;
    // the pool's store: on a partitioned graph the partition-local copy (index = local index, the pool
    // index of the draws); ids are converted through members when the task writes its top-k
    const size_t pbase = part ? (size_t)p * a.member_cap : 0;
    const uint8_t *vbase = (part && !csr_metric(M)) ? a.pvec + pbase * a.st.stride : a.st.vec;
    const int32_t *rbase = part ? a.prow + pbase * k : (srw ? srw : a.rows);
    StoreView sv = a.st;
    sv.vec = vbase;
    if (csr_metric(M) && part) sv.rng = a.pset + pbase;
    // next task (dynamic scheduling), read back at the end of this one
    if (lane == 0) sched[warp] = (long long)(gridDim.x * WPC + atomicAdd(a.task_ctr, 1ull));
    KPROF(const long long tc0 = clock64(); long long c_walk = 0; unsigned long long c_win = 0, c_steps = 0,
          c_fast = 0, c_chunks = 0; long long c_ph[6] = {0, 0, 0, 0, 0, 0};)
    // clear the task's E / X planes
    if (es) {   // E (and X) bitmaps in shared memory
      uint4 *e4 = (uint4 *)ebits;
      for (int w = lane; w < (a.e_bytes >> (xs ? 3 : 4)); w += 32) e4[w] = make_uint4(0, 0, 0, 0);
    }
    if (dsk) {
      uint4 *f4 = (uint4 *)wflt;
      for (int w = lane; w < WFLT_WORDS / 4; w += 32) f4[w] = make_uint4(0, 0, 0, 0);
    }
    if (!xs) {
      const int64_t nw = (m + 15) >> 4;
      uint4 *p4 = (uint4 *)planes;
      for (int64_t w = lane; w < (nw >> 2); w += 32) p4[w] = make_uint4(0, 0, 0, 0);
      for (int64_t w = (nw & ~3ll) + lane; w < nw; w += 32) planes[w] = 0;
    }
    // budget (Q6) -- never more than the pool (Q7)
    int64_t budget = (int64_t)floor((double)m / a.speedup);
    const int64_t lo = m < a.kr ? m : a.kr;
    if (budget < lo) budget = lo;
    if (budget > m) budget = m;

    typename QuerySel<M, L, CPL>::T Q;
    if constexpr (M == M_JW) Q.ptr = jwp + lane * JW_PTR;
    if (!LF && KT == 0) Q.load(a.qs, qrow0 + b, csr_metric(M) ? qscr : nullptr);
    if (LF) {
      const uint8_t *qg = a.qs.vec + (size_t)(qrow0 + b) * a.qs.stride;
      for (int cc = lane; cc < nck; cc += 32) *(uint4 *)(qsm + 16 * cc) = ldg16(qg + 16 * cc);
    }
    const uint64_t h3 = rng_prefix(a.seed, (uint64_t)(pid_base + b), (uint64_t)p);
    __syncwarp();

    WarpTopK<M> top;
    top.init(a.kr);
    int64_t c = 0, ch = 0;
    SkipThr<M> thr;                              // skip rule prepared against the current best key
    uint32_t thr_key = 0;
    bool thr_ok = false;
    auto thr_update = [&]() {
      if (top.cnt > 0 && (!thr_ok || thr_key != top.key_at0)) {
        thr.set(top.key_at0, a.e_num, a.e_den);
        thr_key = top.key_at0;
        thr_ok = true;
      }
    };
    // draw j of chunk c: (pool index, node); pool index -1 past an injected start sequence
    auto draw = [&](int64_t cc) -> int2 {
      const int64_t j = cc * 32 + lane;
      if (a.starts) {
        const int32_t nd = j < a.nstarts ? a.starts[j] : -1;
        return make_int2(nd, nd);
      }
      Perm pm;
      pm.init(h3, (uint64_t)m);
      const int32_t idx = pm.draw(j);
      return make_int2(idx, idx);
    };
    // ---- the draw of a chunk: issue(d) copies the drawn rows into the stage (sets: each lane its token
    // range) and returns the E word of each draw, read in the same round trip.
    const unsigned sb0 = smem_u32(stage);
    auto issue = [&](int2 d, uint64_t tb, uint64_t te) -> uint32_t {
      if constexpr (KT != 0) {
        return 0u;
      } else if constexpr (str_metric(M)) {
        // strings: keys are computed per lane from global memory (StrQuery)
      } else if constexpr (M == M_JAC) {
        const uint64_t a0 = tb & ~3ull;
        const int nch = d.x >= 0 ? ((int)(te - a0) + 3) >> 2 : 0;
        if (nch <= slotch)
          for (int jj = 0; jj < nch; ++jj) cpa16(sb0 + lane * pitch + 16 * jj, a.st.tok + a0 + 4 * jj);
      } else if constexpr (LF) {
        if constexpr (BK != 0) gather_bulk<NCK>(sb0, pitch, vbase, d.y, 32, mbar);
        else gather_lf<NCK>(sb0, pitch, vbase, d.y, 32);
      } else {
        const uint8_t *base = vbase;
        const size_t stride = a.st.stride;
        for (int e = lane; e < 32 * nck; e += 32) {
          const int r = e / nck, t = e - r * nck;
          const int32_t id = __shfl_sync(FULL, d.y, r);
          if (id >= 0) cpa16(sb0 + r * pitch + 16 * t, base + (size_t)id * stride + 16 * t);
        }
      }
      return (!es && d.x >= 0 && (!dsk || wflt_test(wflt, d.x))) ? g_ld(planes + pw(d.x)) : 0u;
    };
    // the E bit of pool node i: set / test (shared bitmap, or the low halves of the global words)
    auto e_set = [&](int32_t i) {
      if (es) atomicOr(ebits + (i >> 5), 1u << (i & 31));
      else g_red_or(planes + pw(i), e_bit(i));
    };
    auto e_smem_test = [&](int32_t i) -> bool { return ((ebits[i >> 5] >> (i & 31)) & 1u) != 0; };
    uint32_t *xbits = ebits + (a.e_bytes >> 2);  // xs: the X bitmap follows the E bitmap
    auto issue_to = [&](uint8_t *dst, int2 d) {
      if constexpr (!csr_metric(M) && KT == 0) {
        if constexpr (LF) {
          gather_lf<NCK>(smem_u32(dst), pitch, vbase, d.y, 32);
        } else {
          const unsigned sb = smem_u32(dst);
          for (int e = lane; e < 32 * nck; e += 32) {
            const int r = e / nck, t = e - r * nck;
            const int32_t id = __shfl_sync(FULL, d.y, r);
            if (id >= 0) cpa16(sb + r * pitch + 16 * t, vbase + (size_t)id * a.st.stride + 16 * t);
          }
        }
      }
    };
    auto offs = [&](int2 d, uint64_t &tb, uint64_t &te) {
      tb = te = 0;
      if (M == M_JAC && d.x >= 0) {
        if (part) {
          const ulonglong2 r = sv.rng[d.y];
          tb = r.x;
          te = r.y;
        } else {
          tb = a.st.off[d.y];
          te = a.st.off[d.y + 1];
        }
      }
    };
    // keys of staged rows (lane r: slot r; lanes >= nrows read slot 0 and are masked by the callers)
    auto keys_of = [&](const uint8_t *stg, int nrows) -> uint32_t {
      if constexpr (csr_metric(M)) {
        return 0u;
      } else if constexpr (LF) {
        const int r = lane < nrows ? lane : 0;
        return lane_key<M, NCK>(qsm, stg + r * pitch, r, SWZ);
      } else {
        return Q.eval_smem(stg, pitch, nck);
      }
    };
    // next chunk's draws dnx (pool loaded; sets: offsets bnx / enx in flight) and dnx2 (pool loads in flight)
    int2 dnx = make_int2(-1, -1), dnx2 = make_int2(-1, -1);
    uint64_t bnx = 0, enx = 0;
    int2 infl = make_int2(-1, -1);               // ns2: the chunk whose rows are in flight
    if (budget > 0) {
      dnx = draw(0);
      if (M == M_JAC) offs(dnx, bnx, enx);
      dnx2 = draw(1);
      if (ns2) {   // prologue: chunk 0 goes out now, chunk 1 at the start of chunk 0
        issue(dnx, 0, 0);
        cp_async_commit();
        infl = dnx;
        dnx = dnx2;
        dnx2 = draw(2);
      }
    }
    // the window: the current chunk, lanes >= wpos not yet processed
    int32_t wl = -1, wnode = -1;
    uint32_t wkey = 0;
    bool wfr0 = false;                           // a valid draw, the first of its node in the chunk
    bool wev = false;                            // its node was evaluated before (E bit)
    int wpos = 32, wslot = -1;
    bool stop = false;

    while (!stop && c < budget) {
      // ------------------------------ restart ------------------------------
      if (wpos >= 32) {
        KPROF(const long long tq0 = clock64();)
        const uint64_t cb = bnx, ce = enx;
        uint32_t ew = 0;
        const uint8_t *cst = stage;              // this chunk's staged rows
        if (ns2) {
          // chunk ch's rows were issued a chunk ago into stage (ch & 1); chunk ch + 1 goes out now
          wl = infl.x;
          wnode = infl.y;
          cst = stage + (ch & 1) * 32 * pitch;
          issue_to(stage + ((ch + 1) & 1) * 32 * pitch, dnx);
          cp_async_commit();
          infl = dnx;
          dnx = dnx2;
          dnx2 = draw(ch + 3);
          cp_async_wait<1>();
        } else {
          wl = dnx.x;
          wnode = dnx.y;
          ew = issue(dnx, cb, ce);
          // the next chunk's pool loads were issued a chunk ago (sets: its offsets now); the one after
          // next starts its pool loads
          dnx = dnx2;
          if (M == M_JAC) offs(dnx, bnx, enx);
          dnx2 = draw(ch + 2);
          if constexpr (BK != 0) bulk_wait(mbar, bph);
          cp_async_wait_all();
        }
        __syncwarp();
        wvec = (uint8_t *)cst;
        const bool ok = wl >= 0;
        if constexpr (KT != 0) {
          wkey = ok ? kt[wl] : 0u;
        } else if constexpr (str_metric(M)) {
          wkey = ok ? Q.key(sv, wnode) : 0u;
        } else if constexpr (M == M_JAC) {
          wkey = 0;
          if (ok) {
            const uint64_t a0 = cb & ~3ull;
            const int rb = (int)(cb - a0), re = (int)(ce - a0);
            if (((re + 3) >> 2) <= slotch) wkey = Q.eval_slot(stage + lane * pitch, rb, re);
            else wkey = Q.eval_slot_global(a.st.tok + a0, rb, re);
          }
        } else {
          wkey = keys_of(cst, 32);
        }
        KPROF(++c_chunks; const long long tq1 = clock64(); c_ph[3] += tq1 - tq0;)
        ++ch;
        const unsigned grp = __match_any_sync(FULL, wl);
        wfr0 = ok && !(grp & lanemask_lt());
        wev = es ? (ok && e_smem_test(wl)) : (ew & e_bit(wl)) != 0;
        wpos = 0;
        wslot = -1;
        // ---- fast path: no fresh draw of the chunk can be accepted against the current s_max: every
        // fresh draw is evaluated once and skipped (so none is a new best and the threshold cannot
        // move), exactly as the sequential loop does draw by draw; the budget is not reached.
        const bool fr = wfr0 && !wev;
        const unsigned fm = __ballot_sync(FULL, fr);
        const unsigned inv = __ballot_sync(FULL, !ok);
        thr_update();
        if (top.cnt > 0 && inv == 0 && c + __popc(fm) <= budget && !__any_sync(FULL, fr && !thr.skip(wkey))) {
          KPROF(const long long tq2 = clock64(); c_ph[4] += tq2 - tq1;)
          if (fr && !dsk) e_set(wl);
          top.insert(fr, wkey, wnode);             // Q5: skipped starts enter the top-k
          const int nf = __popc(fm);
          c += nf;
          s_starts += nf;
          s_skip += nf;
          wpos = 32;
          KPROF(++c_fast;)
          __syncwarp();
          KPROF(c_ph[5] += clock64() - tq2;)
          continue;
        }
        KPROF(++c_win;)
        // prefetch the rows of the draws that could still be accepted (the skip threshold only tightens
        // as s_max improves, so "passes against the current best" is a superset)
        if (a.win_prefetch) {
          const bool cand = fr && (top.cnt == 0 ? lane == __ffs(fm) - 1 : !thr.skip(wkey));
          const unsigned cmk = __ballot_sync(FULL, cand);
          const int r = __popc(cmk & lanemask_lt());
          if (cand && r < WPF) {
            wslot = r;
            const uint8_t *src = (const uint8_t *)rbase + (size_t)wnode * RB;
            const int CU = (RB % 16 == 0) ? 16 : ((RB % 8 == 0) ? 8 : 4);
            for (int u = 0; u < RB; u += CU) cpa_n(smem_u32(wrow) + r * RB + u, src + u, CU);
          }
        }
      }
      const unsigned active = FULL << wpos;
      const bool wvalid = wl >= 0;
      const unsigned invm = __ballot_sync(FULL, !wvalid) & active;
      const unsigned lim = invm ? ((1u << (__ffs(invm) - 1)) - 1u) : FULL;
      // Redraws are free (Q4): a draw of a node evaluated before (E) or drawn by a lower lane
      const bool fresh = lane >= wpos && wvalid && wfr0 && !wev;
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
      if (cmt && !dsk) e_set(wl);
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
      const int64_t jw = (ch - 1) * 32 + al;   // (dsk) the accepted start's draw position: every draw up to it is processed

      // ------------------- hill climbing, eager first improvement -------------------
      // One memory round trip per step: the vectors (lane-form widths) and E / X words of cur's in-pool
      // neighbours are copied together (row_pf: with their rows, so the next step's row is in shared
      // memory; else the chosen neighbour's row is loaded into registers as soon as the move is known).
      // The walk's evaluations reach the top-k in batches (pbuf, flushed at the walk's end).
      int32_t cur = __shfl_sync(FULL, wnode, al);
      uint32_t kcur = __shfl_sync(FULL, wkey, al);
      int32_t curl = __shfl_sync(FULL, wl, al);
      int rs = -1;                               // cur's row in rowbuf slot rs (row_pf)
      int rw = __shfl_sync(FULL, wslot, al);     // ... or in window slot rw
      bool have_nr = false;                      // ... or in nr (loaded after the move)
      int32_t nr = -1;
      int pn = 0;
      auto flush = [&]() {
        if (pn == 0) return;
        __syncwarp();
        const bool has = lane < pn;
        top.insert(has, has ? pkey[lane] : 0u, has ? pid[lane] : -1);
        pn = 0;
        __syncwarp();
      };
      if (rw >= 0) {
        cp_async_wait_all();
        __syncwarp();
      }
      KPROF(const long long tk0 = clock64();)
      for (;;) {
        KPROF(++c_steps; long long ts0 = clock64();)
        ++s_exp;
        if (lane == 0) {                         // cur is expanded (Q9 bookkeeping)
          if (xs) atomicOr(xbits + (curl >> 5), 1u << (curl & 31));
          else g_red_or(planes + pw(curl), x_bit(curl));
        }
        int32_t v = -1, vl = -1;
        if (lane < k) {
          int32_t e2;
          if (rw >= 0) e2 = ((const int32_t *)(wrow + rw * RB))[lane];
          else if (rs >= 0) e2 = ((const int32_t *)(rowbuf + rs * RB))[lane];
          else if (have_nr) e2 = nr;
          else e2 = KT ? rbase[(size_t)cur * k + lane] : __ldg(rbase + (size_t)cur * k + lane);
          v = e2;
          vl = e2;
        }
        rw = -1;
        // Q10: neighbours in another partition are skipped (prow holds -1 for them)
        const bool inpool = v >= 0 && vl >= 0;
        const int32_t lv = inpool ? vl : 0;
        __syncwarp();                            // rowbuf read before the copies below overwrite it
        KPROF(long long ts1 = clock64(); c_ph[0] += ts1 - ts0;)
        // issue: the vectors (lane-form widths), rows (row_pf) and E / X words of the in-pool neighbours
        if constexpr (KT != 0) {
          // keys from the table
        } else if constexpr (LF) {
          if constexpr (BK != 0) gather_bulk<NCK>(smem_u32(wvec), pitch, vbase, inpool ? v : -1, k, mbar);
          else gather_lf<NCK>(smem_u32(wvec), pitch, vbase, inpool ? v : -1, k);
          if (row_pf) {
            const unsigned rb0 = smem_u32(rowbuf);
            const int CU = (RB % 16 == 0) ? 16 : ((RB % 8 == 0) ? 8 : 4), NU = RB / CU;
            const uint8_t *rsrc = (const uint8_t *)rbase;
            for (int e0 = 0; e0 < k * NU; e0 += 32) {
              const int e = e0 + lane, t = e / NU, u = e - t * NU;
              const int32_t vt = __shfl_sync(FULL, inpool ? v : -1, t & 31);
              if (e < k * NU && vt >= 0) cpa_n(rb0 + t * RB + u * CU, rsrc + (size_t)vt * RB + u * CU, CU);
            }
          }
        } else if (row_pf) {
          const unsigned rb0 = smem_u32(rowbuf);
          const int CU = (RB % 16 == 0) ? 16 : ((RB % 8 == 0) ? 8 : 4), NU = RB / CU;
          const uint8_t *rsrc = (const uint8_t *)rbase;
          for (int t0 = 0; t0 < k; t0 += 16) {
            const int t = t0 + (lane & 15);
            const int32_t vt = __shfl_sync(FULL, inpool ? v : -1, t & 31);
            if (t < k && vt >= 0)
              for (int u = lane >> 4; u < NU; u += 2) cpa_n(rb0 + t * RB + u * CU, rsrc + (size_t)vt * RB + u * CU, CU);
          }
        }
        const uint32_t xw = (inpool && !xs) ? g_ld(planes + pw(lv)) : 0u;
        uint32_t key;
        if constexpr (KT != 0) {
          key = inpool ? kt[lv] : 0u;
        } else if constexpr (LF) {
          if constexpr (BK != 0) bulk_wait(mbar, bph);
          cp_async_wait_all();
          __syncwarp();
          key = keys_of(wvec, k);
        } else {
          key = Q.eval(sv, inpool ? v : -1, k);
          cp_async_wait_all();
          __syncwarp();
        }
        bool evb2 = !inpool || (es ? e_smem_test(lv) : (xw & e_bit(lv)) != 0);
        if (dsk && !evb2) {   // drawn before: its draw position is at most the accepted start's
          Perm pm;
          pm.init(h3, (uint64_t)m);
          evb2 = (int64_t)pm.pos((uint32_t)lv) <= jw;
        }
        const bool imp = inpool && closer<M>(key, kcur);
        KPROF(long long ts2 = clock64(); c_ph[1] += ts2 - ts1;)
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
        const bool mv_x = __shfl_sync(FULL, xs ? (inpool && ((xbits[lv >> 5] >> (lv & 31)) & 1u)) : (xw & x_bit(lv)) != 0, fi);
        // the move (if any) is known: its row is loaded now, under the bookkeeping below
        const int32_t ncur = __shfl_sync(FULL, v, fi);
        if (!row_pf && im && !mv_x && lane < k)
          nr = KT ? rbase[(size_t)ncur * k + lane] : __ldg(rbase + (size_t)ncur * k + lane);
        unsigned fm2 = __ballot_sync(FULL, !evb2) & range;
        bool hit2 = false;
        if ((int64_t)__popc(fm2) > budget - c) { fm2 = first_bits(fm2, (int)(budget - c)); hit2 = true; }
        const bool cm2 = (fm2 >> lane) & 1u;
        const int nf2 = __popc(fm2);
        if (cm2) {
          e_set(lv);
          if (dsk) wflt_set(wflt, lv);
        }
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
        if (mv_x) break;                     // Q9: moving onto an expanded node restarts
        cur = ncur;
        kcur = __shfl_sync(FULL, key, fi);
        curl = __shfl_sync(FULL, lv, fi);
        if (row_pf) rs = fi;
        else have_nr = true;
      }
      flush();
      KPROF(c_walk += clock64() - tk0;)
      // the walk may have evaluated nodes the rest of the window drew: re-read their E bits
      if (!stop && wpos < 32) {
        const bool need = lane >= wpos && wfr0 && !wev;
        if (__any_sync(FULL, need)) {
          if (es) {
            if (need) wev = e_smem_test(wl);
          } else {
            const uint32_t ew = need ? g_ld(planes + pw(wl)) : 0u;
            if (need) wev = (ew & e_bit(wl)) != 0;
          }
        }
      }
    }
    KPROF(if (a.prof && lane == 0) {
      auto put = [&](int i, unsigned long long v) { atomicAdd(a.prof + i, v); };
      put(0, (unsigned long long)(clock64() - tc0));
      put(2, (unsigned long long)c_walk);
      put(5, c_win);
      put(6, c_steps);
      put(8, c_fast);
      put(9, c_chunks);
      for (int i = 0; i < 6; ++i) put(10 + i, (unsigned long long)c_ph[i]);
    })
    s_evals += c;
    if (lane < a.kr) {
      const size_t o = ((size_t)b * Pn + pl) * a.kr + lane;
      a.out_ids[o] = lane < top.cnt ? (part ? a.members[pbase + top.id] : top.id) : -1;
      a.out_keys[o] = lane < top.cnt ? top.key : 0u;
    }
    cp_async_wait_all();
    __syncwarp();
    task = *(volatile long long *)(sched + warp);
    __syncwarp();
  }
  if (a.fuse) {   // B = 1: one CTA, warp 0 ran the only task; it runs the insert's update
    if (gw == 0) {
      uint8_t *us = smem + (size_t)WPC * a.wbytes + 16 * WPC;
      int32_t *usm = (int32_t *)(us + 16);
      uint32_t *uq = (uint32_t *)(us + 16 + update_one_smem(a.ub.hcap, a.ub.ballmax));
      BallArgs ub = a.ub;
      ub.n_t = n_t;
      int nb = 0, np = 0;
      update_one_warp<M, L, CPL>(ub, a.out_ids, a.out_keys, usm, (int *)us, csr_metric(M) ? uq : nullptr, &nb, &np, kt,
                                 M == M_JW ? jwp : nullptr, srw);
      s_ball += (unsigned)nb;
      s_prop += (unsigned)np;
    }
    if constexpr (KT != 0) {   // the other warps stage the next insert's key-table row meanwhile
      if (threadIdx.x >= 32 && it + 1 < nseq) stage_kt(it + 1, 32, (int)blockDim.x - 32);
    }
    __syncthreads();   // the insert's rows (global) before the next insert's search and key table
  }
  }   // sequential inserts
  if (a.fuse) {   // the fused launch owns the stats (no memset before it)
    if (gw == 0 && lane == 0) {
      a.stats[0] = s_evals;
      a.stats[1] = s_starts;
      a.stats[2] = s_skip;
      a.stats[3] = s_exp;
      a.stats[4] = s_ball;
      a.stats[5] = s_prop;
    }
    return;
  }
  if (lane == 0) {
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

// shared memory of one warp of K1 (the kernel's carve-up above)
size_t search_warp_bytes(const SearchArgs &a, bool sets) {
  const size_t RB = (size_t)4 * a.k;
  const bool ns2 = !sets && a.e_smem && a.ns2;
  size_t b = (size_t)(ns2 ? 64 : 32) * a.pitch + (a.row_pf ? ((a.k * RB + 15) & ~(size_t)15) : 0) +
             ((WPF * RB + 15) & ~(size_t)15) + 512 + 2 * 32 * 4 + (sets ? QSCR * 4 : 0) +
             (a.metric == M_JW ? 32 * JW_PTR : 0) +
             (a.e_smem ? (size_t)a.e_bytes * ((a.x_smem || a.kt) ? 2 : 1) : 0) +
             (!a.e_smem && a.perm_e ? (size_t)WFLT_WORDS * 4 : 0);
  return (b + 15) & ~(size_t)15;
}
size_t search_smem_bytes(const SearchArgs &a, bool sets) {
  return WPC * search_warp_bytes(a, sets) + 16 * WPC + fuse_bytes(a, sets) +
         (a.kt ? 2 * (((a.n_t + (a.fuse ? a.nseq : 0)) * 4 + 15) & ~15ll) : 0) +
         (a.kt && a.srows ? (((a.n_t + (a.fuse ? a.nseq : 0)) * a.k * 4 + 15) & ~15ll) : 0);
}

// occupancy of a K1 instantiation at a shared-memory size on the current device, cached (a B = 1 insert
// launches K1 once per point: the attribute / occupancy queries would otherwise dominate its host time)
template <int M, int L, int CPL, int MB, int NCK, int PART, int KT, int BK>
static cudaError_t k1_occupancy(size_t smem, int *per_sm, int *nsm) {
  static std::mutex mu;
  static std::map<std::pair<int, size_t>, std::pair<int, int>> cache;
  static std::map<int, size_t> attr;   // per device: the opt-in shared memory size set so far (only grows, so
                                       // that every cached size stays launchable)
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  static std::map<int, int> optin;
  if (!optin.count(dev)) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    optin[dev] = v;
  }
  // a plan that does not fit is refused here, without an API error (cudaGetLastError would report a
  // failed attribute call at the next launch)
  if (smem > (size_t)optin[dev]) return cudaErrorInvalidValue;
  if (smem > 48 * 1024 && smem > attr[dev]) {
    cudaError_t e = cudaFuncSetAttribute(k_search<M, L, CPL, MB, NCK, PART, KT, BK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return e;
    }
    attr[dev] = smem;
  }
  auto it = cache.find({dev, smem});
  if (it != cache.end()) {
    *per_sm = it->second.first;
    *nsm = it->second.second;
    return cudaSuccess;
  }
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(per_sm, k_search<M, L, CPL, MB, NCK, PART, KT, BK>, 32 * WPC, smem);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return e;
  }
  *nsm = 148;
  cudaDeviceGetAttribute(nsm, cudaDevAttrMultiProcessorCount, dev);
  cache[{dev, smem}] = {*per_sm, *nsm};
  return cudaSuccess;
}

template <int M, int L, int CPL, int MB, int NCK, int PART, int KT, int BK>
static cudaError_t run_search(SearchArgs a, cudaStream_t s) {
  const int Pn = a.part_cnt;
  const int64_t T = a.nq * Pn;
  if (T == 0) return cudaSuccess;
  a.wbytes = (int)search_warp_bytes(a, csr_metric(M));
  const size_t smem = search_smem_bytes(a, csr_metric(M));
  // persistent grid: the CTAs that fit at once (dynamic task scheduling balances the tail)
  int per_sm = 0, nsm = 148;
  if (cudaError_t oe = k1_occupancy<M, L, CPL, MB, NCK, PART, KT, BK>(smem, &per_sm, &nsm)) return oe;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  int64_t blocks = std::min<int64_t>((T + WPC - 1) / WPC, (int64_t)per_sm * nsm);
  blocks = std::min<int64_t>(blocks, a.gslots / WPC);
  if (const char *e = getenv("KNNG_GRID")) blocks = std::max<int64_t>(1, std::min<int64_t>(blocks, atoll(e)));   // measurement
  if (T > blocks * WPC) {   // the dynamic task counter is only read when there are more tasks than warps
    cudaError_t me = cudaMemsetAsync(a.task_ctr, 0, sizeof(unsigned long long), s);
    if (me != cudaSuccess) return me;
  }
  if (getenv("KNNG_PROFILE"))
    fprintf(stderr, "KNNG_PROFILE k_search: %lld CTAs x %d warps, %d CTAs per SM resident (%zu B smem each)\n",
            (long long)blocks, WPC, per_sm, smem);
  k_search<M, L, CPL, MB, NCK, PART, KT, BK><<<(unsigned)blocks, 32 * WPC, smem, s>>>(a);
  return cudaGetLastError();
}

#define KNNG_SHAPES(X, M) \
  X(M, 1, 1) X(M, 2, 1) X(M, 4, 1) X(M, 8, 1) X(M, 16, 1) X(M, 32, 1) X(M, 32, 2) X(M, 32, 4)
// fp32 rows of <= 32 chunks: 4 chunks per lane at most, partials in-lane (see VecQuery::reduce)
#define KNNG_SHAPES_F32(X) \
  X(M_F32, 1, 1) X(M_F32, 1, 2) X(M_F32, 1, 3) X(M_F32, 1, 4) X(M_F32, 2, 3) X(M_F32, 2, 4) X(M_F32, 4, 3) \
  X(M_F32, 4, 4) X(M_F32, 8, 3) X(M_F32, 8, 4) X(M_F32, 32, 2) X(M_F32, 32, 4)

// the lane-form widths with their geometry at compile time (search_lane_form)
#define KNNG_LF_SHAPES(X) X(M_U8, 8, 1, 8) X(M_U8, 2, 1, 2) X(M_F32, 8, 3, 24)

bool search_lane_form(const VecGeom &g, int lane_eval) {
  return lane_eval && !csr_metric(g.metric) && lane_eval_ok(g.metric, g.nchunks);
}

cudaError_t launch_search(const VecGeom &g, const SearchArgs &a, cudaStream_t s, int *n_launch) {
  if (n_launch) ++*n_launch;
  if (a.kt) {
#define X(MM, LL, CC) \
  if (g.metric == MM && g.L == LL && g.CPL == CC) return run_search<MM, LL, CC, KNNG_K1_MB, 0, 0, 1, 0>(a, s);
    KNNG_SHAPES(X, M_U8)
    KNNG_SHAPES_F32(X)
    X(M_JAC, 8, 1)
    X(M_JW, 8, 1)
    X(M_COS, 8, 1)
#undef X
    return cudaErrorInvalidValue;
  }
  if (search_lane_form(g, a.lane_eval)) {
#define X(MM, LL, CC, NN) \
  if (g.metric == MM && g.nchunks == NN) \
    return a.bulk ? (a.P > 0 ? run_search<MM, LL, CC, KNNG_K1_MB, NN, 1, 0, 1>(a, s) \
                             : run_search<MM, LL, CC, KNNG_K1_MB, NN, 0, 0, 1>(a, s)) \
                  : (a.P > 0 ? run_search<MM, LL, CC, KNNG_K1_MB, NN, 1, 0, 0>(a, s) \
                             : run_search<MM, LL, CC, KNNG_K1_MB, NN, 0, 0, 0>(a, s));
    KNNG_LF_SHAPES(X)
#undef X
  }
#define X(MM, LL, CC) \
  if (g.metric == MM && g.L == LL && g.CPL == CC) return run_search<MM, LL, CC, KNNG_K1_MB, 0, -1, 0, 0>(a, s);
  KNNG_SHAPES(X, M_U8)
  KNNG_SHAPES_F32(X)
  X(M_JAC, 8, 1)
  X(M_JW, 8, 1)
  X(M_COS, 8, 1)
#undef X
  return cudaErrorInvalidValue;
}

template <int M, int L, int CPL, int MB, int NCK, int PART, int KT, int BK>
static cudaError_t resident(SearchArgs a, int64_t *warps) {
  const size_t smem = search_smem_bytes(a, csr_metric(M));
  int per_sm = 0, nsm = 148;
  if (cudaError_t e = k1_occupancy<M, L, CPL, MB, NCK, PART, KT, BK>(smem, &per_sm, &nsm)) return e;
  *warps = (int64_t)per_sm * nsm * WPC;
  return cudaSuccess;
}

cudaError_t search_resident_warps(const VecGeom &g, const SearchArgs &a, int64_t *warps) {
  if (a.kt) {
#define X(MM, LL, CC) \
  if (g.metric == MM && g.L == LL && g.CPL == CC) return resident<MM, LL, CC, KNNG_K1_MB, 0, 0, 1, 0>(a, warps);
    KNNG_SHAPES(X, M_U8)
    KNNG_SHAPES_F32(X)
    X(M_JAC, 8, 1)
    X(M_JW, 8, 1)
    X(M_COS, 8, 1)
#undef X
    return cudaErrorInvalidValue;
  }
  if (search_lane_form(g, a.lane_eval)) {
#define X(MM, LL, CC, NN) \
  if (g.metric == MM && g.nchunks == NN) \
    return a.bulk ? (a.P > 0 ? resident<MM, LL, CC, KNNG_K1_MB, NN, 1, 0, 1>(a, warps) \
                             : resident<MM, LL, CC, KNNG_K1_MB, NN, 0, 0, 1>(a, warps)) \
                  : (a.P > 0 ? resident<MM, LL, CC, KNNG_K1_MB, NN, 1, 0, 0>(a, warps) \
                             : resident<MM, LL, CC, KNNG_K1_MB, NN, 0, 0, 0>(a, warps));
    KNNG_LF_SHAPES(X)
#undef X
  }
#define X(MM, LL, CC) \
  if (g.metric == MM && g.L == LL && g.CPL == CC) return resident<MM, LL, CC, KNNG_K1_MB, 0, -1, 0, 0>(a, warps);
  KNNG_SHAPES(X, M_U8)
  KNNG_SHAPES_F32(X)
  X(M_JAC, 8, 1)
  X(M_JW, 8, 1)
  X(M_COS, 8, 1)
#undef X
  return cudaErrorInvalidValue;
}

cudaError_t launch_merge_parts(int metric, const int32_t *ci, const uint32_t *ck, int64_t nq, int P, int world, int kr,
                               int32_t *oi, uint32_t *ok, cudaStream_t s) {
  if (nq == 0) return cudaSuccess;
  const unsigned blocks = (unsigned)((nq + 3) / 4);
  if (metric == M_U8) k_merge_parts<M_U8><<<blocks, 128, 0, s>>>(ci, ck, nq, P, world, kr, oi, ok);
  else if (metric == M_F32) k_merge_parts<M_F32><<<blocks, 128, 0, s>>>(ci, ck, nq, P, world, kr, oi, ok);
  else if (metric == M_JAC) k_merge_parts<M_JAC><<<blocks, 128, 0, s>>>(ci, ck, nq, P, world, kr, oi, ok);
  else if (metric == M_JW) k_merge_parts<M_JW><<<blocks, 128, 0, s>>>(ci, ck, nq, P, world, kr, oi, ok);
  else k_merge_parts<M_COS><<<blocks, 128, 0, s>>>(ci, ck, nq, P, world, kr, oi, ok);
  return cudaGetLastError();
}

}  // namespace knng
