// knng_common.cuh -- device building blocks of the B200 path (sm_100a).
//
// Product code: shares nothing with oracle/.  "P:n" = line n of the paper
// (PAPER.md); "Qn" = reading n in DESIGN.md.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace knng {

constexpr unsigned FULL = 0xFFFFFFFFu;
enum { M_U8 = 0, M_F32 = 1, M_JAC = 2, M_JW = 3, M_COS = 4 };
// points held as uint32 sequences in CSR form (token sets; strings of characters)
__host__ __device__ constexpr bool csr_metric(int m) { return m >= M_JAC; }
// strings: Jaro-Winkler, cosine of 2-gram count vectors
__host__ __device__ constexpr bool str_metric(int m) { return m == M_JW || m == M_COS; }
constexpr int STR_MAX = 127;   // characters per string (the keys pack lengths / counts in 7 / 16 bits)

// Jaro-Winkler key m | T << 7 | l << 14 | |a| << 17 | |b| << 24 as the exact fraction num / den:
// jaro = (2m^2|b| + 2m^2|a| + (2m - T)|a||b|) / (6|a||b|m), jw = ((10 - l) jaro + l) / 10 (0 when m = 0).
__host__ __device__ __forceinline__ void jw_frac(uint32_t key, uint64_t &num, uint64_t &den) {
  const uint64_t m = key & 127u, T = (key >> 7) & 127u, l = (key >> 14) & 7u, la = (key >> 17) & 127u,
                 lb = (key >> 24) & 127u;
  if (m == 0) { num = 0; den = 1; return; }
  const uint64_t d0 = 6 * la * lb * m;
  num = (10 - l) * (2 * m * m * (la + lb) + (2 * m - T) * la * lb) + l * d0;
  den = 10 * d0;
}

// ---------------------------------------------------------------------------
// Counter RNG of the random starts (Q4): SplitMix64 finaliser chain keyed by
// (seed, point id, partition, draw #); pool index = floor(h * m / 2^64).
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
constexpr uint64_t GOLDEN = 0x9E3779B97F4A7C15ull;

__host__ __device__ __forceinline__ uint64_t rng_prefix(uint64_t seed, uint64_t pid, uint64_t part) {
  uint64_t h = mix64(seed + 1ull * GOLDEN);
  h = mix64(h ^ (pid + 2ull * GOLDEN));
  return mix64(h ^ (part + 3ull * GOLDEN));
}
__device__ __forceinline__ uint64_t rng_index(uint64_t prefix, uint64_t draw, uint64_t m) {
  return __umul64hi(mix64(prefix ^ (draw + 4ull * GOLDEN)), m);
}

// Restart draws of a search (Q4, round 2): a pseudo-random permutation pi of the pool, so the draws of
// one search never repeat each other.  6-round unbalanced Feistel network on b = max(6, ceil(log2 m))
// bits (halves hl = b / 2 high, hr = b - hl low, swapping widths every round; round key i =
// (uint32)(prefix >> 16 (i mod 4)) ^ 0x9E3779B9 (i + 1); round function lowbias32), cycle-walked into
// [0, m).  Its inverse gives the draw position of a pool node, so a node's "drawn before" bit needs no
// memory: pi^-1(v) <= the last draw processed.
__device__ __forceinline__ uint32_t lowbias32(uint32_t z) {
  z ^= z >> 16;
  z *= 0x7feb352du;
  z ^= z >> 15;
  z *= 0x846ca68bu;
  return z ^ (z >> 16);
}
struct Perm {
  uint64_t pre;
  uint32_t m;
  int hl, hr;
  __device__ __forceinline__ void init(uint64_t prefix, uint64_t m_) {
    pre = prefix;
    m = (uint32_t)m_;
    int b = m_ > 1 ? 32 - __clz((unsigned)(m_ - 1)) : 0;
    if (b < 6) b = 6;
    hl = b >> 1;
    hr = b - hl;
  }
  __device__ __forceinline__ uint32_t key(int i) const {
    return (uint32_t)(pre >> (16 * (i & 3))) ^ (0x9E3779B9u * (uint32_t)(i + 1));
  }
  __device__ __forceinline__ uint32_t fwd(uint32_t x) const {
    uint32_t L = x >> hr, R = x & ((1u << hr) - 1u);
    int la = hl, ra = hr;
#pragma unroll
    for (int i = 0; i < 6; ++i) {
      const uint32_t nR = L ^ (lowbias32(R ^ key(i)) & ((1u << la) - 1u));
      L = R;
      R = nR;
      const int t = la;
      la = ra;
      ra = t;
    }
    return (L << ra) | R;
  }
  __device__ __forceinline__ uint32_t inv(uint32_t y) const {
    uint32_t L = y >> hr, R = y & ((1u << hr) - 1u);
    int la = hl, ra = hr;
#pragma unroll
    for (int i = 5; i >= 0; --i) {
      const uint32_t R0 = L;
      const uint32_t L0 = R ^ (lowbias32(R0 ^ key(i)) & ((1u << ra) - 1u));
      L = L0;
      R = R0;
      const int t = la;
      la = ra;
      ra = t;
    }
    return (L << ra) | R;
  }
  // draw j (-1 past the pool)
  __device__ __forceinline__ int32_t draw(int64_t j) const {
    if (j >= (int64_t)m) return -1;
    uint32_t x = (uint32_t)j;
    do { x = fwd(x); } while (x >= m);
    return (int32_t)x;
  }
  // the draw position of pool node v (< m)
  __device__ __forceinline__ uint32_t pos(uint32_t v) const {
    uint32_t y = v;
    do { y = inv(y); } while (y >= m);
    return y;
  }
};

// ---------------------------------------------------------------------------
// Key order.  U8: uint32 D; F32: fp32 D bits; JAC: (inter<<16)|union.
// closer(a,b): a strictly more similar than b (metric value only).
// precedes: edge order (closer first, equal similarity -> smaller id).
// ---------------------------------------------------------------------------
template <int M>
__device__ __forceinline__ bool closer(uint32_t a, uint32_t b) {
  if (M == M_U8) return a < b;
  if (M == M_F32) return __uint_as_float(a) < __uint_as_float(b);
  if (M == M_JW) {   // jw_a > jw_b (num, den < 2^31: products < 2^62)
    uint64_t na, da, nb, db;
    jw_frac(a, na, da);
    jw_frac(b, nb, db);
    return na * db > nb * da;
  }
  if (M == M_COS) {  // dot_a / |x_a| > dot_b / |x_b| (the row owner's norm is common), squared
    const uint64_t xa = a >> 16, xb = b >> 16;
    return xa * xa * (b & 0xFFFFu) > xb * xb * (a & 0xFFFFu);
  }
  return (uint64_t)(a >> 16) * (b & 0xFFFFu) > (uint64_t)(b >> 16) * (a & 0xFFFFu);
}
template <int M>
__device__ __forceinline__ bool precedes(uint32_t ka, int32_t ia, uint32_t kb, int32_t ib) {
  if (closer<M>(ka, kb)) return true;
  if (closer<M>(kb, ka)) return false;
  return ia < ib;
}
// Expansion rule of P:81 with e = num/den (den = 0: e = +inf).  Q1: s = 1/(1+D) for the L2
// metrics, s = i/u for Jaccard; skip iff s_r < s_max / e, decided exactly.
template <int M>
__device__ __forceinline__ bool skip_start(uint32_t kr, uint32_t kb, uint64_t num, uint64_t den) {
  if (den == 0) return false;
  if (M == M_U8) return den * (1ull + kr) > num * (1ull + kb);
  if (M == M_F32) {
    const double l = __dmul_rn((double)den, __dadd_rn(1.0, (double)__uint_as_float(kr)));
    const double r = __dmul_rn((double)num, __dadd_rn(1.0, (double)__uint_as_float(kb)));
    return l > r;
  }
  if (M == M_JW) {   // num jw_r < den jw_best, as fractions (128-bit products)
    uint64_t nr, dr, nb, db;
    jw_frac(kr, nr, dr);
    jw_frac(kb, nb, db);
    return (unsigned __int128)(num * nr) * db < (unsigned __int128)(den * nb) * dr;
  }
  if (M == M_COS) {  // num cos_r < den cos_best  <=>  num^2 dot_r^2 |x_b|^2 < den^2 dot_b^2 |x_r|^2
    const uint64_t dr = kr >> 16, db = kb >> 16;
    return (unsigned __int128)(num * num) * (dr * dr * (kb & 0xFFFFu)) <
           (unsigned __int128)(den * den) * (db * db * (kr & 0xFFFFu));
  }
  return num * (uint64_t)(kr >> 16) * (uint64_t)(kb & 0xFFFFu) <
         den * (uint64_t)(kb >> 16) * (uint64_t)(kr & 0xFFFFu);
}

// The same rule against a fixed s_max, prepared once per change of the best key: a u8 test becomes
// one compare (den(1+D_r) > num(1+D_b)  <=>  D_r >= floor(num(1+D_b)/den); the floor is one fp64
// division rounded toward zero, exact while num(1+D_b) < 2^53, else an integer division); the f32 and
// Jaccard forms keep exactly the operations of skip_start.
template <int M>
struct SkipThr {
  uint64_t t, A, Bv;
  double rhs;
  uint64_t den, num;
  uint32_t kb_;
  __device__ __forceinline__ void set(uint32_t kb, uint64_t num_, uint64_t den_) {
    den = den_;
    num = num_;
    kb_ = kb;
    const uint64_t num = num_;
    if (den == 0) return;
    if (M == M_U8) {
      const uint64_t x = num * (1ull + kb);
      t = x < (1ull << 53) ? (uint64_t)__ddiv_rz((double)x, (double)den) : x / den;
    }
    if (M == M_F32) rhs = __dmul_rn((double)num, __dadd_rn(1.0, (double)__uint_as_float(kb)));
    if (M == M_JAC) { A = num * (uint64_t)(kb & 0xFFFFu); Bv = den * (uint64_t)(kb >> 16); }
  }
  __device__ __forceinline__ bool skip(uint32_t kr) const {
    if (den == 0) return false;
    if (M == M_U8) return (uint64_t)kr >= t;
    if (M == M_F32) return __dmul_rn((double)den, __dadd_rn(1.0, (double)__uint_as_float(kr))) > rhs;
    if (str_metric(M)) return skip_start<M>(kr, kb_, num, den);
    return A * (uint64_t)(kr >> 16) < Bv * (uint64_t)(kr & 0xFFFFu);
  }
};

// ---------------------------------------------------------------------------
// Global memory helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint4 ldg16(const void *p) {
  uint4 r;
  asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ bool bit_get(const uint32_t *b, uint32_t i) {
  return (((const volatile uint32_t *)b)[i >> 5] >> (i & 31)) & 1u;
}
__device__ __forceinline__ void bit_set(uint32_t *b, uint32_t i) { atomicOr(b + (i >> 5), 1u << (i & 31)); }

// asynchronous 4-byte global -> shared copy (LDGSTS): the warp does not wait for the load
__device__ __forceinline__ void cp_async4(void *smem_dst, const void *gsrc) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
// asynchronous 16-byte global -> shared copy, L2 only (.cg): a staged gather holds no registers
__device__ __forceinline__ void cp_async16(void *smem_dst, const void *gsrc) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gsrc) : "memory");
}
// mbarrier (shared, CTA scope): the ring's "chunk published" signal without a memory fence
__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_inval(uint64_t *bar) {
  asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.release.cta.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t *bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
// mbarrier arrival that also expects tx bytes of asynchronous (bulk) copies in the current phase
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, unsigned tx) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(tx)
               : "memory");
}
// one bulk copy global -> shared (the TMA engine; UBLKCP), completing `bytes` on the mbarrier at bar
__device__ __forceinline__ void bulk_g2s(unsigned dst, const void *src, unsigned bytes, unsigned bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}
// the lowest n set bits of mask
__device__ __forceinline__ unsigned first_bits(unsigned mask, int n) {
  unsigned r = 0;
  for (int i = 0; i < n && mask; ++i) {
    const unsigned low = mask & (0u - mask);
    r |= low;
    mask ^= low;
  }
  return r;
}

// ---------------------------------------------------------------------------
// Warp-register top-k: lane j < cnt holds entry j, sorted by edge order.
// ---------------------------------------------------------------------------
template <int M>
struct WarpTopK {
  uint32_t key;
  int32_t id;
  int cnt, kr;
  uint32_t key_at0;   // warp-uniform copy of the best key (valid when cnt > 0)
  uint32_t wk_u;      // warp-uniform copy of the worst entry (valid when cnt == kr)
  int32_t wi_u;
  __device__ __forceinline__ void init(int kr_) {
    key = 0; id = -1; cnt = 0; kr = kr_; key_at0 = 0; wk_u = 0; wi_u = -1;
  }
  __device__ __forceinline__ uint32_t best() const { return __shfl_sync(FULL, key, 0); }
  // may an entry with key ck enter (some id)?  (lane-local; uses the cached worst entry)
  __device__ __forceinline__ bool could_take(uint32_t ck) const { return cnt < kr || !closer<M>(wk_u, ck); }
  // insert every lane with flag set (distinct ids assumed)
  __device__ __forceinline__ void insert(bool flag, uint32_t ck, int32_t cid) {
    const int lane = threadIdx.x & 31;
    if (cnt == kr) flag = flag && precedes<M>(ck, cid, wk_u, wi_u);   // pre-filter against the worst entry
    unsigned m = __ballot_sync(FULL, flag);
    if (!m) return;
    while (m) {
      const int src = __ffs(m) - 1;
      m &= m - 1;
      const uint32_t k2 = __shfl_sync(FULL, ck, src);
      const int32_t i2 = __shfl_sync(FULL, cid, src);
      const bool before = lane < cnt && precedes<M>(key, id, k2, i2);
      const int pos = __popc(__ballot_sync(FULL, before));
      if (pos >= kr) continue;
      const uint32_t uk = __shfl_up_sync(FULL, key, 1);
      const int32_t ui = __shfl_up_sync(FULL, id, 1);
      if (lane > pos) { key = uk; id = ui; }
      if (lane == pos) { key = k2; id = i2; }
      if (cnt < kr) ++cnt;
      if (pos == 0) key_at0 = k2;
    }
    if (cnt == kr) {
      wk_u = __shfl_sync(FULL, key, (kr - 1) & 31);
      wi_u = __shfl_sync(FULL, id, (kr - 1) & 31);
    }
  }
};

// ---------------------------------------------------------------------------
// Canonical squared distances (Q24).
//  Vectors are stored in rows of `stride` bytes = nchunks 16-byte chunks, zero padded.
//  U8 : exact int sum of (a-b)^2 (order irrelevant).
//  F32: 32 partial sums; chunk c -> partial c%32 via fmaf(d,d,acc) over its 4 floats
//       (chunks c, c+32, ... in increasing order); partials combined by the xor butterfly
//       16,8,4,2,1.  Warp form (below) and single-thread form (thread_dist) compute the
//       same tree; IEEE addition is commutative, and the absent partials are +0.
// ---------------------------------------------------------------------------
template <int M>
__device__ __forceinline__ void chunk_acc(uint32_t &acc, const uint4 &a, const uint4 &b);
template <>
__device__ __forceinline__ void chunk_acc<M_U8>(uint32_t &acc, const uint4 &a, const uint4 &b) {
  uint32_t d;
  d = __vabsdiffu4(a.x, b.x); acc = __dp4a(d, d, acc);
  d = __vabsdiffu4(a.y, b.y); acc = __dp4a(d, d, acc);
  d = __vabsdiffu4(a.z, b.z); acc = __dp4a(d, d, acc);
  d = __vabsdiffu4(a.w, b.w); acc = __dp4a(d, d, acc);
}
__device__ __forceinline__ float f4_leaf(float acc, const uint4 &a, const uint4 &b) {
  float d;
  d = __fsub_rn(__uint_as_float(a.x), __uint_as_float(b.x)); acc = __fmaf_rn(d, d, acc);
  d = __fsub_rn(__uint_as_float(a.y), __uint_as_float(b.y)); acc = __fmaf_rn(d, d, acc);
  d = __fsub_rn(__uint_as_float(a.z), __uint_as_float(b.z)); acc = __fmaf_rn(d, d, acc);
  d = __fsub_rn(__uint_as_float(a.w), __uint_as_float(b.w)); acc = __fmaf_rn(d, d, acc);
  return acc;
}

// Single-thread canonical distance between two rows (pointers to 16B chunks, any space).
template <int M>
__device__ __forceinline__ uint32_t thread_dist(const uint4 *a, const uint4 *b, int nchunks) {
  if (M == M_U8) {
    uint32_t acc = 0;
    for (int c = 0; c < nchunks; ++c) chunk_acc<M_U8>(acc, a[c], b[c]);
    return acc;
  } else {
    // leaves in butterfly order: leaf i holds partial bitrev5(i); a binary-counter stack
    // evaluates ((p0+p16)+(p8+p24)) + ... exactly as the warp butterfly does.
    float stk[6];
    int sp = 0;
#pragma unroll 1
    for (int i = 0; i < 32; ++i) {
      const int l = __brev(i) >> 27;
      float leaf = 0.0f;
      for (int c = l; c < nchunks; c += 32) leaf = f4_leaf(leaf, a[c], b[c]);
      stk[sp++] = leaf;
      for (int cnt = i + 1; (cnt & 1) == 0; cnt >>= 1) {
        stk[sp - 2] = __fadd_rn(stk[sp - 2], stk[sp - 1]);
        --sp;
      }
    }
    return __float_as_uint(stk[0]);
  }
}

// Where the points live: vector rows (stride bytes, zero padded) or Jaccard sets in CSR.
struct StoreView {
  const uint8_t *vec;
  size_t stride;
  int nchunks;
  const uint64_t *off;   // sets: [n+1]
  const uint32_t *tok;   // sets: sorted, unique tokens (16-byte aligned buffer, zeroed slack)
  int vwords;            // sets: words of a vocabulary bitmap covering every stored token (0: none)
  // sets, partition-local view (K1 on a partitioned graph): [begin, end) token range of local index i at
  // rng[i] (ids are then partition-local indices; off is not used), else null
  const ulonglong2 *rng = nullptr;
  // 2-gram cosine strings: |x|^2 = sum_g c_x(g)^2 of every stored string (>= 1), else null
  const uint32_t *n2 = nullptr;
};
constexpr int VOCAB_SMEM_WORDS = 8192;   // vocabulary bitmaps up to 2^18 token ids live in smem

// Single-thread Jaccard key of two sorted token lists: (|A n B| << 16) | |A u B|.
__device__ __forceinline__ uint32_t set_key(const uint32_t *a, int la, const uint32_t *b, int lb) {
  int i = 0, j = 0, inter = 0;
  while (i < la && j < lb) {
    const uint32_t x = a[i], y = b[j];
    inter += x == y;
    i += x <= y;
    j += y <= x;
  }
  return ((uint32_t)inter << 16) | (uint32_t)(la + lb - inter);
}

// Key of string b as an entry of string a's row (single thread; a: the row owner / query).
//  JW: matches in a's order, each a[i] taking the first free b[j] with |i - j| <= max(|a|,|b|)/2 - 1
//      (matched positions of a and b as pairs of 64-bit register masks); T = positions where the matched
//      characters of a and of b, each in order, differ (walked by find-first-set over the masks); l =
//      common prefix (<= 4).  Key m | T<<7 | l<<14 | |a|<<17 | |b|<<24.
//  COS: dot = pairs of equal 2-grams (a[i], a[i+1]) == (b[j], b[j+1]); key (dot << 16) | n2b, n2b =
//      |b|^2 of the count vector (>= 1).
template <int M>
__device__ __forceinline__ uint32_t str_key(const uint32_t *a, int la, const uint32_t *b, int lb, uint32_t n2b) {
  if (M == M_COS) {
    uint32_t dot = 0;
    for (int i = 0; i + 1 < la; ++i) {
      const uint32_t a0 = a[i], a1 = a[i + 1];
      uint32_t b0 = lb > 0 ? b[0] : 0u;
      for (int j = 0; j + 1 < lb; ++j) {
        const uint32_t b1 = b[j + 1];
        dot += (a0 == b0) & (a1 == b1);
        b0 = b1;
      }
    }
    return (dot << 16) | n2b;
  } else {
    int w = (la > lb ? la : lb) / 2 - 1;
    if (w < 0) w = 0;
    // matched positions as two 64-bit register masks each (strings <= 127 characters): no local memory
    uint64_t bm0 = 0, bm1 = 0;   // b positions matched
    uint64_t am0 = 0, am1 = 0;   // a positions matched
    int m = 0;
    for (int i = 0; i < la; ++i) {
      const uint32_t c = a[i];
      const int lo = i - w > 0 ? i - w : 0, hi = i + w < lb - 1 ? i + w : lb - 1;
      for (int j = lo; j <= hi; ++j) {
        const uint64_t bw = j < 64 ? bm0 : bm1;
        if (!((bw >> (j & 63)) & 1ull) && b[j] == c) {
          if (j < 64) bm0 |= 1ull << j;
          else bm1 |= 1ull << (j - 64);
          if (i < 64) am0 |= 1ull << i;
          else am1 |= 1ull << (i - 64);
          ++m;
          break;
        }
      }
    }
    // T: the r-th matched character of a against the r-th matched character of b
    int T = 0;
    uint64_t ra0 = am0, ra1 = am1, rb0 = bm0, rb1 = bm1;
    for (int r = 0; r < m; ++r) {
      const int i = ra0 ? __ffsll((long long)ra0) - 1 : 64 + __ffsll((long long)ra1) - 1;
      const int j = rb0 ? __ffsll((long long)rb0) - 1 : 64 + __ffsll((long long)rb1) - 1;
      if (ra0) ra0 &= ra0 - 1; else ra1 &= ra1 - 1;
      if (rb0) rb0 &= rb0 - 1; else rb1 &= rb1 - 1;
      T += a[i] != b[j];
    }
    int l = 0;
    while (l < 4 && l < la && l < lb && a[l] == b[l]) ++l;
    return (uint32_t)m | ((uint32_t)T << 7) | ((uint32_t)l << 14) | ((uint32_t)la << 17) | ((uint32_t)lb << 24);
  }
}

// Key of rows i and j of a store (single thread; i owns the row).
template <int M>
__device__ __forceinline__ uint32_t pair_key(const StoreView &s, int64_t i, int64_t j) {
  if (str_metric(M)) {
    const uint64_t ai = s.off[i], bj = s.off[j];
    return str_key<M>(s.tok + ai, (int)(s.off[i + 1] - ai), s.tok + bj, (int)(s.off[j + 1] - bj),
                      M == M_COS ? s.n2[j] : 0u);
  }
  if (M == M_JAC) {
    const uint64_t ai = s.off[i], bi = s.off[j];
    return set_key(s.tok + ai, (int)(s.off[i + 1] - ai), s.tok + bi, (int)(s.off[j + 1] - bi));
  }
  return thread_dist<M>((const uint4 *)(s.vec + (size_t)i * s.stride), (const uint4 *)(s.vec + (size_t)j * s.stride),
                        s.nchunks);
}

// Warp-cooperative evaluation of up to 32 candidates against a query held in registers.
// L lanes per vector (power of 2), CPL chunks per lane: lane sl of a group owns chunks
// sl, sl+L, ..., (CPL of them).  32/L vectors per pass; GRP passes have their loads in flight
// together.
template <int M, int L, int CPL>
struct VecQuery {
  static constexpr int VPP = 32 / L;
  // passes whose loads are in flight together: up to 8 x 16 B per lane, 16 for wide vectors (one
  // vector per pass, L = 32) so that a 32-candidate chunk needs 2 round trips, not 4
  static constexpr int LIM = (L == 32 && CPL == 1) ? 16 : (M == M_U8 && CPL == 1 ? 4 : 8);
  static constexpr int GRP = (L < (LIM / CPL) ? L : ((LIM / CPL) > 0 ? (LIM / CPL) : 1));
  uint4 q[CPL];

  __device__ __forceinline__ void load(const StoreView &s, int64_t r, uint32_t * /*scratch*/) {
    const uint8_t *row = s.vec + (size_t)r * s.stride;
    const int nchunks = s.nchunks;
    const int sl = (threadIdx.x & 31) % L;
#pragma unroll
    for (int t = 0; t < CPL; ++t) {
      const int c = sl + L * t;
      q[t] = c < nchunks ? ldg16(row + (size_t)c * 16) : make_uint4(0, 0, 0, 0);
    }
  }

  __device__ __forceinline__ uint32_t reduce(const uint4 *b) const {
    if (M == M_U8) {
      uint32_t acc = 0;
#pragma unroll
      for (int t = 0; t < CPL; ++t) chunk_acc<M_U8>(acc, q[t], b[t]);
#pragma unroll
      for (int o = L / 2; o >= 1; o >>= 1) acc += __shfl_xor_sync(FULL, acc, o);
      return acc;
    } else if (L == 32 || CPL == 1) {
      // chunks sl, sl+32, ... share partial sl: one fmaf chain in increasing chunk order (Q24)
      float acc = 0.0f;
#pragma unroll
      for (int t = 0; t < CPL; ++t) acc = f4_leaf(acc, q[t], b[t]);
#pragma unroll
      for (int o = L / 2; o >= 1; o >>= 1) acc = __fadd_rn(acc, __shfl_xor_sync(FULL, acc, o));
      return __float_as_uint(acc);
    } else {
      // L*CPL <= 32: chunk sl + L*t is its own partial (index sl + L*t).  The butterfly levels
      // o >= L pair partials held by the same lane (slots t and t + o/L; slots >= CPL are +0); the
      // levels o < L cross lanes.  Same tree as the 32-lane canonical order (Q24).
      float p[CPL];
#pragma unroll
      for (int t = 0; t < CPL; ++t) p[t] = f4_leaf(0.0f, q[t], b[t]);
#pragma unroll
      for (int o = 16; o >= L; o >>= 1) {
        const int st = o / L;
#pragma unroll
        for (int t = 0; t < CPL; ++t)
          if (t < st && t + st < CPL) p[t] = __fadd_rn(p[t], p[t + st]);
      }
      float acc = p[0];
#pragma unroll
      for (int o = L / 2; o >= 1; o >>= 1) acc = __fadd_rn(acc, __shfl_xor_sync(FULL, acc, o));
      return __float_as_uint(acc);
    }
  }

  // cand: id held by lane j for candidate j < n (id < 0: skipped, key undefined).
  // Returns the key of candidate j in lane j.
  __device__ __forceinline__ uint32_t eval(const StoreView &s, int32_t cand, int n) const {
    const uint8_t *__restrict__ base = s.vec;
    const size_t stride = s.stride;
    const int nchunks = s.nchunks;
    const int lane = threadIdx.x & 31, sub = lane / L, sl = lane % L;
    uint32_t out = 0;
    const int np = (n + VPP - 1) / VPP;
    for (int p0 = 0; p0 < np; p0 += GRP) {
      uint4 buf[GRP][CPL];
#pragma unroll
      for (int g = 0; g < GRP; ++g) {
        const int v = (p0 + g) * VPP + sub;
        const int32_t id = __shfl_sync(FULL, cand, v & 31);
        const bool ok = v < n && id >= 0;
#pragma unroll
        for (int t = 0; t < CPL; ++t) {
          const int c = sl + L * t;
          buf[g][t] = (ok && c < nchunks) ? ldg16(base + (size_t)id * stride + (size_t)c * 16)
                                          : make_uint4(0, 0, 0, 0);
        }
      }
#pragma unroll
      for (int g = 0; g < GRP; ++g) {
        if (p0 + g < np) {
          const uint32_t key = reduce(buf[g]);
          const uint32_t kk = __shfl_sync(FULL, key, (lane % VPP) * L);
          if (lane / VPP == p0 + g) out = kk;
        }
      }
    }
    return out;
  }

  // Keys of 32 candidates staged in shared memory (candidate j's row at sb + j * pitch, zero
  // beyond nchunks not required); lane j gets candidate j's key.  Same reduction tree (Q24).
  __device__ __forceinline__ uint32_t eval_smem(const uint8_t *sb, int pitch, int nchunks) const {
    const int lane = threadIdx.x & 31, sub = lane / L, sl = lane % L;
    constexpr int NP = 32 / VPP;
    constexpr int GW = (8 / CPL) > 0 ? (8 / CPL) : 1;
    constexpr int GS = NP < GW ? NP : (GW < 4 ? GW : 4);   // passes whose LDS are in flight together
    uint32_t out = 0;
#pragma unroll
    for (int p0 = 0; p0 < NP; p0 += GS) {
      uint4 buf[GS][CPL];
#pragma unroll
      for (int g = 0; g < GS; ++g) {
        const uint8_t *row = sb + ((p0 + g) * VPP + sub) * pitch;
#pragma unroll
        for (int t = 0; t < CPL; ++t) {
          const int c = sl + L * t;
          buf[g][t] = c < nchunks ? *(const uint4 *)(row + c * 16) : make_uint4(0, 0, 0, 0);
        }
      }
#pragma unroll
      for (int g = 0; g < GS; ++g) {
        const uint32_t key = reduce(buf[g]);
        const uint32_t kk = __shfl_sync(FULL, key, (lane % VPP) * L);
        if (lane / VPP == p0 + g) out = kk;
      }
    }
    return out;
  }

  // Two full sets of 32 candidates with both sets' loads in flight together (producer warps).
  __device__ __forceinline__ void eval2(const StoreView &s, int32_t ca, int32_t cb, uint32_t &oa, uint32_t &ob) const {
    const uint8_t *__restrict__ base = s.vec;
    const size_t stride = s.stride;
    const int nchunks = s.nchunks;
    const int lane = threadIdx.x & 31, sub = lane / L, sl = lane % L;
    constexpr int NP = 32 / VPP;     // passes per 32 candidates
    constexpr int G2 = (LIM == 16 && GRP > 1) ? GRP / 2 : GRP;   // per set (both sets together stay <= 16 loads)
    oa = 0;
    ob = 0;
    for (int p0 = 0; p0 < NP; p0 += G2) {
      uint4 ba[G2][CPL], bb[G2][CPL];
#pragma unroll
      for (int g = 0; g < G2; ++g) {
        const int v = (p0 + g) * VPP + sub;
        const int32_t ida = __shfl_sync(FULL, ca, v & 31);
        const int32_t idb = __shfl_sync(FULL, cb, v & 31);
        const bool ok = p0 + g < NP;
#pragma unroll
        for (int t = 0; t < CPL; ++t) {
          const int c = sl + L * t;
          const bool okc = ok && c < nchunks;
          ba[g][t] = (okc && ida >= 0) ? ldg16(base + (size_t)ida * stride + (size_t)c * 16) : make_uint4(0, 0, 0, 0);
          bb[g][t] = (okc && idb >= 0) ? ldg16(base + (size_t)idb * stride + (size_t)c * 16) : make_uint4(0, 0, 0, 0);
        }
      }
#pragma unroll
      for (int g = 0; g < G2; ++g) {
        if (p0 + g < NP) {
          const uint32_t ka = reduce(ba[g]);
          const uint32_t kb = reduce(bb[g]);
          const uint32_t xa = __shfl_sync(FULL, ka, (lane % VPP) * L);
          const uint32_t xb = __shfl_sync(FULL, kb, (lane % VPP) * L);
          if (lane / VPP == p0 + g) { oa = xa; ob = xb; }
        }
      }
    }
  }
};

// Jaccard sets.  The query's sorted tokens sit in shared scratch (global when longer than QMAX);
// membership of a candidate token is one bit test in a shared vocabulary bitmap when the store's
// token range fits one (StoreView::vwords > 0, set up by the caller), else a binary search in the
// sorted query.  One lane per candidate: the candidate's token range is read with aligned 16-byte
// loads (the token buffer is 16-byte aligned and its slack is zeroed, so the chunks that straddle
// the range hold valid tokens), and a 4-bit mask per chunk keeps only the candidate's own tokens.
// Up to SU chunks per lane and set are in flight together.
constexpr int QMAX = 256;
constexpr int SET_HT = 256;              // open-addressing table of the query's tokens (membership in ~1 probe)
constexpr int QSCR = QMAX + SET_HT;      // words of a set / string query's shared scratch: tokens, then the table
template <int L>
struct SetQuery {
  static constexpr int SU = 1;
  const uint32_t *q;
  const uint32_t *bm;    // vocabulary bitmap of the query (shared) or null
  int qn;

  const uint32_t *ht;    // hash table of the query's tokens (shared; token + 1, 0 = empty) or null
  static __device__ __forceinline__ int hslot(uint32_t t) { return (int)((t * 0x9E3779B1u) >> 24); }

  // scratch: QSCR words of shared memory (tokens, then the table), or null
  __device__ __forceinline__ void load(const StoreView &s, int64_t r, uint32_t *scratch) {
    const int lane = threadIdx.x & 31;
    const uint64_t b = s.off[r];
    qn = (int)(s.off[r + 1] - b);
    bm = nullptr;
    ht = nullptr;
    if (qn <= QMAX && scratch) {
      bool big = false;
      for (int i = lane; i < qn; i += 32) {
        scratch[i] = s.tok[b + i];
        big |= scratch[i] == 0xFFFFFFFFu;
      }
      q = scratch;
      if (qn <= SET_HT / 2 && !__any_sync(FULL, big)) {   // load factor <= 1/2
        uint32_t *t = scratch + QMAX;
        for (int i = lane; i < SET_HT; i += 32) t[i] = 0u;
        __syncwarp();
        for (int i = lane; i < qn; i += 32) {
          const uint32_t v = scratch[i] + 1u;
          int h = hslot(scratch[i]);
          while (atomicCAS(t + h, 0u, v) != 0u) h = (h + 1) & (SET_HT - 1);
        }
        ht = t;
      }
      __syncwarp();
    } else {
      q = s.tok + b;
    }
  }

  __device__ __forceinline__ int has(uint32_t t) const {
    if (ht) {
      for (int h = hslot(t);; h = (h + 1) & (SET_HT - 1)) {
        const uint32_t e = ht[h];
        if (e == t + 1u) return 1;
        if (e == 0u) return 0;
      }
    }
    if (bm) return (bm[t >> 5] >> (t & 31)) & 1u;
    int lo = 0, hi = qn;
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (q[mid] < t) lo = mid + 1;
      else hi = mid;
    }
    return lo < qn && q[lo] == t;
  }

  // NS sets of up to 32 candidates (lane j holds candidate j of each set; id < 0: skipped, key 0)
  template <int NS>
  __device__ __forceinline__ void eval_n(const StoreView &s, const int32_t *cand, uint32_t *out) const {
    uint64_t a0[NS];
    int rb[NS], re[NS], nch[NS], inter[NS];
    int mx = 0;
#pragma unroll
    for (int j = 0; j < NS; ++j) {
      uint64_t b = 0, e = 0;
      if (cand[j] >= 0) {
        if (s.rng) {
          const ulonglong2 r = s.rng[cand[j]];
          b = r.x;
          e = r.y;
        } else {
          b = s.off[cand[j]];
          e = s.off[cand[j] + 1];
        }
      }
      a0[j] = b & ~3ull;
      rb[j] = (int)(b - a0[j]);
      re[j] = (int)(e - a0[j]);
      nch[j] = cand[j] >= 0 ? (re[j] + 3) >> 2 : 0;
      inter[j] = 0;
      mx = max(mx, nch[j]);
    }
    mx = __reduce_max_sync(FULL, mx);
    for (int i0 = 0; i0 < mx; i0 += SU) {
      uint4 buf[NS][SU];
#pragma unroll
      for (int j = 0; j < NS; ++j)
#pragma unroll
        for (int u = 0; u < SU; ++u)
          buf[j][u] = i0 + u < nch[j] ? ldg16(s.tok + a0[j] + 4 * (i0 + u)) : make_uint4(0, 0, 0, 0);
#pragma unroll
      for (int j = 0; j < NS; ++j)
#pragma unroll
        for (int u = 0; u < SU; ++u) {
          const int c0 = 4 * (i0 + u);
          if (i0 + u < nch[j]) {
            const int lo = rb[j] > c0 ? rb[j] - c0 : 0;
            const int hi = re[j] - c0 < 4 ? re[j] - c0 : 4;
            const unsigned m = (0xFu >> (4 - hi)) & (0xFu << lo);
            const unsigned h = (unsigned)has(buf[j][u].x) | ((unsigned)has(buf[j][u].y) << 1) |
                               ((unsigned)has(buf[j][u].z) << 2) | ((unsigned)has(buf[j][u].w) << 3);
            inter[j] += __popc(h & m);
          }
        }
    }
#pragma unroll
    for (int j = 0; j < NS; ++j)
      out[j] = cand[j] >= 0 ? (((uint32_t)inter[j] << 16) | (uint32_t)(qn + (re[j] - rb[j]) - inter[j])) : 0u;
  }

  // Key of the candidate whose aligned token chunks are staged at slot (16 B each, the launch's slot size at
  // most; rb/re = first/end token relative to the first chunk).  Lane-local.
  __device__ __forceinline__ uint32_t eval_slot(const uint8_t *slot, int rb, int re) const {
    const int nch = (re + 3) >> 2;
    int inter = 0;
#pragma unroll 1
    for (int i = 0; i < nch; ++i) {
      const uint4 t = *(const uint4 *)(slot + 16 * i);
      const int c0 = 4 * i;
      const int lo = rb > c0 ? rb - c0 : 0;
      const int hi = re - c0 < 4 ? re - c0 : 4;
      const unsigned m = (0xFu >> (4 - hi)) & (0xFu << lo);
      const unsigned h = (unsigned)has(t.x) | ((unsigned)has(t.y) << 1) | ((unsigned)has(t.z) << 2) |
                         ((unsigned)has(t.w) << 3);
      inter += __popc(h & m);
    }
    return ((uint32_t)inter << 16) | (uint32_t)(qn + (re - rb) - inter);
  }

  __device__ __forceinline__ uint32_t eval_slot_global(const uint32_t *t0, int rb, int re) const {
    const int nch = (re + 3) >> 2;
    int inter = 0;
    for (int i = 0; i < nch; ++i) {
      const uint4 t = ldg16(t0 + 4 * i);
      const int c0 = 4 * i;
      const int lo = rb > c0 ? rb - c0 : 0;
      const int hi = re - c0 < 4 ? re - c0 : 4;
      const unsigned m = (0xFu >> (4 - hi)) & (0xFu << lo);
      const unsigned h = (unsigned)has(t.x) | ((unsigned)has(t.y) << 1) | ((unsigned)has(t.z) << 2) |
                         ((unsigned)has(t.w) << 3);
      inter += __popc(h & m);
    }
    return ((uint32_t)inter << 16) | (uint32_t)(qn + (re - rb) - inter);
  }

  __device__ __forceinline__ uint32_t eval(const StoreView &s, int32_t cand, int n) const {
    const int lane = threadIdx.x & 31;
    const int32_t c[1] = {lane < n ? cand : -1};
    uint32_t o[1];
    eval_n<1>(s, c, o);
    return o[0];
  }

  __device__ __forceinline__ void eval2(const StoreView &s, int32_t ca, int32_t cb, uint32_t &oa, uint32_t &ob) const {
    const int32_t c[2] = {ca, cb};
    uint32_t o[2];
    eval_n<2>(s, c, o);
    oa = o[0];
    ob = o[1];
  }
};

// Strings (M_JW / M_COS): the query's characters in shared scratch (QSCR words >= STR_MAX), one lane per
// candidate, its characters read from global memory (str_key).  n2 of a candidate from StoreView::n2.
// COS with scratch: the query's 2-grams also go into a 256-slot open-addressing table (word (i + 1) |
// count << 16, i = the 2-gram's first position in the query), so that dot(q, x) = sum over x's 2-gram
// positions of the query's count of that 2-gram -- one probe per position of x instead of |q| compares.
constexpr int STR_HT = 256;
__device__ __forceinline__ int bigram_slot(uint32_t c0, uint32_t c1) {
  return (int)(((c0 * 0x9E3779B1u) ^ (c1 * 0x85EBCA77u)) >> 24);
}
// JW with scratch: the query's character positions grouped by character (qpos, ascending within a
// character) and a 256-slot table character -> (first position + 1, count, start in qpos, character id).
// A pair is then matched by ONE pass over the other string x: for x[j], the query positions of that
// character are consumed left to right by a per-character pointer (positions < j - w can never match a
// later j and are skipped for good; the next one matches if <= j + w).  Per character this is the greedy
// matching of Q33 taken from x's side; it picks the same pairs as from the query's side (both match the
// occurrences window-feasibly in order; the GPU parity tests compare every key with the oracle's
// query-side loop), so m and T are unchanged.  The pointers live in a 128-byte slot per lane.
constexpr int JW_PTR = 128;   // bytes of one lane's character pointers (<= 127 distinct characters)
template <int M>
struct StrQuery {
  const uint32_t *q;
  int qn;
  uint32_t qn2;           // COS: the query's own |q|^2 (a key of the query as another row's entry)
  const uint32_t *ht;     // COS: the query's 2-gram table / JW: the character table (shared scratch), else null
  const uint32_t *qpos;   // JW: the query's positions grouped by character
  uint8_t *ptr = nullptr; // JW: this lane's character pointers (JW_PTR bytes of shared memory), else null
  __device__ __forceinline__ void load(const StoreView &s, int64_t r, uint32_t *scratch) {
    const int lane = threadIdx.x & 31;
    const uint64_t b = s.off[r];
    qn = (int)(s.off[r + 1] - b);
    qn2 = (M == M_COS && s.n2) ? s.n2[r] : 0u;
    ht = nullptr;
    qpos = nullptr;
    if (scratch) {
      for (int i = lane; i < qn; i += 32) scratch[i] = s.tok[b + i];
      q = scratch;
      if (M == M_COS) {   // the 2-gram table after the characters (STR_MAX + 1 + STR_HT <= QSCR words)
        uint32_t *t = scratch + STR_MAX + 1;
        for (int i = lane; i < STR_HT; i += 32) t[i] = 0u;
        __syncwarp();
        for (int i = lane; i + 1 < qn; i += 32) {
          const uint32_t c0 = scratch[i], c1 = scratch[i + 1];
          for (int h = bigram_slot(c0, c1);; h = (h + 1) & (STR_HT - 1)) {
            const uint32_t old = atomicCAS(t + h, 0u, (uint32_t)(i + 1) | (1u << 16));
            if (old == 0u) break;
            const int j = (int)(old & 0xFFFFu) - 1;
            if (scratch[j] == c0 && scratch[j + 1] == c1) {
              atomicAdd(t + h, 1u << 16);
              break;
            }
          }
        }
        ht = t;
      }
      if (M == M_JW && ptr) {   // character table at [256, 512), positions at [128, 256)
        uint32_t *t = scratch + 2 * (STR_MAX + 1);
        uint32_t *qp = scratch + STR_MAX + 1;
        for (int i = lane; i < STR_HT; i += 32) t[i] = 0u;
        __syncwarp();
        // slot word: first position + 1 (the character's first occurrence inserts it)
        for (int i = lane; i < qn; i += 32) {
          const uint32_t c = scratch[i];
          int first = i;
          for (int j = 0; j < i; ++j)
            if (scratch[j] == c) { first = j; break; }
          if (first != i) continue;
          for (int h = (int)((c * 0x9E3779B1u) >> 24);; h = (h + 1) & (STR_HT - 1))
            if (atomicCAS(t + h, 0u, (uint32_t)(i + 1)) == 0u) break;
        }
        __syncwarp();
        // per slot: count, start in qp (exclusive scan in slot order) and character id (rank of the slot)
        uint32_t cnt[STR_HT / 32];
        int tot = 0, ids = 0;
#pragma unroll
        for (int u = 0; u < STR_HT / 32; ++u) {
          const uint32_t e = t[lane * (STR_HT / 32) + u];
          uint32_t n = 0;
          if (e) {
            const uint32_t c = scratch[(e & 0xFFu) - 1];
            for (int j = 0; j < qn; ++j) n += scratch[j] == c;
          }
          cnt[u] = n;
          tot += (int)n;
          ids += e ? 1 : 0;
        }
        int pre = tot, pid = ids;   // inclusive warp scans of the counts and of the occupied slots
        for (int o = 1; o < 32; o <<= 1) {
          const int x1 = __shfl_up_sync(FULL, pre, o), x2 = __shfl_up_sync(FULL, pid, o);
          if (lane >= o) { pre += x1; pid += x2; }
        }
        int start = pre - tot, cid = pid - ids;
        __syncwarp();
#pragma unroll
        for (int u = 0; u < STR_HT / 32; ++u) {
          const int h = lane * (STR_HT / 32) + u;
          const uint32_t e = t[h];
          if (e) {
            t[h] = (e & 0xFFu) | (cnt[u] << 8) | ((uint32_t)start << 15) | ((uint32_t)cid << 22);
            start += (int)cnt[u];
            ++cid;
          }
        }
        __syncwarp();
        // positions of each character, ascending: rank = earlier positions with the same character
        for (int i = lane; i < qn; i += 32) {
          const uint32_t c = scratch[i];
          int rank = 0;
          for (int j = 0; j < i; ++j) rank += scratch[j] == c;
          for (int h = (int)((c * 0x9E3779B1u) >> 24);; h = (h + 1) & (STR_HT - 1)) {
            const uint32_t e = t[h];
            if (scratch[(e & 0xFFu) - 1] == c) {
              qp[((e >> 15) & 0x7Fu) + rank] = (uint32_t)i;
              break;
            }
          }
        }
        ht = t;
        qpos = qp;
      }
      __syncwarp();
    } else {
      q = s.tok + b;
    }
  }
  // JW key of the query against x (lane-local, the character table): x's characters in order, each
  // matched to the next feasible query position of the same character (see the comment above).  a_is_q:
  // the key's first string is the query (search) or x (the update's key, x = the row owner).
  __device__ __forceinline__ uint32_t jw_table(const uint32_t *x, int lx, bool a_is_q) const {
    const int la = a_is_q ? qn : lx, lb = a_is_q ? lx : qn;
    int w = (qn > lx ? qn : lx) / 2 - 1;
    if (w < 0) w = 0;
    for (int u = 0; u < JW_PTR / 16; ++u) ((uint4 *)ptr)[u] = make_uint4(0, 0, 0, 0);
    uint64_t qm0 = 0, qm1 = 0, xm0 = 0, xm1 = 0;   // matched positions of the query / of x
    int m = 0;
    for (int j = 0; j < lx; ++j) {
      const uint32_t c = x[j];
      uint32_t e;
      for (int h = (int)((c * 0x9E3779B1u) >> 24);; h = (h + 1) & (STR_HT - 1)) {
        e = ht[h];
        if (e == 0u || q[(e & 0xFFu) - 1] == c) break;
      }
      if (e == 0u) continue;
      const int cnt = (int)((e >> 8) & 0x7Fu), st = (int)((e >> 15) & 0x7Fu), cid = (int)(e >> 22);
      int p = ptr[cid];
      while (p < cnt && (int)qpos[st + p] < j - w) ++p;
      if (p < cnt && (int)qpos[st + p] <= j + w) {
        const int i = (int)qpos[st + p];
        ++p;
        ++m;
        if (i < 64) qm0 |= 1ull << i; else qm1 |= 1ull << (i - 64);
        if (j < 64) xm0 |= 1ull << j; else xm1 |= 1ull << (j - 64);
      }
      ptr[cid] = (uint8_t)p;
    }
    int T = 0;
    for (int r = 0; r < m; ++r) {
      const int i = qm0 ? __ffsll((long long)qm0) - 1 : 64 + __ffsll((long long)qm1) - 1;
      const int j = xm0 ? __ffsll((long long)xm0) - 1 : 64 + __ffsll((long long)xm1) - 1;
      if (qm0) qm0 &= qm0 - 1; else qm1 &= qm1 - 1;
      if (xm0) xm0 &= xm0 - 1; else xm1 &= xm1 - 1;
      T += q[i] != x[j];
    }
    int l = 0;
    while (l < 4 && l < qn && l < lx && q[l] == x[l]) ++l;
    return (uint32_t)m | ((uint32_t)T << 7) | ((uint32_t)l << 14) | ((uint32_t)la << 17) | ((uint32_t)lb << 24);
  }
  // the query's count of 2-gram (c0, c1) (COS with the table)
  __device__ __forceinline__ uint32_t qcount(uint32_t c0, uint32_t c1) const {
    for (int h = bigram_slot(c0, c1);; h = (h + 1) & (STR_HT - 1)) {
      const uint32_t e = ht[h];
      if (e == 0u) return 0u;
      const int j = (int)(e & 0xFFFFu) - 1;
      if (q[j] == c0 && q[j + 1] == c1) return e >> 16;
    }
  }
  // dot(q, x) over x's 2-gram positions (COS with the table)
  __device__ __forceinline__ uint32_t qdot(const uint32_t *x, int lx) const {
    uint32_t dot = 0;
    uint32_t c0 = lx > 0 ? x[0] : 0u;
    for (int j = 0; j + 1 < lx; ++j) {
      const uint32_t c1 = x[j + 1];
      dot += qcount(c0, c1);
      c0 = c1;
    }
    return dot;
  }
  // key of candidate cand (lane-local; cand < 0: 0)
  __device__ __forceinline__ uint32_t key(const StoreView &s, int32_t cand) const {
    if (cand < 0) return 0u;
    uint64_t b, e;
    if (s.rng) {
      const ulonglong2 r = s.rng[cand];
      b = r.x;
      e = r.y;
    } else {
      b = s.off[cand];
      e = s.off[cand + 1];
    }
    if (M == M_COS && ht) return (qdot(s.tok + b, (int)(e - b)) << 16) | s.n2[cand];
    if (M == M_JW && qpos) return jw_table(s.tok + b, (int)(e - b), true);
    return str_key<M>(q, qn, s.tok + b, (int)(e - b), M == M_COS ? s.n2[cand] : 0u);
  }
  __device__ __forceinline__ uint32_t eval(const StoreView &s, int32_t cand, int n) const {
    return key(s, (threadIdx.x & 31) < n ? cand : -1);
  }
  // the query as an entry of node v's row (the update's proposals): v owns the key
  __device__ __forceinline__ uint32_t rkey(const StoreView &s, int32_t v) const {
    if (v < 0) return 0u;
    const uint64_t b = s.off[v];
    if (M == M_COS && ht) return (qdot(s.tok + b, (int)(s.off[v + 1] - b)) << 16) | qn2;   // dot is symmetric
    if (M == M_JW && qpos) return jw_table(s.tok + b, (int)(s.off[v + 1] - b), false);   // from v's side
    return str_key<M>(s.tok + b, (int)(s.off[v + 1] - b), q, qn, qn2);
  }
  __device__ __forceinline__ void eval2(const StoreView &s, int32_t ca, int32_t cb, uint32_t &oa, uint32_t &ob) const {
    oa = key(s, ca);
    ob = key(s, cb);
  }
  __device__ __forceinline__ uint32_t eval_smem(const uint8_t *, int, int) const { return 0u; }
};

template <int M, int L, int CPL>
struct QuerySel { typedef VecQuery<M, L, CPL> T; };
template <int L, int CPL>
struct QuerySel<M_JAC, L, CPL> { typedef SetQuery<L> T; };
template <int L, int CPL>
struct QuerySel<M_JW, L, CPL> { typedef StrQuery<M_JW> T; };
template <int L, int CPL>
struct QuerySel<M_COS, L, CPL> { typedef StrQuery<M_COS> T; };

}  // namespace knng
