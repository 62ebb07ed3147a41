/*
 * knng_oracle.c -- CPU ORACLE for the online approximate k-nn graph of
 * arXiv 1602.06819 (Debatty, Michiardi, Mees, Thonnard, "Fast online k-nn
 * graph building").  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load or call this library.  The product path
 * (paper_1602_06819_b200/) never links it, and it shares no code, header,
 * table or helper with the CUDA path.
 *
 * It is deliberately plain and slow: every function follows the paper's
 * text in the paper's order.  Citations "P:n" are lines of PAPER.md (the
 * LaTeX source), with the section / algorithm they fall in.  Where the
 * paper is silent the reading taken is the one listed in DESIGN.md
 * ("Readings", numbered Q1..Q31 as in SURVEY.md section 8(c)).
 *
 * Build:  gcc -O2 -ffp-contract=off -fPIC -shared -pthread -o liboracle.so knng_oracle.c -lm
 * (no fast-math; -ffp-contract=off so that fp32 distances are computed in
 * exactly the canonical order of reading Q24).
 *
 * Parity status per function:
 *   or_key_of            pinned (closed forms, fp64 brute force)
 *   or_rng_draw          parity unpinned by the paper (Q4); pinned only by a
 *                        second, independent Python implementation (KAT)
 *   or_rng_perm          (the restart draws, Q4) parity unpinned by the paper; pinned by an
 *                        independent Python implementation (KAT), exhaustive bijection checks
 *                        and a uniformity check of pi(0)
 *   or_exact_rows        pinned (hand examples, brute force in numpy)
 *   or_ignns_search      pinned (W3 hand traces, budget >= |pool| => linear search, a literal
 *                        re-derivation of the walk without the Q9 shortcut in tests/pyref.py);
 *                        its full_scan mode (the GNNS baseline) pinned the same way
 *   or_insert_batch      pinned (W1, W2, 1-D exactness, B=1 == literal Alg.1+2)
 *   or_insert_sequential pinned (W1, W2 sequential)
 *   or_partition_kmedoids pinned (W7 hand trace, balance bound, brute hop sums)
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ */
/* Metrics.  P:286 (synthetic: euclidean distance), P:292 (set / n-gram  */
/* similarity).  Keys are packed into 32 bits:                          */
/*   OR_U8  : D = sum_j (a_j-b_j)^2, exact integer (Q25: squared L2)    */
/*   OR_F32 : D = fp32 squared L2 in the canonical order (Q24), as bits */
/*   OR_JAC : (inter << 16) | union of two token sets                   */
/*   OR_JW  : Jaro-Winkler of two strings (section 7.1.2):        */
/*            m | T << 7 | l << 14 | |a| << 17 | |b| << 24               */
/*   OR_COS : cosine of the 2-gram count vectors (section 7.1.3): */
/*            (dot << 16) | max(|b|^2, 1), b = the row's other end       */
/* Strings are sequences of uint32 characters (<= 127) held like sets    */
/* (tok / off), in their original order.                                 */
/* ------------------------------------------------------------------ */
enum { OR_U8 = 0, OR_F32 = 1, OR_JAC = 2, OR_JW = 3, OR_COS = 4 };

typedef struct {
  int metric;
  int dim;                 /* u8 / f32 only */
  const uint8_t *u8;       /* [n][dim] */
  const float *f32;        /* [n][dim] */
  const uint64_t *off;     /* JAC: [n+1] offsets into tok */
  const uint32_t *tok;     /* JAC: sorted, unique tokens per set */
} or_store;

/* A "point" is either a row of a store or an external query.  */
typedef struct {
  const uint8_t *u8;
  const float *f32;
  const uint32_t *tok;
  int64_t ntok;
} or_point;

static or_point store_point(const or_store *S, int64_t i) {
  or_point p;
  memset(&p, 0, sizeof p);
  if (S->metric == OR_U8) p.u8 = S->u8 + (size_t)i * S->dim;
  else if (S->metric == OR_F32) p.f32 = S->f32 + (size_t)i * S->dim;
  else { p.tok = S->tok + S->off[i]; p.ntok = (int64_t)(S->off[i + 1] - S->off[i]); }
  return p;
}

static uint32_t float_bits(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }
static float bits_float(uint32_t u) { float f; memcpy(&f, &u, 4); return f; }

/* Reading Q24: the fp32 squared distance is defined by a fixed evaluation
 * order.  32 partial sums ("lanes"); 4-float chunk c goes to lane c mod 32;
 * inside a chunk the dims are taken in order with acc = fmaf(d, d, acc),
 * d = a - b in fp32.  Then the 32 partials are combined by the xor
 * butterfly with offsets 16, 8, 4, 2, 1 (acc[l] = acc[l] + acc[l ^ o]). */
static float f32_canonical_l2sq(const float *a, const float *b, int dim) {
  float acc[32];
  int l, c, t, o;
  for (l = 0; l < 32; ++l) acc[l] = 0.0f;
  for (c = 0; 4 * c < dim; ++c) {
    for (t = 0; t < 4; ++t) {
      int idx = 4 * c + t;
      if (idx < dim) {
        float d = a[idx] - b[idx];
        acc[c % 32] = fmaf(d, d, acc[c % 32]);
      }
    }
  }
  for (o = 16; o >= 1; o >>= 1) {
    float nxt[32];
    for (l = 0; l < 32; ++l) nxt[l] = acc[l] + acc[l ^ o];
    for (l = 0; l < 32; ++l) acc[l] = nxt[l];
  }
  return acc[0];
}

/* Jaro-Winkler (Jaro similarity with the Winkler prefix boost, prefix <= 4,
 * scaling 0.1), the textbook definition step by step:
 *   window w = max(|a|, |b|) / 2 - 1 (floor, at least 0);
 *   a character a[i] matches the first not yet matched b[j] with b[j] == a[i] and |i - j| <= w,
 *   taking i in order;  m = the number of matches;
 *   T = the number of positions at which the matched characters of a and of b, each read in
 *   order, differ (t = T / 2 transpositions);
 *   jaro = (m/|a| + m/|b| + (m - t)/m) / 3  (0 when m = 0);
 *   l = the common prefix length, at most 4;  jw = jaro + l * 0.1 * (1 - jaro).
 * The key keeps (m, T, l, |a|, |b|): jw is recovered exactly as a fraction (or_jw_fraction). */
static uint32_t jw_key(const uint32_t *a, int64_t la, const uint32_t *b, int64_t lb) {
  unsigned char amatch[128], bmatch[128];
  int64_t w = (la > lb ? la : lb) / 2 - 1, i, j, m = 0, T = 0, l = 0;
  if (w < 0) w = 0;
  memset(amatch, 0, sizeof amatch);
  memset(bmatch, 0, sizeof bmatch);
  for (i = 0; i < la; ++i) {
    int64_t lo = i - w > 0 ? i - w : 0, hi = i + w < lb - 1 ? i + w : lb - 1;
    for (j = lo; j <= hi; ++j) {
      if (!bmatch[j] && b[j] == a[i]) { bmatch[j] = 1; amatch[i] = 1; ++m; break; }
    }
  }
  j = 0;
  for (i = 0; i < la; ++i) {
    if (!amatch[i]) continue;
    while (!bmatch[j]) ++j;
    if (a[i] != b[j]) ++T;
    ++j;
  }
  while (l < 4 && l < la && l < lb && a[l] == b[l]) ++l;
  return (uint32_t)(m | (T << 7) | (l << 14) | (la << 17) | (lb << 24));
}

/* jw = N / D exactly: jaro = (2 m^2 |b| + 2 m^2 |a| + (2m - T) |a| |b|) / (6 |a| |b| m) and
 * jw = ((10 - l) jaro + l) / 10.  m = 0: 0 / 1. */
void or_jw_fraction(uint32_t key, uint64_t *num, uint64_t *den) {
  uint64_t m = key & 127, T = (key >> 7) & 127, l = (key >> 14) & 7, la = (key >> 17) & 127, lb = (key >> 24) & 127;
  uint64_t n0, d0;
  if (m == 0) { *num = 0; *den = 1; return; }
  n0 = 2 * m * m * lb + 2 * m * m * la + (2 * m - T) * la * lb;
  d0 = 6 * la * lb * m;
  *num = (10 - l) * n0 + l * d0;
  *den = 10 * d0;
}

/* Cosine of the 2-gram count vectors: a string's 2-grams are its contiguous
 * pairs (s[i], s[i+1]); dot = sum over 2-grams g of c_a(g) c_b(g) = the number of position pairs
 * (i, j) with equal 2-grams; |b|^2 = sum_g c_b(g)^2 likewise.  cos = dot / (|a| |b|), 0 when either
 * string is shorter than 2 (zero vector).  The key keeps dot and |b|^2 (1 for a zero vector): within
 * one row or one query |a| is common, so cos_1 > cos_2 <=> dot_1^2 |b_2|^2 > dot_2^2 |b_1|^2. */
static uint32_t cos2_key(const uint32_t *a, int64_t la, const uint32_t *b, int64_t lb) {
  int64_t i, j, dot = 0, nb = 0;
  for (i = 0; i + 1 < la; ++i)
    for (j = 0; j + 1 < lb; ++j)
      if (a[i] == b[j] && a[i + 1] == b[j + 1]) ++dot;
  for (i = 0; i + 1 < lb; ++i)
    for (j = 0; j + 1 < lb; ++j)
      if (b[i] == b[j] && b[i + 1] == b[j + 1]) ++nb;
  if (nb == 0) nb = 1;
  return (uint32_t)((dot << 16) | nb);
}

static uint32_t key_of(const or_store *S, or_point a, or_point b) {
  if (S->metric == OR_U8) {
    int32_t D = 0;
    int j;
    for (j = 0; j < S->dim; ++j) {
      int32_t d = (int32_t)a.u8[j] - (int32_t)b.u8[j];
      D += d * d;
    }
    return (uint32_t)D;
  } else if (S->metric == OR_F32) {
    return float_bits(f32_canonical_l2sq(a.f32, b.f32, S->dim));
  } else if (S->metric == OR_JW) {
    return jw_key(a.tok, a.ntok, b.tok, b.ntok);
  } else if (S->metric == OR_COS) {
    return cos2_key(a.tok, a.ntok, b.tok, b.ntok);
  } else {
    /* |A n B| by merging two sorted lists; |A u B| = |A| + |B| - |A n B| */
    int64_t i = 0, j = 0, inter = 0;
    while (i < a.ntok && j < b.ntok) {
      if (a.tok[i] == b.tok[j]) { ++inter; ++i; ++j; }
      else if (a.tok[i] < b.tok[j]) ++i;
      else ++j;
    }
    return (uint32_t)((inter << 16) | (a.ntok + b.ntok - inter));
  }
}

/* "closer(a, b)": key a is strictly more similar than key b (metric value only). */
static int closer(int metric, uint32_t a, uint32_t b) {
  if (metric == OR_U8) return a < b;
  if (metric == OR_F32) return bits_float(a) < bits_float(b);
  if (metric == OR_JW) {          /* jw_a > jw_b as fractions */
    uint64_t na, da, nb, db;
    or_jw_fraction(a, &na, &da);
    or_jw_fraction(b, &nb, &db);
    return (unsigned __int128)na * db > (unsigned __int128)nb * da;
  }
  if (metric == OR_COS) {         /* dot_a / |x_a| > dot_b / |x_b|, squared */
    uint64_t da = a >> 16, na = a & 0xFFFF, db = b >> 16, nb = b & 0xFFFF;
    return (unsigned __int128)da * da * nb > (unsigned __int128)db * db * na;
  }
  {
    int64_t ia = a >> 16, ua = a & 0xFFFF, ib = b >> 16, ub = b & 0xFFFF;
    return ia * ub > ib * ua;      /* i_a/u_a > i_b/u_b, exact (C.1) */
  }
}

/* Edge order (C.1): closer key first, equal similarity -> smaller id. */
static int precedes(int metric, uint32_t ka, int64_t ida, uint32_t kb, int64_t idb) {
  if (closer(metric, ka, kb)) return 1;
  if (closer(metric, kb, ka)) return 0;
  return ida < idb;
}

/* Skip rule: discard r if similarity(q, r) < s_max / e, e = num/den.
 * Q1: for the L2 metrics s = 1/(1+D); s_r < s_max/e  <=>  den*(1+D_r) > num*(1+D_best).
 * For Jaccard s = i/u; s_r < s_max/e  <=>  num*i_r*u_best < den*i_best*u_r.
 * den == 0 encodes e = +inf (never skip). */
static int skip_start(int metric, uint32_t kr, uint32_t kbest, uint64_t num, uint64_t den) {
  if (den == 0) return 0;
  if (metric == OR_U8) {
    uint64_t lhs = den * (1ull + (uint64_t)kr), rhs = num * (1ull + (uint64_t)kbest);
    return lhs > rhs;
  } else if (metric == OR_F32) {
    volatile double lhs = (double)den * (1.0 + (double)bits_float(kr));
    volatile double rhs = (double)num * (1.0 + (double)bits_float(kbest));
    return lhs > rhs;
  } else if (metric == OR_JW) {   /* s = jw: num * jw_r < den * jw_best, as fractions */
    uint64_t nr, dr, nbst, dbst;
    or_jw_fraction(kr, &nr, &dr);
    or_jw_fraction(kbest, &nbst, &dbst);
    return (unsigned __int128)num * nr * dbst < (unsigned __int128)den * nbst * dr;
  } else if (metric == OR_COS) {  /* s = cos (|a| common): num dot_r / |x_r| < den dot_b / |x_b|, squared */
    unsigned __int128 dr = kr >> 16, nr = kr & 0xFFFF, db = kbest >> 16, nbst = kbest & 0xFFFF;
    return (unsigned __int128)num * num * dr * dr * nbst < (unsigned __int128)den * den * db * db * nr;
  } else {
    uint64_t ir = kr >> 16, ur = kr & 0xFFFF, ib = kbest >> 16, ub = kbest & 0xFFFF;
    return num * ir * ub < den * ib * ur;
  }
}

/* ------------------------------------------------------------------ */
/* RNG (reading Q4): uniform draw with replacement from the pool, keyed */
/* by (seed, point id, partition, draw #).  SplitMix64 finaliser chain. */
/* ------------------------------------------------------------------ */
static uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
#define OR_GOLDEN 0x9E3779B97F4A7C15ull

uint64_t or_rng_hash(uint64_t seed, uint64_t pid, uint64_t part, uint64_t draw) {
  uint64_t h = mix64(seed + 1ull * OR_GOLDEN);
  h = mix64(h ^ (pid + 2ull * OR_GOLDEN));
  h = mix64(h ^ (part + 3ull * OR_GOLDEN));
  h = mix64(h ^ (draw + 4ull * OR_GOLDEN));
  return h;
}

/* index = floor(h * m / 2^64) */
uint64_t or_rng_draw(uint64_t seed, uint64_t pid, uint64_t part, uint64_t draw, uint64_t m) {
  unsigned __int128 prod = (unsigned __int128)or_rng_hash(seed, pid, part, draw) * m;
  return (uint64_t)(prod >> 64);
}

/* Restart draws (reading Q4, round 2): the draws of one search are a pseudo-random PERMUTATION of the
 * pool, pi(0), pi(1), ..., so a draw never repeats an earlier draw; a draw of a node a walk evaluated
 * is still skipped for free.  pi is a 6-round (unbalanced) Feistel network on b = max(6, ceil(log2 m)) bits
 * with cycle walking (apply F until the value is < m), keyed by the (seed, pid, part) prefix:
 *   prefix = mix64(mix64(mix64(seed + G) ^ (pid + 2G)) ^ (part + 3G))
 *   key_i  = (uint32)(prefix >> 16 (i mod 4)) ^ 0x9E3779B9 (i + 1)         (i = 0..5, 32-bit)
 *   F(x):  L = x >> hr, R = x mod 2^hr (hl = b / 2, hr = b - hl bits);
 *          round i: (L, R) <- (R, L ^ (lowbias32(R ^ key_i) mod 2^|L|))  (the halves swap widths)
 * lowbias32(z): z ^= z >> 16; z *= 0x7feb352d; z ^= z >> 15; z *= 0x846ca68b; z ^= z >> 16. */
static uint32_t lowbias32(uint32_t z) {
  z ^= z >> 16; z *= 0x7feb352du; z ^= z >> 15; z *= 0x846ca68bu; z ^= z >> 16;
  return z;
}
static uint32_t feistel(uint64_t prefix, uint32_t x, int hl, int hr) {
  uint32_t L = x >> hr, R = x & ((1u << hr) - 1u);
  int la = hl, ra = hr, i, t;
  for (i = 0; i < 6; ++i) {
    uint32_t key = (uint32_t)(prefix >> (16 * (i & 3))) ^ (0x9E3779B9u * (uint32_t)(i + 1));
    uint32_t nR = L ^ (lowbias32(R ^ key) & ((1u << la) - 1u));
    L = R; R = nR;
    t = la; la = ra; ra = t;
  }
  return (L << ra) | R;
}
/* pi(j) for 0 <= j < m (m <= 2^31); -1 when j >= m (the pool is exhausted) */
int64_t or_rng_perm(uint64_t seed, uint64_t pid, uint64_t part, uint64_t j, uint64_t m) {
  uint64_t prefix = mix64(mix64(mix64(seed + 1ull * OR_GOLDEN) ^ (pid + 2ull * OR_GOLDEN)) ^ (part + 3ull * OR_GOLDEN));
  int b = 0, hl, hr;
  uint32_t x;
  if (j >= m) return -1;
  while ((1ull << b) < m) ++b;
  if (b < 6) b = 6;                        /* tiny pools: walk down from 64 (a 4-bit Feistel mixes poorly) */
  hl = b / 2; hr = b - hl;
  x = (uint32_t)j;
  do { x = feistel(prefix, x, hl, hr); } while (x >= m);
  return (int64_t)x;
}

/* ------------------------------------------------------------------ */
/* Neighbour list of capacity k, sorted by edge order.                 */
/* ------------------------------------------------------------------ */
typedef struct {
  int cap, cnt;
  uint32_t *key;
  int32_t *id;
} or_list;

/* Insert (key, id) keeping the k best by edge order; returns 1 if accepted.
 * Duplicate ids are rejected (neighbour lists hold distinct ids). */
static int list_insert(int metric, or_list *L, uint32_t key, int32_t id) {
  int i, pos;
  if (L->cnt == L->cap && !precedes(metric, key, id, L->key[L->cnt - 1], L->id[L->cnt - 1]))
    return 0;
  for (i = 0; i < L->cnt; ++i)
    if (L->id[i] == id) return 0;
  pos = 0;
  while (pos < L->cnt && precedes(metric, L->key[pos], L->id[pos], key, id)) ++pos;
  if (L->cnt < L->cap) L->cnt++;
  for (i = L->cnt - 1; i > pos; --i) { L->key[i] = L->key[i - 1]; L->id[i] = L->id[i - 1]; }
  L->key[pos] = key;
  L->id[pos] = id;
  return 1;
}

/* ------------------------------------------------------------------ */
/* Exact rows (AL1): row v = the first k of all u != v in edge order. */
/* ------------------------------------------------------------------ */
void or_exact_rows(int metric, int dim, const void *data, const uint64_t *off,
                   int64_t n, int k, const int64_t *rows, int64_t nrows,
                   int32_t *out_ids, uint32_t *out_keys) {
  or_store S;
  int64_t r, u;
  S.metric = metric; S.dim = dim;
  S.u8 = (const uint8_t *)data; S.f32 = (const float *)data;
  S.off = off; S.tok = (const uint32_t *)data;
  for (r = 0; r < nrows; ++r) {
    int64_t v = rows[r];
    or_list L;
    L.cap = k; L.cnt = 0; L.key = out_keys + r * k; L.id = out_ids + r * k;
    for (u = 0; u < n; ++u) {
      if (u == v) continue;
      list_insert(metric, &L, key_of(&S, store_point(&S, v), store_point(&S, u)), (int32_t)u);
    }
    for (u = L.cnt; u < k; ++u) { L.id[u] = -1; L.key[u] = 0; }
  }
}

/* ------------------------------------------------------------------ */
/* iGNNS, P:73-89 (section 3), with readings Q3-Q11.                   */
/* ------------------------------------------------------------------ */
typedef struct {
  int64_t evals;       /* committed similarity evaluations (the budgeted count) */
  int64_t starts;      /* random starts evaluated */
  int64_t skipped;     /* starts discarded by the expansion rule */
  int64_t expansions;  /* nodes whose neighbour list was scanned */
} or_search_stats;

typedef struct {           /* per-thread scratch indexed by node id */
  int64_t n;
  uint8_t *evaluated;
  uint8_t *expanded;
  uint32_t *keyv;
  int32_t *touched;        /* list of evaluated ids, to reset the marks */
} or_scratch;

static int scratch_init(or_scratch *W, int64_t n) {
  W->n = n;
  W->evaluated = (uint8_t *)calloc((size_t)n + 1, 1);
  W->expanded = (uint8_t *)calloc((size_t)n + 1, 1);
  W->keyv = (uint32_t *)calloc((size_t)n + 1, 4);
  W->touched = (int32_t *)calloc((size_t)n + 1, 4);
  return W->evaluated && W->expanded && W->keyv && W->touched;
}
static void scratch_free(or_scratch *W) {
  free(W->evaluated); free(W->expanded); free(W->keyv); free(W->touched);
}

typedef struct {
  const or_store *S;
  int k;                    /* graph degree (row width) */
  const int32_t *rows;      /* snapshot rows [n_t][k] */
  const int32_t *pool;      /* pool nodes (ascending); NULL => pool = 0..m-1 */
  int64_t m;                /* |pool| */
  const uint8_t *part_of;   /* NULL (unpartitioned) or partition of each node */
  int part;                 /* partition searched (0 when unpartitioned) */
  double speedup;
  uint64_t e_num, e_den;
  uint64_t seed;
  const int32_t *starts;    /* test hook: explicit start sequence (Q4 override) */
  int64_t nstarts;
  int full_scan;            /* 1: the GNNS baseline's walk (section 2.2): evaluate every
                               neighbour of the current node, move to the most similar one */
} or_search_cfg;

/* Q6: budget = max(min(k, |pool|), floor(|pool| / speedup)). */
int64_t or_budget(int64_t m, int k, double speedup) {
  int64_t b = (int64_t)floor((double)m / speedup);
  int64_t lo = m < k ? m : k;
  return b > lo ? b : lo;
}

static int in_pool(const or_search_cfg *C, int32_t v) {
  if (C->part_of == NULL) return 1;
  return C->part_of[v] == C->part;
}

/* Search for query q (global id pid for the RNG stream).  Result: top-k_r in T. */
static void ignns(const or_search_cfg *C, or_point q, int64_t pid, int kr,
                  or_scratch *W, or_list *T, or_search_stats *st) {
  const int metric = C->S->metric;
  const int64_t budget = or_budget(C->m, kr, C->speedup);
  int64_t c = 0;           /* similarities computed */
  int64_t j = 0;           /* draw counter */
  int64_t ntouched = 0;
  int first = 1;
  int64_t i;
  memset(st, 0, sizeof *st);
  T->cnt = 0;

  for (;;) {
    /* ---- restart with a random node ---- */
    int32_t r, cur;
    uint32_t kr_key, kcur, best_before;
    int have_best;
    /* stop at the budget or when every pool node is evaluated (Q7);
     * evaluations are distinct pool nodes, so |evaluated| == c */
    if (c == budget || c == C->m) break;
    do {
      if (C->starts != NULL) {
        if (j >= C->nstarts) goto done;    /* injected sequence exhausted */
        r = C->starts[j++];
      } else {
        int64_t idx = or_rng_perm(C->seed, (uint64_t)pid, (uint64_t)C->part, (uint64_t)j++, (uint64_t)C->m);
        if (idx < 0) goto done;            /* every pool node drawn (unreachable while c < m) */
        r = C->pool ? C->pool[idx] : (int32_t)idx;
      }
    } while (W->evaluated[r]);            /* Q4: redraw of an evaluated node is free */
    have_best = T->cnt > 0;
    best_before = have_best ? T->key[0] : 0;  /* s_max: most similar found so far */
    kr_key = key_of(C->S, q, store_point(C->S, r));
    ++c; ++st->starts;
    W->evaluated[r] = 1; W->keyv[r] = kr_key; W->touched[ntouched++] = r;
    list_insert(metric, T, kr_key, r);    /* Q5: a skipped start still enters top-k */
    /* P:81 expansion rule; Q3: the first start is never skipped */
    if (!first && have_best && skip_start(metric, kr_key, best_before, C->e_num, C->e_den)) {
      ++st->skipped;
      continue;
    }
    first = 0;
    cur = r; kcur = kr_key;

    /* ---- GNNS baseline walk: scan all k neighbours, move to the most similar one if it
     * improves on cur (ties -> the first in row order); same budget, restart and cache rules ---- */
    if (C->full_scan) {
      for (;;) {
        int t;
        int32_t best = -1;
        uint32_t kbest = 0;
        W->expanded[cur] = 1;
        ++st->expansions;
        for (t = 0; t < C->k; ++t) {
          int32_t v = C->rows[(size_t)cur * C->k + t];
          uint32_t kv;
          if (v < 0 || !in_pool(C, v)) continue;
          if (!W->evaluated[v]) {
            if (c == budget) goto done;  /* the over-budget evaluation is not performed */
            kv = key_of(C->S, q, store_point(C->S, v));
            ++c;
            W->evaluated[v] = 1; W->keyv[v] = kv; W->touched[ntouched++] = v;
            list_insert(metric, T, kv, v);
          } else {
            kv = W->keyv[v];
          }
          if (closer(metric, kv, kcur) && (best < 0 || closer(metric, kv, kbest))) { best = v; kbest = kv; }
        }
        if (best < 0) break;               /* local maximum: restart */
        cur = best; kcur = kbest;
        if (W->expanded[cur]) break;       /* Q9 (same argument: the re-walk repeats the same choices) */
      }
      continue;
    }
    /* ---- hill climbing with eager first-improvement descent ---- */
    for (;;) {
      int moved = 0, t;
      W->expanded[cur] = 1;
      ++st->expansions;
      for (t = 0; t < C->k; ++t) {       /* Q8: stored row order */
        int32_t v = C->rows[(size_t)cur * C->k + t];
        uint32_t kv;
        if (v < 0 || !in_pool(C, v)) continue;   /* Q10: edges leaving the pool are skipped */
        if (!W->evaluated[v]) {
          if (c == budget) goto done;    /* the over-budget evaluation is not performed */
          kv = key_of(C->S, q, store_point(C->S, v));
          ++c;
          W->evaluated[v] = 1; W->keyv[v] = kv; W->touched[ntouched++] = v;
          list_insert(metric, T, kv, v);
        } else {
          kv = W->keyv[v];               /* cached similarity: free */
        }
        if (closer(metric, kv, kcur)) {  /* first strictly better neighbour */
          cur = v; kcur = kv; moved = 1;
          break;
        }
      }
      if (!moved) break;                 /* local maximum: restart */
      if (W->expanded[cur]) break;       /* Q9: re-walking an expanded node adds nothing */
    }
  }
done:
  st->evals = c;
  for (i = 0; i < ntouched; ++i) {
    W->evaluated[W->touched[i]] = 0;
    W->expanded[W->touched[i]] = 0;
  }
  /* expanded nodes are always evaluated nodes, so the loop above clears both */
}

/* Public single search (used by pins).  pool may be NULL (pool = 0..m-1). */
int64_t or_ignns_search(int metric, int dim, const void *data, const uint64_t *off,
                        int64_t n_store, const int32_t *rows, int k,
                        const int32_t *pool, int64_t m, const uint8_t *part_of, int part,
                        const void *qdata, const uint32_t *qtok, int64_t qntok,
                        int kr, double speedup, uint64_t e_num, uint64_t e_den,
                        uint64_t seed, int64_t pid,
                        const int32_t *starts, int64_t nstarts,
                        int32_t *out_ids, uint32_t *out_keys, int64_t *out_stats4, int full_scan) {
  or_store S;
  or_search_cfg C;
  or_scratch W;
  or_list T;
  or_point q;
  or_search_stats st;
  int i;
  S.metric = metric; S.dim = dim;
  S.u8 = (const uint8_t *)data; S.f32 = (const float *)data;
  S.off = off; S.tok = (const uint32_t *)data;
  memset(&C, 0, sizeof C);
  C.S = &S; C.k = k; C.rows = rows; C.pool = pool; C.m = m;
  C.part_of = part_of; C.part = part; C.speedup = speedup;
  C.e_num = e_num; C.e_den = e_den; C.seed = seed;
  C.starts = starts; C.nstarts = nstarts; C.full_scan = full_scan;
  memset(&q, 0, sizeof q);
  q.u8 = (const uint8_t *)qdata; q.f32 = (const float *)qdata; q.tok = qtok; q.ntok = qntok;
  if (!scratch_init(&W, n_store)) return -5;
  T.cap = kr; T.cnt = 0; T.key = out_keys; T.id = out_ids;
  ignns(&C, q, pid, kr, &W, &T, &st);
  for (i = T.cnt; i < kr; ++i) { out_ids[i] = -1; out_keys[i] = 0; }
  scratch_free(&W);
  if (out_stats4) {
    out_stats4[0] = st.evals; out_stats4[1] = st.starts;
    out_stats4[2] = st.skipped; out_stats4[3] = st.expansions;
  }
  return T.cnt;
}

/* ------------------------------------------------------------------ */
/* Graph state shared by the batched and sequential insert paths.       */
/* The caller (Python, numpy) owns every array; capacity must hold      */
/* n_t + B rows.                                                        */
/* ------------------------------------------------------------------ */
typedef struct {
  int metric, dim, k;
  void *data;             /* store: u8 / f32 rows, or JAC tokens */
  uint64_t *off;          /* JAC offsets [cap+1] */
  int64_t n;              /* current graph size n_t */
  int32_t *ids;           /* [cap][k] */
  uint32_t *keys;         /* [cap][k] */
  /* partitioned graphs (P > 1 or partitioned == 1) */
  int P;                  /* 0 => unpartitioned */
  uint8_t *part_of;       /* [cap] */
  int32_t *members;       /* [P][member_cap], ascending ids */
  int64_t *member_cnt;    /* [P] */
  int64_t member_cap;
  const int32_t *medoids; /* [P] */
} or_graph;

typedef struct {
  double speedup;
  uint64_t e_num, e_den;
  int depth;
  uint64_t seed;
  int nthreads;
  int full_scan;          /* graph_search only: the GNNS baseline walk */
  int route;              /* 1: search only the partition of the nearest medoid (reading Q18's variant) */
} or_params;

typedef struct { int32_t node; uint32_t key; int32_t qid; } or_prop;

static or_store graph_store(const or_graph *G) {
  or_store S;
  S.metric = G->metric; S.dim = G->dim;
  S.u8 = (const uint8_t *)G->data; S.f32 = (const float *)G->data;
  S.off = G->off; S.tok = (const uint32_t *)G->data;
  return S;
}

/* Step 1 of a batch (Alg. 1 "Search"; partitioned: Alg. 3):
 * result C_i = top-k over the P per-partition searches.  */
typedef struct {
  const or_graph *G;
  const or_params *prm;
  int64_t first_query;     /* global id of batch point 0 (RNG stream key) */
  int64_t b0, b1;          /* batch slice handled by this worker */
  int32_t *cand_ids;       /* [B][k] */
  uint32_t *cand_keys;
  int64_t *stats;          /* [B][4] summed over partitions */
  const int64_t *qpoint;   /* store index of each batch point, or -1 for external */
  const void *qdata;       /* external queries (graph_search) */
  const uint64_t *qoff;
  int pid_is_index;        /* graph_search: stream key = query index */
  int kr;                  /* result width (graph_search may ask kr != k) */
  int rc;
} or_search_job;

static int nearest_medoid(const or_graph *G, or_point x);

static void *search_worker(void *arg) {
  or_search_job *J = (or_search_job *)arg;
  const or_graph *G = J->G;
  or_store S = graph_store(G);
  or_scratch W;
  uint32_t *tk = (uint32_t *)malloc(sizeof(uint32_t) * J->kr);
  int32_t *ti = (int32_t *)malloc(sizeof(int32_t) * J->kr);
  int64_t b;
  if (!scratch_init(&W, G->n) || !tk || !ti) { J->rc = -5; return NULL; }
  for (b = J->b0; b < J->b1; ++b) {
    or_point q;
    or_list Cq;
    int64_t pid = J->pid_is_index ? b : J->first_query + b;
    int p, nparts = G->P > 0 ? G->P : 1, t;
    if (J->qpoint) q = store_point(&S, J->qpoint[b]);
    else {
      memset(&q, 0, sizeof q);
      if (G->metric == OR_U8) q.u8 = (const uint8_t *)J->qdata + (size_t)b * G->dim;
      else if (G->metric == OR_F32) q.f32 = (const float *)J->qdata + (size_t)b * G->dim;
      else { q.tok = (const uint32_t *)J->qdata + J->qoff[b]; q.ntok = (int64_t)(J->qoff[b + 1] - J->qoff[b]); }
    }
    Cq.cap = J->kr; Cq.cnt = 0; Cq.key = J->cand_keys + b * J->kr; Cq.id = J->cand_ids + b * J->kr;
    for (t = 0; t < 4; ++t) J->stats[b * 4 + t] = 0;
    {
      int p0 = 0, p1 = nparts;
      /* routing variant (Q18: "queries sent to partitions by medoid distance"): only the partition of
       * the nearest medoid (ties -> lowest p, as placement) is searched */
      if (J->prm->route && G->P > 0) { p0 = nearest_medoid(G, q); p1 = p0 + 1; }
    for (p = p0; p < p1; ++p) {
      or_search_cfg C;
      or_list T;
      or_search_stats st;
      memset(&C, 0, sizeof C);
      C.S = &S; C.k = G->k; C.rows = G->ids;
      if (G->P > 0) {
        C.pool = G->members + (size_t)p * G->member_cap;
        C.m = G->member_cnt[p];
        C.part_of = G->part_of; C.part = p;
      } else {
        C.pool = NULL; C.m = G->n; C.part_of = NULL; C.part = 0;
      }
      C.speedup = J->prm->speedup; C.e_num = J->prm->e_num; C.e_den = J->prm->e_den;
      C.seed = J->prm->seed;
      C.full_scan = J->prm->full_scan;
      T.cap = J->kr; T.cnt = 0; T.key = tk; T.id = ti;
      ignns(&C, q, pid, J->kr, &W, &T, &st);
      /* Alg. 3: keep the k most similar of the k*p candidates */
      for (t = 0; t < T.cnt; ++t) list_insert(G->metric, &Cq, T.key[t], T.id[t]);
      J->stats[b * 4 + 0] += st.evals; J->stats[b * 4 + 1] += st.starts;
      J->stats[b * 4 + 2] += st.skipped; J->stats[b * 4 + 3] += st.expansions;
    }
    }
    for (t = Cq.cnt; t < J->kr; ++t) { Cq.id[t] = -1; Cq.key[t] = 0; }
  }
  scratch_free(&W);
  free(tk); free(ti);
  J->rc = 0;
  return NULL;
}

static int run_searches(or_search_job *proto, int64_t B, int nthreads) {
  int t, rc = 0;
  or_search_job *jobs;
  pthread_t *th;
  if (nthreads < 1) nthreads = 1;
  if (nthreads > B) nthreads = (int)(B > 0 ? B : 1);
  jobs = (or_search_job *)calloc(nthreads, sizeof *jobs);
  th = (pthread_t *)calloc(nthreads, sizeof *th);
  for (t = 0; t < nthreads; ++t) {
    jobs[t] = *proto;
    jobs[t].b0 = B * t / nthreads;
    jobs[t].b1 = B * (t + 1) / nthreads;
    if (nthreads == 1) search_worker(&jobs[t]);
    else pthread_create(&th[t], NULL, search_worker, &jobs[t]);
  }
  for (t = 0; t < nthreads; ++t) {
    if (nthreads > 1) pthread_join(th[t], NULL);
    if (jobs[t].rc) rc = jobs[t].rc;
  }
  free(jobs); free(th);
  return rc;
}

/* Update ball of Alg. 2 with dedup (Q12) over the snapshot
 * (Q13): L1 = ids of C(x); for d = 1..DEPTH every node v of L_d is
 * evaluated and, if d < DEPTH, its unseen snapshot neighbours form
 * L_{d+1}.  A proposal (v, D, id_x) is emitted when (D, id_x) precedes
 * row_v[k-1] in edge order (Q14).  Returns the number of ball nodes. */
static int64_t update_ball(const or_graph *G, or_point x, int32_t idx, const int32_t *C_ids,
                           int depth, uint8_t *seen, int32_t *buf, int64_t bufcap,
                           or_prop *props, int64_t *nprops, int32_t qid) {
  or_store S = graph_store(G);
  const int k = G->k;
  int64_t lo = 0, hi = 0, i, t, nball = 0;
  int d;
  for (t = 0; t < k; ++t) {
    int32_t v = C_ids[t];
    if (v < 0 || seen[v]) continue;
    seen[v] = 1; buf[hi++] = v;
  }
  for (d = 1; d <= depth; ++d) {
    int64_t nhi = hi;
    for (i = lo; i < hi; ++i) {
      int32_t v = buf[i];
      uint32_t D;
      if (d < depth) {
        for (t = 0; t < k; ++t) {
          int32_t u = G->ids[(size_t)v * k + t];
          if (u < 0 || seen[u]) continue;
          if (nhi >= bufcap) return -1;
          seen[u] = 1; buf[nhi++] = u;
        }
      }
      D = key_of(&S, store_point(&S, v), x);   /* v's similarity to x, as v's row holds it */
      ++nball;
      if (precedes(G->metric, D, idx, G->keys[(size_t)v * k + k - 1], G->ids[(size_t)v * k + k - 1])) {
        props[*nprops].node = v; props[*nprops].key = D; props[*nprops].qid = qid;
        ++*nprops;
      }
    }
    lo = hi; hi = nhi;
  }
  for (i = 0; i < hi; ++i) seen[buf[i]] = 0;
  return nball;
}

static int g_sort_metric;
static int prop_cmp(const void *pa, const void *pb) {
  const or_prop *a = (const or_prop *)pa, *b = (const or_prop *)pb;
  if (a->qid != b->qid) return a->qid < b->qid ? -1 : 1;
  if (closer(g_sort_metric, a->key, b->key)) return -1;
  if (closer(g_sort_metric, b->key, a->key)) return 1;
  if (a->node != b->node) return a->node < b->node ? -1 : 1;
  return 0;
}

/* Nearest medoid (A8): argmin_p D(x, medoid_p), ties -> lowest p. */
static int nearest_medoid(const or_graph *G, or_point x) {
  or_store S = graph_store(G);
  int p, best = 0;
  uint32_t kb = 0;
  for (p = 0; p < G->P; ++p) {
    uint32_t kp = key_of(&S, x, store_point(&S, G->medoids[p]));
    if (p == 0 || closer(G->metric, kp, kb)) { best = p; kb = kp; }
  }
  return best;
}

/* ------------------------------------------------------------------ */
/* graph_insert_batch semantics (C.2): the batch's points must already  */
/* be stored at rows n_t .. n_t+B-1 of the store (ids n_t+i).           */
/* out_stats: [B][6] = evals, starts, skipped, expansions, ball, props. */
/* ------------------------------------------------------------------ */
int or_insert_batch(int metric, int dim, void *data, uint64_t *off, int k,
                    int64_t n_t, int32_t *ids, uint32_t *keys,
                    int P, uint8_t *part_of, int32_t *members, int64_t *member_cnt,
                    int64_t member_cap, const int32_t *medoids,
                    int64_t B, double speedup, uint64_t e_num, uint64_t e_den, int depth,
                    uint64_t seed, int nthreads, int64_t *out_stats, int route) {
  or_graph G;
  or_params prm;
  or_search_job J;
  or_store S;
  int32_t *cand_ids;
  uint32_t *cand_keys;
  int64_t *sstats, *qpoint, i, j, t, nprops = 0, bufcap;
  or_prop *props;
  uint8_t *seen;
  int32_t *buf;
  int rc;

  memset(&G, 0, sizeof G);
  G.metric = metric; G.dim = dim; G.k = k; G.data = data; G.off = off; G.n = n_t;
  G.ids = ids; G.keys = keys; G.P = P; G.part_of = part_of; G.members = members;
  G.member_cnt = member_cnt; G.member_cap = member_cap; G.medoids = medoids;
  prm.speedup = speedup; prm.e_num = e_num; prm.e_den = e_den; prm.depth = depth;
  prm.seed = seed; prm.nthreads = nthreads; prm.full_scan = 0; prm.route = route;
  S = graph_store(&G);
  if (B <= 0) return 0;

  cand_ids = (int32_t *)malloc(sizeof(int32_t) * B * k);
  cand_keys = (uint32_t *)malloc(sizeof(uint32_t) * B * k);
  sstats = (int64_t *)calloc((size_t)B * 4, sizeof(int64_t));
  qpoint = (int64_t *)malloc(sizeof(int64_t) * B);
  for (i = 0; i < B; ++i) qpoint[i] = n_t + i;

  /* 1. search every point of the batch on the snapshot G_t (graph size n_t) */
  memset(&J, 0, sizeof J);
  J.G = &G; J.prm = &prm; J.first_query = n_t; J.kr = k; J.cand_ids = cand_ids; J.cand_keys = cand_keys;
  J.stats = sstats; J.qpoint = qpoint; J.pid_is_index = 0;
  rc = run_searches(&J, B, nthreads);
  if (rc) { free(cand_ids); free(cand_keys); free(sstats); free(qpoint); return rc; }

  /* 3. update balls over the snapshot -> proposals (Alg. 2) */
  /* ball size <= k + k^2 + ... + k^DEPTH, and <= n_t */
  bufcap = 1;
  for (t = 0, i = 1; t < depth && bufcap < n_t; ++t) { i *= k; bufcap += i; }
  if (bufcap > n_t) bufcap = n_t;
  props = (or_prop *)malloc(sizeof(or_prop) * (size_t)(B * bufcap + 1));
  seen = (uint8_t *)calloc((size_t)n_t + 1, 1);
  buf = (int32_t *)malloc(sizeof(int32_t) * (size_t)(bufcap + 1));
  for (i = 0; i < B; ++i) {
    int64_t nb = update_ball(&G, store_point(&S, n_t + i), (int32_t)(n_t + i), cand_ids + i * k,
                             depth, seen, buf, bufcap, props, &nprops, (int32_t)i);
    if (out_stats) out_stats[i * 6 + 4] = nb;
  }
  free(seen); free(buf);

  /* 2. new rows: top-k of C_i u {(D(x_i, x_j), n_t + j) : j != i} (Q15) */
  for (i = 0; i < B; ++i) {
    or_list L;
    L.cap = k; L.cnt = 0; L.key = keys + (size_t)(n_t + i) * k; L.id = ids + (size_t)(n_t + i) * k;
    for (t = 0; t < k; ++t)
      if (cand_ids[i * k + t] >= 0) list_insert(metric, &L, cand_keys[i * k + t], cand_ids[i * k + t]);
    for (j = 0; j < B; ++j) {
      if (j == i) continue;
      list_insert(metric, &L, key_of(&S, store_point(&S, n_t + i), store_point(&S, n_t + j)), (int32_t)(n_t + j));
    }
    for (t = L.cnt; t < k; ++t) { L.id[t] = -1; L.key[t] = 0; }
  }

  /* 4. apply proposals in (qid, key, node) order: row_v = top-k(row_v u proposals) */
  g_sort_metric = metric;
  qsort(props, (size_t)nprops, sizeof(or_prop), prop_cmp);
  for (i = 0; i < nprops; ++i) {
    or_list L;
    int32_t v = props[i].node;
    L.cap = k; L.cnt = k; L.key = keys + (size_t)v * k; L.id = ids + (size_t)v * k;
    list_insert(metric, &L, props[i].key, (int32_t)(n_t + props[i].qid));
  }
  if (out_stats) {
    for (i = 0; i < B; ++i) {
      for (t = 0; t < 4; ++t) out_stats[i * 6 + t] = sstats[i * 4 + t];
      out_stats[i * 6 + 5] = 0;
    }
    for (i = 0; i < nprops; ++i) out_stats[props[i].qid * 6 + 5] += 1;
  }
  free(props);

  /* 5. placement of each new point at its nearest medoid (Alg. 5) */
  if (P > 0) {
    for (i = 0; i < B; ++i) {
      int p = nearest_medoid(&G, store_point(&S, n_t + i));
      if (member_cnt[p] >= member_cap) { rc = -8; break; }
      part_of[n_t + i] = (uint8_t)p;
      members[(size_t)p * member_cap + member_cnt[p]++] = (int32_t)(n_t + i);
    }
  }
  free(cand_ids); free(cand_keys); free(sstats); free(qpoint);
  return rc;
}

/* ------------------------------------------------------------------ */
/* Literal sequential add: Alg. 1 + Alg. 2 as   */
/* printed (Q / Q_next lists, re-enqueueing allowed), for one new node   */
/* stored at row n_t.  Only two choices are added to the printed text:   */
/* the new node itself is never enqueued (no self-edges) and a node's    */
/* list rejects an id it already holds.  Used to pin B=1 of the batched  */
/* semantics (C.2 "With B = 1, steps 1-4 are exactly Alg. 1 + Alg. 2").  */
/* ------------------------------------------------------------------ */
int or_insert_sequential(int metric, int dim, void *data, uint64_t *off, int k,
                         int64_t n_t, int32_t *ids, uint32_t *keys,
                         double speedup, uint64_t e_num, uint64_t e_den, int depth,
                         uint64_t seed, int64_t *out_stats) {
  or_graph G;
  or_params prm;
  or_search_job J;
  or_store S;
  int64_t qpoint = n_t, sstats[4], qcap, qn, nn, i, t;
  int32_t *Q, *Qn, *tmp;
  int32_t newid = (int32_t)n_t;
  or_point x;
  int d, rc;
  memset(&G, 0, sizeof G);
  G.metric = metric; G.dim = dim; G.k = k; G.data = data; G.off = off; G.n = n_t;
  G.ids = ids; G.keys = keys;
  prm.speedup = speedup; prm.e_num = e_num; prm.e_den = e_den; prm.depth = depth;
  prm.seed = seed; prm.nthreads = 1; prm.full_scan = 0; prm.route = 0;
  S = graph_store(&G);
  x = store_point(&S, n_t);

  /* neighborlist = iGNNS(graph, new, k)   -- Search */
  memset(&J, 0, sizeof J);
  J.G = &G; J.prm = &prm; J.first_query = n_t; J.kr = k;
  J.cand_ids = ids + (size_t)n_t * k; J.cand_keys = keys + (size_t)n_t * k;
  J.stats = sstats; J.qpoint = &qpoint; J.pid_is_index = 0;
  J.b0 = 0; J.b1 = 1;
  search_worker(&J);
  rc = J.rc;
  if (rc) return rc;

  /* Update(graph, new, neighborlist) -- Alg. 2 */
  /* the printed Alg. 2 re-enqueues: level d holds at most k^d entries */
  qcap = 1;
  for (d = 0, t = 1; d <= depth; ++d) {
    t *= k; qcap += t;
    if (qcap > (1ll << 28)) return -1;   /* literal queues too large: use the batched path */
  }
  Q = (int32_t *)malloc(sizeof(int32_t) * (size_t)qcap);
  Qn = (int32_t *)malloc(sizeof(int32_t) * (size_t)qcap);
  qn = 0;
  for (t = 0; t < k; ++t)                       /* Q.addAll(neighborlist) */
    if (ids[(size_t)n_t * k + t] >= 0) Q[qn++] = ids[(size_t)n_t * k + t];
  if (out_stats) { out_stats[4] = 0; out_stats[5] = 0; }
  for (d = 1; d <= depth; ++d) {                /* for d in 1..DEPTH */
    nn = 0;
    for (i = 0; i < qn; ++i) {                  /* while Q.hasNodes(): node = Q.pop() */
      int32_t node = Q[i];
      uint32_t D;
      or_list L;
      for (t = 0; t < k; ++t) {                 /* Q_next.addAll(neighbors of node) */
        int32_t u = ids[(size_t)node * k + t];
        if (u < 0 || u == newid) continue;
        Qn[nn++] = u;
      }
      D = key_of(&S, store_point(&S, node), x); /* compute similarity(new, node), as node's row holds it */
      if (out_stats) out_stats[4] += 1;
      L.cap = k; L.cnt = k; L.key = keys + (size_t)node * k; L.id = ids + (size_t)node * k;
      if (list_insert(metric, &L, D, newid) && out_stats) out_stats[5] += 1;  /* if needed, add new */
    }
    tmp = Q; Q = Qn; Qn = tmp; qn = nn;         /* Q.addAll(Q_next); Q_next.empty() */
  }
  free(Q); free(Qn);
  if (out_stats) for (t = 0; t < 4; ++t) out_stats[t] = sstats[t];
  return 0;
}

/* ------------------------------------------------------------------ */
/* graph_search: step 1 only, stream key = query index (C.2).           */
/* ------------------------------------------------------------------ */
int or_graph_search(int metric, int dim, void *data, uint64_t *off, int k,
                    int64_t n_t, int32_t *ids, uint32_t *keys,
                    int P, uint8_t *part_of, int32_t *members, int64_t *member_cnt,
                    int64_t member_cap,
                    const void *qdata, const uint64_t *qoff, int64_t nq, int kr,
                    double speedup, uint64_t e_num, uint64_t e_den, uint64_t seed,
                    int nthreads, int32_t *out_ids, uint32_t *out_keys, int64_t *out_stats4, int full_scan,
                    const int32_t *medoids, int route) {
  or_graph G;
  or_params prm;
  or_search_job J;
  int rc;
  memset(&G, 0, sizeof G);
  G.metric = metric; G.dim = dim; G.k = k; G.data = data; G.off = off; G.n = n_t;
  G.ids = ids; G.keys = keys; G.P = P; G.part_of = part_of; G.members = members;
  G.member_cnt = member_cnt; G.member_cap = member_cap;
  prm.speedup = speedup; prm.e_num = e_num; prm.e_den = e_den; prm.depth = 1;
  prm.seed = seed; prm.nthreads = nthreads; prm.full_scan = full_scan; prm.route = route;
  G.medoids = medoids;
  memset(&J, 0, sizeof J);
  J.G = &G; J.prm = &prm; J.first_query = 0; J.kr = kr; J.cand_ids = out_ids; J.cand_keys = out_keys;
  J.stats = out_stats4; J.qpoint = NULL; J.qdata = qdata; J.qoff = qoff; J.pid_is_index = 1;
  rc = run_searches(&J, nq, nthreads);
  return rc;
}

/* ------------------------------------------------------------------ */
/* Balanced k-medoids, Alg. 4, readings Q21-Q23.            */
/* ------------------------------------------------------------------ */

/* Assign comparison: is cluster a's score sim(m_a,u)*w_a strictly above b's?
 * w = 1 - size/cap, s = 1/(1+D) (L2) or i/u (JAC); cross-multiplied. */
static int assign_better(int metric, uint32_t ka, int64_t sa, uint32_t kb, int64_t sb, int64_t cap) {
  if (metric == OR_U8) {
    /* (cap-sa)/(1+Da) > (cap-sb)/(1+Db)  <=>  (cap-sa)(1+Db) > (cap-sb)(1+Da) */
    unsigned __int128 l = (unsigned __int128)(uint64_t)(cap - sa) * (1ull + kb);
    unsigned __int128 r = (unsigned __int128)(uint64_t)(cap - sb) * (1ull + ka);
    return l > r;
  } else if (metric == OR_F32) {
    volatile double l = (double)(cap - sa) * (1.0 + (double)bits_float(kb));
    volatile double r = (double)(cap - sb) * (1.0 + (double)bits_float(ka));
    return l > r;
  } else {
    /* i_a (cap-sa) / u_a > i_b (cap-sb) / u_b */
    int64_t ia = ka >> 16, ua = ka & 0xFFFF, ib = kb >> 16, ub = kb & 0xFFFF;
    return ia * (cap - sa) * ub > ib * (cap - sb) * ua;
  }
}

static int assign_equal(int metric, uint32_t ka, int64_t sa, uint32_t kb, int64_t sb, int64_t cap) {
  return !assign_better(metric, ka, sa, kb, sb, cap) && !assign_better(metric, kb, sb, ka, sa, cap);
}

/* hop sum of candidate c over cluster members (undirected, induced); unreachable = |C| */
static int64_t hop_sum(int64_t c, const int32_t *mem, int64_t sz,
                       const int64_t *adj_off, const int32_t *adj, int32_t *dist, int32_t *queue) {
  int64_t qh = 0, qt = 0, s = 0, i;
  for (i = 0; i < sz; ++i) dist[i] = -1;
  dist[c] = 0; queue[qt++] = (int32_t)c;
  while (qh < qt) {
    int32_t u = queue[qh++];
    for (i = adj_off[u]; i < adj_off[u + 1]; ++i) {
      int32_t w = adj[i];
      if (dist[w] < 0) { dist[w] = dist[u] + 1; queue[qt++] = w; }
    }
  }
  for (i = 0; i < sz; ++i) s += dist[i] >= 0 ? dist[i] : sz;
  (void)mem;
  return s;
}

/* The update step of Alg. 4 for assignment part[0..n): per cluster, the member minimising the
 * hop sum in the cluster-induced undirected view (Q29) -- every member when |C| <= exact_limit, else
 * (Q22) the current medoid (if a member) and ncand-1 draws of stream (seed, tag, it*P + p, j).
 * Unreachable members cost |C|; ties -> smaller id.  Empty clusters keep their medoid.  Returns the
 * total hop sum of the chosen medoids; scratch arrays are sized n (adj: 2nk). */
static int64_t update_medoids(int64_t n, int k, const int32_t *ids, int P, const uint8_t *part,
                              const int32_t *med, int32_t *newmed, uint64_t seed, uint64_t tag, int64_t it,
                              int64_t exact_limit, int ncand, int64_t *local, int32_t *mem, int32_t *deg,
                              int64_t *adj_off, int32_t *adj, int32_t *dist, int32_t *queue) {
  int64_t cost = 0, i;
  int p, j;
  for (p = 0; p < P; ++p) {
    int64_t sz = 0, bestc = -1, bests = 0, c;
    for (i = 0; i < n; ++i) if (part[i] == p) { local[i] = sz; mem[sz++] = (int32_t)i; } else local[i] = -1;
    /* cluster-induced undirected adjacency (Q29) */
    for (i = 0; i < sz; ++i) deg[i] = 0;
    for (i = 0; i < sz; ++i) {
      int t;
      for (t = 0; t < k; ++t) {
        int32_t u = ids[(size_t)mem[i] * k + t];
        if (u >= 0 && local[u] >= 0) { deg[i]++; deg[local[u]]++; }
      }
    }
    adj_off[0] = 0;
    for (i = 0; i < sz; ++i) adj_off[i + 1] = adj_off[i] + deg[i];
    for (i = 0; i < sz; ++i) deg[i] = 0;
    for (i = 0; i < sz; ++i) {
      int t;
      for (t = 0; t < k; ++t) {
        int32_t u = ids[(size_t)mem[i] * k + t];
        if (u >= 0 && local[u] >= 0) {
          int64_t lu = local[u];
          adj[adj_off[i] + deg[i]++] = (int32_t)lu;
          adj[adj_off[lu] + deg[lu]++] = (int32_t)i;
        }
      }
    }
    if (sz == 0) { newmed[p] = med[p]; continue; }
    if (sz <= exact_limit) {
      for (c = 0; c < sz; ++c) {
        int64_t s = hop_sum(c, mem, sz, adj_off, adj, dist, queue);
        if (bestc < 0 || s < bests) { bestc = c; bests = s; }   /* ties -> smaller id (ascending scan) */
      }
    } else {
      /* Q22: candidates = {current medoid if member} u ncand-1 seeded draws */
      int64_t cnt = 0;
      int32_t *cl = (int32_t *)malloc(sizeof(int32_t) * ncand);
      if (local[med[p]] >= 0) cl[cnt++] = (int32_t)local[med[p]];
      for (j = 0; j < ncand - 1; ++j)
        cl[cnt++] = (int32_t)or_rng_draw(seed, tag, (uint64_t)(it * P + p), (uint64_t)j, (uint64_t)sz);
      for (j = 0; j < cnt; ++j) {
        int64_t s;
        c = cl[j];
        s = hop_sum(c, mem, sz, adj_off, adj, dist, queue);
        if (bestc < 0 || s < bests || (s == bests && mem[c] < mem[bestc])) { bestc = c; bests = s; }
      }
      free(cl);
    }
    newmed[p] = mem[bestc];
    cost += bests;
  }
  return cost;
}

/* part_out[n], medoids_io[P] (output), cost_out[max_iter+1] (costs of accepted
 * iterations, -1 padded).  Returns number of accepted iterations or <0 on error. */
int or_partition_kmedoids(int metric, int dim, const void *data, const uint64_t *off,
                          int64_t n, int k, const int32_t *ids,
                          int P, double imbalance, int max_iter, uint64_t seed,
                          uint8_t *part_out, int32_t *medoids_out, int64_t *cost_out,
                          int64_t exact_limit, int ncand, const int32_t *init_medoids) {
  or_store S;
  int64_t cap, i, it, accepted = 0, prev_cost = -1;
  int32_t *med = (int32_t *)malloc(sizeof(int32_t) * P);
  int32_t *newmed = (int32_t *)malloc(sizeof(int32_t) * P);
  uint8_t *part = (uint8_t *)malloc((size_t)n);
  int64_t *size = (int64_t *)malloc(sizeof(int64_t) * P);
  int64_t *local = (int64_t *)malloc(sizeof(int64_t) * n);
  int32_t *dist = (int32_t *)malloc(sizeof(int32_t) * n);
  int32_t *queue = (int32_t *)malloc(sizeof(int32_t) * n);
  int32_t *mem = (int32_t *)malloc(sizeof(int32_t) * n);
  int64_t *adj_off = (int64_t *)malloc(sizeof(int64_t) * (n + 1));
  int32_t *adj = (int32_t *)malloc(sizeof(int32_t) * (size_t)(2 * n * k + 1));
  int32_t *deg = (int32_t *)malloc(sizeof(int32_t) * n);
  uint32_t *dk = (uint32_t *)malloc(sizeof(uint32_t) * P);
  int p, j;
  S.metric = metric; S.dim = dim;
  S.u8 = (const uint8_t *)data; S.f32 = (const float *)data;
  S.off = off; S.tok = (const uint32_t *)data;

  if (P < 1 || n < P) return -1;
  cap = (int64_t)ceil((double)n * imbalance / (double)P);   /* F4 capacity, ceil */
  if (cap * P < n) return -4;
  if (cost_out) for (i = 0; i <= max_iter; ++i) cost_out[i] = -1;

  /* Randomly pick P initial medoids (Alg. 4 line 1): distinct draws, duplicates skipped */
  if (init_medoids) {
    for (p = 0; p < P; ++p) med[p] = init_medoids[p];
  } else {
    int got = 0;
    uint64_t jd = 0;
    while (got < P) {
      int32_t cnd = (int32_t)or_rng_draw(seed, 0xFFFFFFFFull, 0, jd++, (uint64_t)n);
      int dup = 0;
      for (j = 0; j < got; ++j) if (med[j] == cnd) dup = 1;
      if (!dup) med[got++] = cnd;
    }
  }

  for (it = 0; it < max_iter; ++it) {
    int64_t cost = 0;
    int changed = 0;
    /* ---- Assign (greedy, nodes in ascending id, Q21 c = 1) ---- */
    for (p = 0; p < P; ++p) size[p] = 0;
    for (i = 0; i < n; ++i) {
      int best = -1;
      for (p = 0; p < P; ++p) dk[p] = key_of(&S, store_point(&S, i), store_point(&S, med[p]));
      for (p = 0; p < P; ++p) {
        if (size[p] >= cap) continue;           /* full clusters are ineligible */
        if (best < 0 || assign_better(metric, dk[p], size[p], dk[best], size[best], cap)) best = p;
        else if (assign_equal(metric, dk[p], size[p], dk[best], size[best], cap)) {
          if (size[p] < size[best] || (size[p] == size[best] && med[p] < med[best])) best = p;
        }
      }
      part[i] = (uint8_t)best;
      size[best]++;
    }
    /* ---- Update: new medoid = member minimising the hop sum ---- */
    cost = update_medoids(n, k, ids, P, part, med, newmed, seed, 0xFFFFFFFEull, it, exact_limit, ncand,
                          local, mem, deg, adj_off, adj, dist, queue);
    /* Q23: accept only if the hop-sum cost does not rise */
    if (it > 0 && cost > prev_cost) break;
    memcpy(part_out, part, (size_t)n);
    if (cost_out) cost_out[accepted] = cost;
    accepted++;
    prev_cost = cost;
    for (p = 0; p < P; ++p) if (newmed[p] != med[p]) changed = 1;
    memcpy(med, newmed, sizeof(int32_t) * P);
    if (!changed) break;
  }
  memcpy(medoids_out, med, sizeof(int32_t) * P);
  free(med); free(newmed); free(part); free(size); free(local); free(dist); free(queue);
  free(mem); free(adj_off); free(adj); free(deg); free(dk);
  return (int)accepted;
}

/* Alg. 5's last step, "compute new medoids" (F5): the update step of Alg. 4
 * on the current partition part_of[0..n) -- nodes keep their partitions; medoids_io[P] in/out.
 * Candidate draws use stream (seed, 0xFFFFFFFD, epoch*P + p, j).  Returns 0, the total hop sum in
 * *cost_out. */
int or_recompute_medoids(int64_t n, int k, const int32_t *ids, int P, const uint8_t *part_of, int32_t *medoids_io,
                         uint64_t seed, int64_t epoch, int64_t exact_limit, int ncand, int64_t *cost_out) {
  int64_t *local = (int64_t *)malloc(sizeof(int64_t) * n);
  int32_t *dist = (int32_t *)malloc(sizeof(int32_t) * n);
  int32_t *queue = (int32_t *)malloc(sizeof(int32_t) * n);
  int32_t *mem = (int32_t *)malloc(sizeof(int32_t) * n);
  int64_t *adj_off = (int64_t *)malloc(sizeof(int64_t) * (n + 1));
  int32_t *adj = (int32_t *)malloc(sizeof(int32_t) * (size_t)(2 * n * k + 1));
  int32_t *deg = (int32_t *)malloc(sizeof(int32_t) * n);
  int32_t *newmed = (int32_t *)malloc(sizeof(int32_t) * P);
  int64_t cost = update_medoids(n, k, ids, P, part_of, medoids_io, newmed, seed, 0xFFFFFFFDull, epoch, exact_limit,
                                ncand, local, mem, deg, adj_off, adj, dist, queue);
  memcpy(medoids_io, newmed, sizeof(int32_t) * P);
  if (cost_out) *cost_out = cost;
  free(local); free(dist); free(queue); free(mem); free(adj_off); free(adj); free(deg); free(newmed);
  return 0;
}

/* ------------------------------------------------------------------ */
/* Small exported wrappers used by the pins.                           */
/* ------------------------------------------------------------------ */
uint32_t or_key(int metric, int dim, const void *a, int64_t na, const void *b, int64_t nb) {
  or_store S;
  or_point pa, pb;
  memset(&S, 0, sizeof S);
  S.metric = metric; S.dim = dim;
  memset(&pa, 0, sizeof pa); memset(&pb, 0, sizeof pb);
  pa.u8 = (const uint8_t *)a; pa.f32 = (const float *)a; pa.tok = (const uint32_t *)a; pa.ntok = na;
  pb.u8 = (const uint8_t *)b; pb.f32 = (const float *)b; pb.tok = (const uint32_t *)b; pb.ntok = nb;
  return key_of(&S, pa, pb);
}
int or_closer(int metric, uint32_t a, uint32_t b) { return closer(metric, a, b); }
int or_precedes(int metric, uint32_t ka, int64_t ida, uint32_t kb, int64_t idb) {
  return precedes(metric, ka, ida, kb, idb);
}
int or_skip(int metric, uint32_t kr, uint32_t kbest, uint64_t num, uint64_t den) {
  return skip_start(metric, kr, kbest, num, den);
}
int or_nearest_medoid(int metric, int dim, const void *data, const uint64_t *off,
                      const int32_t *medoids, int P, const void *x, int64_t nx) {
  or_graph G;
  or_point px;
  memset(&G, 0, sizeof G);
  G.metric = metric; G.dim = dim; G.data = (void *)data; G.off = (uint64_t *)off;
  G.P = P; G.medoids = medoids;
  memset(&px, 0, sizeof px);
  px.u8 = (const uint8_t *)x; px.f32 = (const float *)x; px.tok = (const uint32_t *)x; px.ntok = nx;
  return nearest_medoid(&G, px);
}

/* ------------------------------------------------------------------ */
/* Staged batch (the same steps as or_insert_batch, split the way a     */
/* distributed run splits them: searches per partition range, balls    */
/* per query range, then one commit).  Used by the multi-process tests. */
/* ------------------------------------------------------------------ */
/* per-partition candidates of batch points stored at rows n_t+b, b in [0,B), for partitions
 * [plo, phi): out [B][phi-plo][k] (-1/0 padded) */
int or_stage_search(int metric, int dim, void *data, uint64_t *off, int k, int64_t n_t, int32_t *ids,
                    uint32_t *keys, int P, uint8_t *part_of, int32_t *members, int64_t *member_cnt,
                    int64_t member_cap, int64_t B, int plo, int phi, double speedup, uint64_t e_num,
                    uint64_t e_den, uint64_t seed, int32_t *out_ids, uint32_t *out_keys, int64_t *out_evals) {
  or_graph G;
  or_store S;
  or_scratch W;
  int64_t b;
  int p, t, np = phi - plo;
  memset(&G, 0, sizeof G);
  G.metric = metric; G.dim = dim; G.k = k; G.data = data; G.off = off; G.n = n_t;
  G.ids = ids; G.keys = keys; G.P = P; G.part_of = part_of; G.members = members;
  G.member_cnt = member_cnt; G.member_cap = member_cap;
  S = graph_store(&G);
  if (!scratch_init(&W, n_t)) return -5;
  for (b = 0; b < B; ++b) {
    for (p = plo; p < phi; ++p) {
      or_search_cfg C;
      or_list T;
      or_search_stats st;
      memset(&C, 0, sizeof C);
      C.S = &S; C.k = k; C.rows = ids;
      if (P > 0) {
        C.pool = members + (size_t)p * member_cap; C.m = member_cnt[p]; C.part_of = part_of; C.part = p;
      } else {
        C.pool = NULL; C.m = n_t; C.part_of = NULL; C.part = 0;
      }
      C.speedup = speedup; C.e_num = e_num; C.e_den = e_den; C.seed = seed;
      T.cap = k; T.cnt = 0;
      T.key = out_keys + ((size_t)b * np + (p - plo)) * k;
      T.id = out_ids + ((size_t)b * np + (p - plo)) * k;
      ignns(&C, store_point(&S, n_t + b), n_t + b, k, &W, &T, &st);
      for (t = T.cnt; t < k; ++t) { T.id[t] = -1; T.key[t] = 0; }
      if (out_evals) *out_evals += st.evals;
    }
  }
  scratch_free(&W);
  return 0;
}

/* update balls of queries [qlo, qhi) given their search results C [B][k] (all B):
 * props [qhi-qlo][ballmax] as (node, key) int pairs, counts [qhi-qlo] */
int or_stage_ball(int metric, int dim, void *data, uint64_t *off, int k, int64_t n_t, int32_t *ids,
                  uint32_t *keys, const int32_t *C_ids, int64_t qlo, int64_t qhi, int depth, int64_t ballmax,
                  int32_t *props, int32_t *prop_cnt) {
  or_graph G;
  or_store S;
  uint8_t *seen;
  int32_t *buf;
  or_prop *tmp;
  int64_t q, i;
  memset(&G, 0, sizeof G);
  G.metric = metric; G.dim = dim; G.k = k; G.data = data; G.off = off; G.n = n_t;
  G.ids = ids; G.keys = keys;
  S = graph_store(&G);
  seen = (uint8_t *)calloc((size_t)n_t + 1, 1);
  buf = (int32_t *)malloc(sizeof(int32_t) * (size_t)(ballmax + 1));
  tmp = (or_prop *)malloc(sizeof(or_prop) * (size_t)(ballmax + 1));
  for (q = qlo; q < qhi; ++q) {
    int64_t np = 0;
    update_ball(&G, store_point(&S, n_t + q), (int32_t)(n_t + q), C_ids + q * k, depth, seen, buf, ballmax, tmp,
                &np, (int32_t)q);
    prop_cnt[q - qlo] = (int32_t)np;
    for (i = 0; i < np; ++i) {
      props[((q - qlo) * ballmax + i) * 2 + 0] = tmp[i].node;
      props[((q - qlo) * ballmax + i) * 2 + 1] = (int32_t)tmp[i].key;
    }
  }
  free(seen); free(buf); free(tmp);
  return 0;
}

/* apply proposals of nslots query slots (slot b proposes id n_t + b), in (qid, key, node) order */
int or_stage_apply(int metric, int k, int64_t n_t, int32_t *ids, uint32_t *keys, int64_t nslots, int64_t ballmax,
                   const int32_t *props, const int32_t *prop_cnt) {
  int64_t b, i, n = 0;
  or_prop *all;
  for (b = 0; b < nslots; ++b) n += prop_cnt[b];
  all = (or_prop *)malloc(sizeof(or_prop) * (size_t)(n + 1));
  n = 0;
  for (b = 0; b < nslots; ++b)
    for (i = 0; i < prop_cnt[b]; ++i) {
      all[n].node = props[(b * ballmax + i) * 2 + 0];
      all[n].key = (uint32_t)props[(b * ballmax + i) * 2 + 1];
      all[n].qid = (int32_t)b;
      ++n;
    }
  g_sort_metric = metric;
  qsort(all, (size_t)n, sizeof(or_prop), prop_cmp);
  for (i = 0; i < n; ++i) {
    or_list L;
    int32_t v = all[i].node;
    L.cap = k; L.cnt = k; L.key = keys + (size_t)v * k; L.id = ids + (size_t)v * k;
    list_insert(metric, &L, all[i].key, (int32_t)(n_t + all[i].qid));
  }
  free(all);
  return 0;
}
