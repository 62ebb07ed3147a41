/*
 * knng.h -- C ABI of the B200-native online approximate k-nn graph library
 * (arXiv 1602.06819, Debatty et al., "Fast online k-nn graph building").
 *
 * Citations: "P:n" = line n of the paper's LaTeX source, with the
 * section / algorithm it falls in.  Readings Qn of points the paper leaves
 * open are listed in DESIGN.md ("Readings").
 *
 * Conventions (all calls):
 *  - extern "C", no C++ or torch types; every call returns int status
 *    (KNNG_OK = 0, < 0 = error) and never throws.  The message of the last
 *    error of the calling thread is graph_last_error().
 *  - Inputs are caller-owned and only read during the call.  Outputs go to
 *    caller-allocated buffers.  The graph handle and all device memory it
 *    uses are owned by the library until graph_free().
 *  - "host" pointers are ordinary CPU memory; "device" pointers are CUDA
 *    global memory on the handle's device.  knng_points.data_on_device says
 *    which one a point buffer is; output buffers are host memory unless the
 *    call has an *_on_device flag.
 *  - One handle must not be used by two threads at once.  Work is issued on
 *    the handle's CUDA stream (knng_runtime.cuda_stream, or a stream the
 *    library creates); every call returns after that stream has finished the
 *    call's work.
 *  - There is no CPU fallback: every step of every call runs in the
 *    library's CUDA kernels (sm_100a).  Without a usable device the calls
 *    fail with KNNG_ERR_CUDA.
 */
#ifndef KNNG_H_
#define KNNG_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (error names follow SPEC.md: S:120) ---- */
#define KNNG_OK                     0
#define KNNG_ERR_INVALID_ARG       -1  /* metric/dim mismatch, k<1, speedup<1, e<1, depth<1, ... */
#define KNNG_ERR_INSUFFICIENT      -2  /* n <= k: a k-nn graph needs more than k items */
#define KNNG_ERR_EMPTY             -3  /* empty graph / empty partition */
#define KNNG_ERR_CAPACITY_INFEAS   -4  /* P * ceil(n*imbalance/P) < n */
#define KNNG_ERR_OOM               -5  /* device allocation failed */
#define KNNG_ERR_CUDA              -6  /* CUDA runtime/launch error, or no device */
#define KNNG_ERR_NCCL              -7  /* NCCL error (multi-GPU) */
#define KNNG_ERR_CAPACITY_EXCEEDED -8  /* store full: n_t + B > capacity */

/* ---- metrics ----
 * KNNG_L2SQ_U8        uint8 vectors; key D = sum_j (a_j - b_j)^2 as exact uint32 (
 *                     Q25: squared L2, monotone in L2).
 * KNNG_L2SQ_F32       fp32 vectors; key D = fp32 squared L2 in the canonical evaluation order
 *                     of reading Q24, returned as the float's bits.
 * KNNG_JACCARD_U32SET sorted, duplicate-free uint32 token sets (set-similarity stand-in for
 *                     P:292); key = (|A n B| << 16) | |A u B|, similarity = inter/union,
 *                     compared exactly by cross-multiplication.
 * KNNG_JARO_WINKLER   strings (section 7.1.2: the SPAM subjects' measure):
 *                     Jaro similarity with the Winkler prefix boost (common prefix l <= 4, scaling
 *                     0.1), matching window max(|a|,|b|)/2 - 1, T = matched characters out of order
 *                     (t = T/2 transpositions).  key = m | T << 7 | l << 14 | |a| << 17 | |b| << 24;
 *                     jw = ((10-l)(2m^2|b| + 2m^2|a| + (2m-T)|a||b|) + 6 l |a||b| m) / (60 |a||b| m),
 *                     compared exactly as fractions.
 * KNNG_COSINE_2GRAM   strings (section 7.1.3: the Wikipedia pages' measure):
 *                     cosine of the count vectors of the 2-grams (contiguous character pairs); a string
 *                     shorter than 2 is the zero vector (cosine 0).  The key of b in a's row (or in
 *                     query a's result) = (dot << 16) | max(|b|^2, 1): a's norm is common to every key
 *                     a row or a search compares, so cos_1 > cos_2 <=> dot_1^2 |b_2|^2 > dot_2^2 |b_1|^2.
 *                     Keys are therefore directed (a row holds its owner's keys); JW keys are symmetric.
 *                     Strings: unpartitioned graphs only (partition_kmedoids returns INVALID_ARG).
 * Edge order (all metrics): more similar key first, equal similarity -> smaller id.
 * Every neighbour row is sorted by edge order. */
typedef enum {
  KNNG_L2SQ_U8 = 0,
  KNNG_L2SQ_F32 = 1,
  KNNG_JACCARD_U32SET = 2,
  KNNG_JARO_WINKLER = 3,
  KNNG_COSINE_2GRAM = 4
} knng_metric;

/* A set of points.  Vectors: data = u8[n*dim] or f32[n*dim], row-major.
 * Sets: data = uint32 tokens (each set sorted ascending, no duplicates), offsets = uint64[n+1]
 * (set i is data[offsets[i] .. offsets[i+1])), dim ignored; sets hold <= 32767 tokens (the key packs
 * the union |A u B| <= 65534 into 16 bits; longer sets fail with INVALID_ARG, host or device input).
 * Strings (KNNG_JARO_WINKLER, KNNG_COSINE_2GRAM): the same CSR form, one uint32 character (code unit)
 * per element in string order, 0..127 characters per string (the keys pack lengths in 7 bits).
 * data_on_device = 1: data (and offsets) are device pointers on the handle's GPU. */
typedef struct {
  int32_t metric;
  int32_t dim;
  int64_t n;
  const void *data;
  const uint64_t *offsets;
  int32_t data_on_device;
} knng_points;

/* Parameters of iGNNS and of the update (Alg. 2).
 *  speedup        budget of one search = max(min(k, |pool|), floor(|pool| / speedup)) similarity
 *                 evaluations (reading Q6); speedup >= 1.
 *  expansion_num/den  expansion e = num/den >= 1 of the restart skip rule; den = 0 means
 *                 e = +inf (never skip).  1.2 = 6/5.  num, den <= 65535.
 *  depth          DEPTH of the update (Alg. 2), 1..10.
 *  seed           key of the counter RNG of the random starts (reading Q4): results are a pure
 *                 function of (inputs, params, seed).
 *  start_override test hook (graph_search only, unpartitioned graphs): host array of node ids used
 *                 as the start sequence of every query instead of RNG draws; NULL in production.
 *  full_scan      graph_search only: 1 = the GNNS baseline's walk (Hajebi et al., section 2.2):
 *                 the similarity of EVERY neighbour of the current node is computed and the walk moves
 *                 to the most similar one (the first in row order among equals) if it improves; with
 *                 expansion_den = 0 (no restart skipping) this is GNNS, the baseline iGNNS is compared
 *                 with.  0 = iGNNS's eager first-improvement walk.
 *  route          partitioned graphs: 1 = search only the partition of the query's nearest medoid
 *                 (ties -> lowest p, as placement) -- the "queries sent to partitions by medoid
 *                 distance" variant of reading Q18; 0 = every partition (Alg. 3).  Single-GPU
 *                 handles only (INVALID_ARG on a multi-GPU handle). */
typedef struct {
  double speedup;
  uint32_t expansion_num, expansion_den;
  int32_t depth;
  uint64_t seed;
  const int32_t *start_override;
  int32_t start_override_len;
  int32_t full_scan;
  int32_t route;
} knng_params;

/* Counters and per-phase device times of the last call (CUDA events on the handle's stream). */
typedef struct {
  int64_t search_evals;       /* committed similarity evaluations of the searches (P:89 units) */
  int64_t search_starts;      /* random starts evaluated */
  int64_t search_skipped;     /* starts discarded by the expansion rule */
  int64_t search_expansions;  /* nodes whose neighbour row was scanned */
  int64_t ball_nodes;         /* update-ball nodes evaluated (Alg. 2) */
  int64_t proposals;          /* (node, new point) replacements proposed by the balls */
  int64_t allpair_pairs;      /* intra-batch pairs evaluated (ordered, i != j) */
  int64_t kernel_launches;    /* kernels launched by the call */
  float ms_search, ms_allpairs, ms_update, ms_merge, ms_total;
} knng_stats;

/* Runtime placement.  device: CUDA ordinal.  cuda_stream: cudaStream_t to issue work on, or NULL.
 * capacity: maximum number of points the graph will hold (0 = 2 * n0).
 * Multi-GPU (one process per GPU): world = number of ranks, rank = this process's rank, and
 * nccl_unique_id = the same 128-byte id on every rank (graph_nccl_unique_id() on rank 0, broadcast
 * by the caller, e.g. over torch.distributed).  The library then owns an NCCL communicator: every
 * rank holds a full replica of the graph, makes the same calls with the same inputs, and
 * graph_insert_batch runs the distributed insert (Alg. 3 + Alg. 5,
 * P:164-178).  world = 1 with a non-NULL id builds a 1-rank communicator (tests). */
typedef struct {
  int32_t device;
  int32_t rank, world;
  const void *nccl_unique_id;
  void *cuda_stream;
  int64_t capacity;
} knng_runtime;

typedef struct knng_graph knng_graph;   /* opaque */

/* graph_init -- build the EXACT k-nn graph of pts (AL1 "brute force"): row v = the first k
 * of all u != v in edge order.  Ids are 0..n-1 in input order.
 * Errors: INVALID_ARG (k < 1 or k > 32, bad metric/dim, null pointers), INSUFFICIENT (n <= k),
 * OOM, CUDA.  *out receives a new handle (NULL on error). */
int graph_init(const knng_points *pts, int32_t k, const knng_runtime *rt, knng_graph **out);

/* graph_insert_batch -- add a batch of B points (Alg. 1 + Alg. 2; distributed form
 * Alg. 5, when partitioned).  On a multi-GPU handle every rank passes the same batch:
 * partitioned graphs search the rank's P/world partitions, unpartitioned ones the rank's share of
 * the queries; NCCL all-gathers on the handle's stream exchange the candidates and proposals (no
 * host synchronisation in between) and every replica ends identical to the 1-GPU result; the
 * counters in *st are summed over the ranks.  Ids are n_t .. n_t+B-1 in batch order
 * (*first_id_out = n_t).  Semantics: every point is searched
 * with iGNNS on the snapshot G_t (RNG stream keyed by its id); its row is the top-k of its
 * search result and the other batch points; the update balls (DEPTH levels over the snapshot)
 * propose the new ids; every touched row becomes top-k(row u proposals); partitioned graphs
 * place each point at its nearest medoid.  B = 1 is exactly the paper's sequential
 * algorithm.  pts->metric/dim must match the graph.  st may be NULL.
 * Errors: INVALID_ARG, CAPACITY_EXCEEDED, EMPTY (a partition is empty), OOM, CUDA. */
int graph_insert_batch(knng_graph *g, const knng_points *pts, const knng_params *p,
                       int64_t *first_id_out, knng_stats *st);

/* graph_insert_sequential -- add n points ONE AFTER ANOTHER: point i is inserted as a batch of one
 * on the graph that point i-1 left (the paper's sequential Alg. 1 + Alg. 2 per point, P:109-151,
 * i.e. the online stream of Section 4), so the result equals n calls of graph_insert_batch with
 * B = 1.  On an unpartitioned single-GPU handle the whole sequence runs in ONE launch (one warp
 * searches and updates point after point; the graph stays on the device, no host round trip between
 * points); otherwise the library loops over the points.  Ids n_t .. n_t+n-1 (*first_id_out = n_t);
 * *st sums the counters of the n inserts.  Arguments, layout and errors as graph_insert_batch. */
int graph_insert_sequential(knng_graph *g, const knng_points *pts, const knng_params *p,
                            int64_t *first_id_out, knng_stats *st);

/* graph_search -- iGNNS k_r-nn search of nq queries on the current graph (read-only; P:73-89,
 * Alg. 3 P:166-178 when partitioned).  Query i uses RNG stream (seed, i, partition).
 * ids_out int32[nq*kr], keys_out uint32[nq*kr], sorted by edge order; -1 / 0 pad when the pool
 * holds fewer than kr nodes.  out_on_device = 1: the output pointers are device memory.
 * Errors: INVALID_ARG (kr < 1 or kr > 32), EMPTY, OOM, CUDA. */
int graph_search(knng_graph *g, const knng_points *queries, int32_t kr, const knng_params *p,
                 int32_t *ids_out, uint32_t *keys_out, int32_t out_on_device, knng_stats *st);

/* partition_kmedoids -- balanced k-medoids of the graph into P partitions (Alg. 4, P:188-243;
 * readings Q21-Q23): capacity ceil(n*imbalance/P); greedy assignment in ascending id to the
 * eligible cluster maximising similarity(m,n) * (1 - |C|/capacity); medoid = member minimising
 * the hop sum in the cluster-induced undirected subgraph (exact when |C| <= 4096, else over
 * {current medoid} + 63 seeded candidates); an iteration is kept only if the total hop sum does
 * not rise.  The graph becomes partitioned: later searches run per partition and inserts place
 * points at the nearest medoid.  part_out: uint8[n] or NULL; medoids_out: int32[P];
 * cost_out: int64[max_iter+1] or NULL (hop-sum cost of each kept iteration, -1 padded);
 * init_medoids: int32[P] test hook or NULL.  All host pointers.  P in 1..255.
 * Returns the number of kept iterations (>= 1) or an error:
 * INVALID_ARG, CAPACITY_INFEAS, OOM, CUDA. */
int partition_kmedoids(knng_graph *g, int32_t P, double imbalance, int32_t max_iter,
                       uint64_t seed, uint8_t *part_out, int32_t *medoids_out, int64_t *cost_out,
                       const int32_t *init_medoids);

/* graph_recompute_medoids -- the last step of Alg. 5 ("compute new medoids"; F5):
 * the update step of Alg. 4 on the CURRENT partition (nodes keep their partitions; the inserted ones
 * were placed at their nearest medoid): every medoid becomes the member minimising the hop sum in its
 * cluster-induced undirected subgraph -- exact when |C| <= 4096, else over {current medoid} + 63
 * draws of stream (seed, 0xFFFFFFFD, epoch * P + p, j) (reading Q22).  Later inserts are placed by
 * the new medoids.  medoids_out: int32[P] or NULL; cost_out: total hop sum or NULL (host pointers).
 * Errors: INVALID_ARG (not partitioned, epoch < 0, a staged batch pending), OOM, CUDA. */
int graph_recompute_medoids(knng_graph *g, uint64_t seed, int64_t epoch, int32_t *medoids_out, int64_t *cost_out);

/* ---- Staged insert: the multi-GPU building blocks (all buffers are DEVICE pointers) ----
 * graph_insert_batch == stage_search(all partitions) + stage_update(world 1, all queries) +
 * stage_commit.  With G ranks each holding a full replica of the graph (same inputs, same calls),
 * the distributed insert of Alg. 5 is, on every rank r:
 *   1. graph_insert_stage_search over the rank's partitions [r*P/G, (r+1)*P/G) and all queries
 *      (q_lo = q_hi = -1): it ingests the batch (rows n_t..n_t+B-1) and writes cand [B][P/G][k]
 *      (ids int32, keys uint32; -1/0 padded);
 *   2. all-gather cand over the ranks -> [G][B][P/G][k] (rank-major) ("the compute nodes send the
 *      k.p candidates", Alg. 3);
 *   3. graph_insert_stage_update(world = G, gathered cand, query shard [q_lo, q_hi)): merges the
 *      candidates (identical on every rank), computes the new rows of the shard's points (top-k of C_i
 *      and the batch) into new_ids/new_keys [q_hi-q_lo][k] (NULL: straight into the graph, 1 GPU), and
 *      runs the update balls of the shard into props int2[q_hi-q_lo][ballmax] (node, key) and
 *      prop_cnt int32[q_hi-q_lo];
 *   4. all-gather new rows, props, prop_cnt over equal-size shards (S = ceil(B/G) slots per rank,
 *      counts 0 in the padding) -> [G*S][k], [G*S][ballmax], [G*S];
 *   5. graph_insert_stage_commit(nq_slots = G*S, gathered buffers; new rows NULL if already in the
 *      graph): writes the new rows, applies every proposal (slot b proposes id n_t + b) and places the
 *      new points; the replicas stay bit-identical and equal the single-GPU call for every G.
 * Unpartitioned graphs shard the queries instead: stage_search(part [0,1), queries [r*S, r*S+S) of the
 * batch) writes cand [S][1][k]; the all-gather gives [G*S][k] whose row b is query b; stage_update is
 * then called with world = 1 and that buffer (the batch of G*S_local points is one snapshot batch).
 * ballmax = graph_ball_bound(g, depth) evaluated BEFORE stage_search (it depends on n_t).
 * Errors: INVALID_ARG (bad ranges, a pending batch, P % G != 0), CAPACITY_EXCEEDED, OOM, CUDA. */
int64_t graph_ball_bound(const knng_graph *g, int32_t depth);
int graph_insert_stage_search(knng_graph *g, const knng_points *pts, const knng_params *p, int32_t part_lo,
                              int32_t part_hi, int64_t q_lo, int64_t q_hi, int32_t *cand_ids, uint32_t *cand_keys,
                              knng_stats *st);
int graph_insert_stage_update(knng_graph *g, const knng_params *p, int32_t world, const int32_t *cand_ids_all,
                              const uint32_t *cand_keys_all, int64_t q_lo, int64_t q_hi, int32_t *props,
                              int32_t *prop_cnt, int32_t *new_ids, uint32_t *new_keys, knng_stats *st);
int graph_insert_stage_commit(knng_graph *g, const knng_params *p, int64_t nq_slots, const int32_t *props_all,
                              const int32_t *prop_cnt_all, const int32_t *new_ids_all, const uint32_t *new_keys_all,
                              knng_stats *st);

/* graph_get_rows -- copy rows [first, first+count) to host: ids int32[count*k],
 * keys uint32[count*k] (either may be NULL).  Errors: INVALID_ARG, CUDA. */
int graph_get_rows(const knng_graph *g, int64_t first, int64_t count, int32_t *ids, uint32_t *keys);

/* graph_get_partition -- part uint8[n] (may be NULL), medoids int32[P] (may be NULL), *P_out.
 * P_out = 0 for an unpartitioned graph.  Errors: INVALID_ARG, CUDA. */
int graph_get_partition(const knng_graph *g, uint8_t *part, int32_t *medoids, int32_t *P_out);

/* graph_size / graph_degree: current n_t and k (-1 on a NULL handle). */
int64_t graph_size(const knng_graph *g);
int32_t graph_degree(const knng_graph *g);

/* graph_free -- release the handle and all its device memory.  NULL is a no-op. */
void graph_free(knng_graph *g);

/* graph_last_error -- message of the last non-zero status of this thread ("" if none). */
const char *graph_last_error(void);

/* graph_nccl_unique_id -- write a new 128-byte NCCL unique id to id_out (host memory), for
 * knng_runtime.nccl_unique_id.  Call on one rank and broadcast it.  Errors: INVALID_ARG, NCCL
 * (libnccl.so.2 is loaded at run time; the single-GPU calls never need it). */
int graph_nccl_unique_id(void *id_out);

/* graph_world -- ranks of the handle's communicator (1 without one; -1 on a NULL handle). */
int32_t graph_world(const knng_graph *g);

#ifdef __cplusplus
}
#endif
#endif /* KNNG_H_ */
