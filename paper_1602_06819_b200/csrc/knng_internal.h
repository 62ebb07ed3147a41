// knng_internal.h -- kernel argument blocks and launchers shared by the .cu files of the
// product library (not part of the C ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "knng_common.cuh"

namespace knng {

// Device scratch owned by a graph handle (never process-global: a handle is bound to one device and
// one stream, and two handles may be used from two threads).  Grown on demand.
struct Scratch {
  void *p = nullptr;
  size_t bytes = 0;
  cudaError_t ensure(size_t need) {
    if (need <= bytes) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    cudaError_t e = cudaMalloc(&p, need);
    if (e == cudaSuccess) bytes = need;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
};
// scratch of the dense exact steps (A0 build, A5 all-pairs): column-split partial rows and norms
struct DenseScratch {
  Scratch part, norm;
};

// Vector store geometry: rows of `stride` bytes (= nchunks * 16, zero padded).
struct VecGeom {
  int metric;
  int nchunks;
  size_t stride;
  int L, CPL;   // lanes per vector and chunks per lane of the warp evaluator
};

struct BallArgs {
  StoreView st;
  int32_t *ids;                // rows (snapshot until the merge)
  uint32_t *keys;
  int k;
  int64_t n_t;
  int64_t B;
  int depth;
  const int32_t *C;            // search results [B][k] (all B queries of the batch)
  int64_t q0;                  // this launch handles queries q0 .. q0+nqb-1 (props index is local)
  int64_t nqb;
  int32_t *hash;               // per warp slot, hcap entries
  int hcap;
  int32_t *list;               // per warp slot, ballmax entries
  int ballmax;
  int smem_ball;               // 1: hash + list in shared memory (small balls), else the global slots
  int2 *props;                 // [B][ballmax] (node, key)
  int32_t *prop_cnt;           // [B]
  unsigned long long *stats;   // [4] ball nodes [5] proposals
};

struct SearchArgs {
  int metric;                  // M_U8 / M_F32 / M_JAC (the kernel's template metric)
  StoreView st;                // the graph's points
  StoreView qs;                // the queries (== st for inserts)
  int64_t qrow0;               // query b is row qrow0 + b of qs
  const int32_t *rows;         // snapshot rows [n_t][k]
  int k;
  int64_t n_t;
  int64_t nq;
  int64_t pid_base;            // RNG point id of query b = pid_base + b
  // partitions (P == 0: unpartitioned, pool = 0..n_t-1); this launch searches partitions
  // [part_lo, part_lo + part_cnt) (part_lo = 0, part_cnt = 1 when unpartitioned)
  int P;
  int part_lo, part_cnt;
  const int32_t *members;      // [P][member_cap]
  int64_t member_cap;
  const int64_t *member_cnt;   // [P] (device)
  const uint8_t *part_of;      // [cap]
  const int32_t *local_idx;    // [cap]
  // the partition-local store (P > 0): K1 draws, walks and ranks partition-local indices and converts its
  // top-k to ids through members at the end (members[p] is ascending, so ties by local index are ties by id)
  const int32_t *prow;         // [P][member_cap][k]: local index of each entry in the row owner's partition, -1 across
  const uint8_t *pvec;         // [P][member_cap][stride] (vector metrics)
  const ulonglong2 *pset;      // [P][member_cap] token ranges (sets)
  // parameters
  double speedup;
  uint64_t e_num, e_den, seed;
  int kr;
  const int32_t *starts;       // injected start sequence (device, unpartitioned graphs) or null
  int nstarts;
  // per-task visited state: the E (evaluated) / X (expanded) bit planes of every warp slot
  uint32_t *gbits;             // [gslots][de_words]
  int64_t gslots;              // warp slots of gbits (resident warps of the launch)
  int64_t de_words;            // ceil(max pool / 16), rounded up to a multiple of 4
  // outputs
  int32_t *out_ids;            // [nq][part_cnt][kr]
  uint32_t *out_keys;
  unsigned long long *stats;   // [0] evals [1] starts [2] skipped [3] expansions
  unsigned long long *prof;    // cycle counters (profile builds, KNNG_PROFILE=1), else null
  unsigned long long *task_ctr;  // dynamic task scheduler counter (zeroed by the launcher)
  int pitch;                   // bytes per staged row (vectors: stride + 16) / set slot
  int wbytes;                  // shared memory of one warp (set by the launcher)
  int swz;                     // 1: staged rows are swizzled 16-byte chunks (lane-form widths, nchunks % 8 == 0)
  int lane_eval;               // 1: one lane per staged row where the width allows
  int win_prefetch;            // 1: prefetch the rows of a window's possible starts
  int e_smem;                  // 1: the E bitmap of a task lives in the warp's shared memory (e_bytes, 1 bit per
                               // pool node; X stays in the global words) -- the latency-bound plans
  int e_bytes;                 // bytes of one bitmap (16-byte multiple)
  int x_smem;                  // (e_smem) 1: the X bitmap too (after E); KT launches always
  int ns2;                     // 1 (with e_smem): two chunk stages, chunk c + 1's rows in flight while c is processed
  int row_pf;                  // 1: a walk step copies the rows of all of cur's neighbours with their vectors
  int perm_e;                  // 1 (global E words): draws set no E bits (the permutation draws never repeat and a
                               // walk neighbour's "drawn before" is pi^-1(v) <= the last processed draw); the
                               // words hold the walk evaluations, filtered per warp in shared memory
                               // (0: the chosen neighbour's row is loaded once the move is known)
  int full_scan;               // 1: the GNNS baseline walk (all k neighbours, move to the best)
  int bulk;                    // 1 (lane-form widths, one chunk stage): rows gathered by TMA bulk copies
  const int32_t *route;        // routed search (reading Q18's variant): partition of query b, else null
  // B = 1 fused launch (one task): after the search, the same warp runs the update of the insert
  // (update_one_warp with ub, C = out_ids / out_keys) and writes stats[0..5] itself
  int fuse;
  int nseq;                    // (fuse) sequential inserts: rows n_t .. n_t + nseq - 1 (ingested), one after another
  BallArgs ub;
  int kt;                      // (fuse) 1: the keys against all n_t pool nodes precomputed (ktm) and staged in smem
  int srows;                   // (kt) 1: the rows (ids) of nodes 0 .. n_t + nseq - 1 kept in shared memory too
  const uint32_t *ktm;         // (kt) [nseq][ktm_ld] key matrix of the sequence (launch_keymat)
  int64_t ktm_ld;
};
size_t search_smem_bytes(const SearchArgs &a, bool sets);
// warps of one K1 launch that can be resident at once (sizes the per-warp E / X planes)
cudaError_t search_resident_warps(const VecGeom &g, const SearchArgs &a, int64_t *warps);
// keys of points qrow0 + i (i < B) against nodes 0 .. n0 + i - 1 into out [B][ld] (the KT launches)
cudaError_t launch_keymat(int metric, const StoreView &st, int64_t qrow0, int64_t n0, int64_t B, int64_t ld,
                          uint32_t *out, cudaStream_t s);
// K1 computes keys one lane per staged row for this width (the compile-time lane-form kernels)
bool search_lane_form(const VecGeom &g, int lane_eval);


// Launchers (return cudaError_t of the launch)
cudaError_t launch_search(const VecGeom &g, const SearchArgs &a, cudaStream_t s, int *n_launch);
// gathered candidates: rank-major [world][nq][P/world][kr]
cudaError_t launch_merge_parts(int metric, const int32_t *cand_ids, const uint32_t *cand_keys, int64_t nq,
                               int P, int world, int kr, int32_t *out_ids, uint32_t *out_keys, cudaStream_t s);
cudaError_t launch_allpairs(const VecGeom &g, const StoreView &st, int64_t n_t, int64_t B, int64_t q_lo, int64_t nq,
                            int k, const int32_t *Ci, const uint32_t *Ck, int32_t *oi, uint32_t *ok, DenseScratch *ws,
                            cudaStream_t s);
cudaError_t launch_ball(const VecGeom &g, const BallArgs &a, int64_t nslots, cudaStream_t s);
// B = 1: new row, ball, proposals and their application for one insert (one warp, one launch)
cudaError_t launch_update_one(const VecGeom &g, const BallArgs &a, const uint32_t *Ckeys, cudaStream_t s);
cudaError_t launch_merge_props(int metric, int32_t *ids, uint32_t *keys, int k, int64_t n_t, int64_t B,
                               const int2 *props, const int32_t *prop_cnt, int ballmax, int32_t *ncnt,
                               int32_t *nfill, int32_t *noff, int32_t *scan_tmp, int2 *sorted,
                               cudaStream_t s, int *n_launch, int32_t *prow = nullptr, int64_t member_cap = 0,
                               const uint8_t *part_of = nullptr, const int32_t *local_idx = nullptr);
// the partition-local store of nodes [first, first + count) (rows, and vectors or token ranges)
struct LocalStore {
  int32_t *prow;
  uint8_t *pvec;
  ulonglong2 *pset;
  int64_t cap;
};
cudaError_t launch_local_store(const StoreView &st, const int32_t *ids, int k, int64_t first, int64_t count,
                               const uint8_t *part_of, const int32_t *local_idx, const LocalStore &ls, cudaStream_t s);
cudaError_t exclusive_scan_i32(const int32_t *in, int32_t *out, int32_t *tmp, int64_t n, cudaStream_t s);
cudaError_t launch_tc_topk_u8(const VecGeom &g, const uint8_t *vec, int64_t row0, int64_t nrows, int64_t col0,
                              int64_t ncols, int k, const int32_t *sid, const uint32_t *skey, int64_t ny, int32_t *pi,
                              uint32_t *pk, Scratch *norm, cudaStream_t s);
cudaError_t launch_tc_topk_f32(const VecGeom &g, const uint8_t *vec, int64_t row0, int64_t nrows, int64_t col0,
                               int64_t ncols, int k, const int32_t *sid, const uint32_t *skey, int64_t ny, int32_t *pi,
                               uint32_t *pk, Scratch *norm, cudaStream_t s);
cudaError_t launch_exact_build(const VecGeom &g, const StoreView &st, int64_t n, int k, int32_t *ids,
                               uint32_t *keys, DenseScratch *ws, cudaStream_t s);
// nearest medoid of queries [qrow0, qrow0 + nq) of qs (ties -> lowest p): the routing target
cudaError_t launch_route_target(const VecGeom &g, const StoreView &qs, int64_t qrow0, int64_t nq, const StoreView &st,
                                int P, const int32_t *medoids, int32_t *target, cudaStream_t s);
cudaError_t launch_place(const VecGeom &g, const StoreView &st, int64_t n_t, int64_t B, int P,
                         const int32_t *medoids, int32_t *members, int64_t member_cap, int64_t *member_cnt,
                         uint8_t *part_of, int32_t *local_idx, int32_t *target_tmp, cudaStream_t s);

}  // namespace knng
