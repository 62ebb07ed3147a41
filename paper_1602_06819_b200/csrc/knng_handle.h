// knng_handle.h -- the graph handle and host helpers shared by the C-ABI implementation files.
#pragma once
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/knng.h"
#include "knng_internal.h"

std::string &knng_err_slot();
int knng_fail(int code, const char *fmt, ...);
#define fail knng_fail

#define CK(x)                                                                                       \
  do {                                                                                              \
    cudaError_t e_ = (x);                                                                           \
    if (e_ != cudaSuccess)                                                                          \
      return fail(e_ == cudaErrorMemoryAllocation ? KNNG_ERR_OOM : KNNG_ERR_CUDA, "%s: %s (%s:%d)", \
                  #x, cudaGetErrorString(e_), __FILE__, __LINE__);                                  \
  } while (0)

struct DBuf {
  void *p = nullptr;
  size_t bytes = 0;
  cudaError_t ensure(size_t need) {
    if (need <= bytes) return cudaSuccess;
    need += need / 4;             // grow geometrically: batches grow the pool a little each time
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
  template <class T>
  T *as() const { return (T *)p; }
};

struct knng_graph {
  int metric = 0, dim = 0, k = 0;
  int64_t n = 0, cap = 0;
  int64_t pend_B = 0;                           // batch ingested by stage_search, not yet committed
  int pend_parts = 0;                           // partitions stage_search searched for the pending batch
  int pend_route = 0;                           // ... or 1: the batch was searched on its routed partitions
  const knng::BallArgs *fuse_b1 = nullptr;   // set by insert_seq around its search launch (B = 1 fused)
  int64_t fuse_nseq = 0;
  DBuf w_ktm;                                // [nseq][ld] key matrix of a sequence on a small graph (KT)                     // ... and the number of sequential inserts of that launch
  DBuf w_route;                                 // routing targets of a search
  knng::VecGeom geom{};
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  uint8_t *vec = nullptr;                       // vectors (u8 / f32 rows)
  uint64_t *off = nullptr;                      // sets: [cap+1] offsets into tok
  uint32_t *tok = nullptr;                      // sets: tokens (strings: characters)
  uint32_t *sn2 = nullptr;                      // 2-gram cosine strings: |x|^2 of every stored string [cap]
  int64_t tok_cap = 0, tok_n = 0;               // token capacity / tokens in use (host mirror)
  // partitioned graphs: the partition-local store K1 reads (index = (p, local index), member_cap = cap rows per
  // partition): prow [P][cap][k] local index of each row entry in the row owner's partition (-1 across),
  // pvec [P][cap][stride] the vectors (vector metrics), pset [P][cap] the [begin, end) token ranges (sets)
  int32_t *prow = nullptr;
  uint8_t *pvec = nullptr;
  ulonglong2 *pset = nullptr;
  int local_P = 0;                              // partitions the local store is allocated for
  uint32_t tok_max = 0;
  int64_t tprof_n = 0;                          // KNNG_PROFILE: tasks of the last search                         // largest stored token (valid when tok_n > 0)
  int32_t *ids = nullptr;
  uint32_t *keys = nullptr;
  int32_t *ncnt = nullptr, *nfill = nullptr, *noff = nullptr, *scan_tmp = nullptr;
  // partitions
  int P = 0;
  uint8_t *part_of = nullptr;
  int32_t *local_idx = nullptr;
  int32_t *members = nullptr;
  int64_t *member_cnt = nullptr;
  int32_t *medoids = nullptr;
  std::vector<int32_t> h_medoids;
  // workspaces
  DBuf w_bits, w_cand_i, w_cand_k, w_C_i, w_C_k, w_hash, w_list, w_props, w_prop_cnt, w_sorted, w_stats,
      w_target, w_query, w_starts;
  DBuf w_qoff, w_qtok, w_qn2;
  knng::DenseScratch w_dense;                    // A0 / A5 partial rows and norms
  // multi-GPU (knng_runtime.world > 1, or a 1-rank communicator for tests): the library's NCCL
  // communicator and the buffers of the two all-gathers of graph_insert_batch
  void *comm = nullptr;
  int rank = 0, world = 1;
  DBuf w_dci, w_dck, w_gci, w_gck, w_dprops, w_dcnt, w_dnid, w_dnkey, w_gprops, w_gcnt, w_gnid, w_gnkey, w_dstats;
  // partition sizes: the host keeps an upper bound (exact after an asynchronous read-back) so that
  // sizing a search never waits on the device
  int64_t *h_cnt = nullptr;                     // pinned [P]
  cudaEvent_t ev_cnt = nullptr;
  bool cnt_pending = false;
  int64_t cnt_n = 0;                            // graph size the pending read-back describes
  int64_t pool_bound = 0;
  DBuf w_tprof;                                 // KNNG_PROFILE: per-task consumer cycles of the last search
  cudaEvent_t ev[6] = {};
};

inline knng::StoreView graph_store_view(const knng_graph *g) {
  knng::StoreView v;
  v.vec = g->vec;
  v.stride = g->geom.stride;
  v.nchunks = g->geom.nchunks;
  v.off = g->off;
  v.tok = g->tok;
  v.n2 = g->sn2;
  const int64_t vw = g->tok_n > 0 ? ((int64_t)g->tok_max + 32) / 32 : 0;
  v.vwords = (g->metric == KNNG_JACCARD_U32SET && vw > 0 && vw <= knng::VOCAB_SMEM_WORDS) ? (int)vw : 0;
  return v;
}

inline knng::LocalStore graph_local_store(const knng_graph *g) {
  knng::LocalStore ls;
  ls.prow = g->prow;
  ls.pvec = g->pvec;
  ls.pset = g->pset;
  ls.cap = g->cap;
  return ls;
}
