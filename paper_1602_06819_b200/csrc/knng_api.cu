// knng_api.cu -- the C ABI of include/knng.h: graph handle, HBM layout, and the batch
// pipeline of graph_insert_batch (search -> partition merge -> all-pairs -> update balls ->
// ordered merge -> placement), all stream-ordered on the handle's CUDA stream.
//
// HBM layout of a handle (capacity N_cap points, degree k):
//   vec      uint8 [N_cap][stride]   vectors, rows zero-padded to 16-byte chunks
//   ids      int32 [N_cap][k]        neighbour rows, sorted by edge order
//   keys     uint32[N_cap][k]        their keys
//   part_of  uint8 [N_cap], local_idx int32[N_cap], members int32[P][N_cap]   (partitioned)
//   ncnt/nfill/noff int32[N_cap]     proposal bucketing of the merge (kept zeroed)
// plus per-batch workspaces grown on demand.
#include <cuda_runtime.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <vector>

#include "../../include/knng.h"
#include "knng_common.cuh"
#include "knng_internal.h"

#include "knng_handle.h"
#include "knng_nccl.h"

using namespace knng;

std::string &knng_err_slot() {
  static thread_local std::string e;
  return e;
}

int knng_fail(int code, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  knng_err_slot() = buf;
  return code;
}

static int elem_bytes(int metric) { return metric == KNNG_L2SQ_U8 ? 1 : 4; }
// points held as uint32 sequences in CSR form: token sets, strings of characters
static bool csr_points(int metric) {
  return metric == KNNG_JACCARD_U32SET || metric == KNNG_JARO_WINKLER || metric == KNNG_COSINE_2GRAM;
}
static bool str_points(int metric) { return metric == KNNG_JARO_WINKLER || metric == KNNG_COSINE_2GRAM; }

static int geom_for(int metric, int dim, VecGeom *g) {
  if (csr_points(metric)) {   // sets / strings: one lane per candidate (L = 8: the set evaluator's instantiation)
    g->metric = metric;
    g->nchunks = 0;
    g->stride = 0;
    g->L = 8;
    g->CPL = 1;
    return 0;
  }
  const size_t row = (size_t)dim * elem_bytes(metric);
  const int C = (int)((row + 15) / 16);
  g->metric = metric;
  g->nchunks = C;
  g->stride = (size_t)C * 16;
  if (metric == KNNG_L2SQ_F32 && C <= 32) {   // <= 4 chunks per lane, in-lane canonical partials
    int L = 1;
    while (L * 4 < C) L <<= 1;
    g->L = L;
    g->CPL = (C + L - 1) / L;
  } else if (C <= 32) {
    int L = 1;
    while (L < C) L <<= 1;
    g->L = L;
    g->CPL = 1;
  } else if (C <= 64) {
    g->L = 32; g->CPL = 2;
  } else if (C <= 128) {
    g->L = 32; g->CPL = 4;
  } else {
    return -1;
  }
  return 0;
}

static int check_points(const knng_points *p, const char *what) {
  if (!p) return fail(KNNG_ERR_INVALID_ARG, "%s: null points", what);
  if (p->metric != KNNG_L2SQ_U8 && p->metric != KNNG_L2SQ_F32 && !csr_points(p->metric))
    return fail(KNNG_ERR_INVALID_ARG, "%s: bad metric %d", what, p->metric);
  if (!csr_points(p->metric) && p->dim < 1) return fail(KNNG_ERR_INVALID_ARG, "%s: dim < 1", what);
  if (p->n < 0) return fail(KNNG_ERR_INVALID_ARG, "%s: n < 0", what);
  if (p->n > 0 && !p->data) return fail(KNNG_ERR_INVALID_ARG, "%s: null data", what);
  if (csr_points(p->metric) && !p->offsets) return fail(KNNG_ERR_INVALID_ARG, "%s: null offsets", what);
  return 0;
}

// copy n points (row-major, dim*elem bytes each) into padded rows starting at dst
static int copy_rows(knng_graph *g, uint8_t *dst, const knng_points *p) {
  if (p->n == 0) return 0;
  const size_t row = (size_t)p->dim * elem_bytes(p->metric);
  CK(cudaMemcpy2DAsync(dst, g->geom.stride, p->data, row, row, (size_t)p->n,
                       p->data_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, g->stream));
  return 0;
}

__global__ void k_token_max(const uint32_t *tok, int64_t n, unsigned *out) {
  unsigned m = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    m = max(m, tok[i]);
  m = __reduce_max_sync(0xFFFFFFFFu, m);
  if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}

// longest set of a device CSR batch (sets must hold <= KNNG_SET_MAX tokens: the key packs the union
// |A u B| <= 2 * KNNG_SET_MAX into 16 bits)
__global__ void k_max_set_len(const uint64_t *off, int64_t n, unsigned long long *out) {
  unsigned long long m = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    m = max(m, (unsigned long long)(off[i + 1] - off[i]));
  for (int o = 16; o >= 1; o >>= 1) m = max(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));
  if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}
static constexpr uint64_t KNNG_SET_MAX = 32767;
static uint64_t csr_max_len(int metric) { return str_points(metric) ? (uint64_t)STR_MAX : KNNG_SET_MAX; }

// 2-gram cosine strings: |x|^2 = sum_g c_x(g)^2 = the number of position pairs with equal 2-grams, for
// strings [first, first + count) of a store (thread per string; 1 for strings shorter than 2, whose
// count vector is zero -- their cosine with anything is 0 whatever the norm)
__global__ void k_str_norms(const uint64_t *off, const uint32_t *tok, int64_t first, int64_t count, uint32_t *n2) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const uint32_t *x = tok + off[first + i];
  const int L = (int)(off[first + i + 1] - off[first + i]);
  uint32_t c = 0;
  for (int a = 0; a + 1 < L; ++a)
    for (int b = 0; b + 1 < L; ++b) c += (x[a] == x[b]) & (x[a + 1] == x[b + 1]);
  n2[first + i] = c > 0 ? c : 1u;
}

__global__ void k_rebase_offsets(const uint64_t *in, int64_t n, uint64_t base, uint64_t *out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i <= n) out[i] = base + (in[i] - in[0]);
}

// append n sets (CSR, host or device) to a token/offset store: off[row0 .. row0+n] and
// tok[tok_n ..]; grows the token buffer geometrically.  Returns the tokens appended.
static int append_sets(knng_graph *g, const knng_points *p, uint64_t **off_dst_base, uint32_t **tok_buf,
                       int64_t *tok_cap, int64_t row0, int64_t tok0, int64_t *ntok_out, uint32_t *tok_max = nullptr) {
  uint64_t first = 0, last = 0;
  if (p->data_on_device) {
    unsigned long long *dm = nullptr, mlen = 0;
    CK(cudaMallocAsync((void **)&dm, 8, g->stream));
    CK(cudaMemsetAsync(dm, 0, 8, g->stream));
    if (p->n > 0) k_max_set_len<<<(unsigned)std::min<int64_t>((p->n + 255) / 256, 1024), 256, 0, g->stream>>>(p->offsets, p->n, dm);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(&mlen, dm, 8, cudaMemcpyDeviceToHost, g->stream));
    CK(cudaMemcpyAsync(&first, p->offsets, 8, cudaMemcpyDeviceToHost, g->stream));
    CK(cudaMemcpyAsync(&last, p->offsets + p->n, 8, cudaMemcpyDeviceToHost, g->stream));
    CK(cudaFreeAsync(dm, g->stream));
    CK(cudaStreamSynchronize(g->stream));
    if (mlen > csr_max_len(p->metric))
      return fail(KNNG_ERR_INVALID_ARG, "set / string longer than %llu", (unsigned long long)csr_max_len(p->metric));
  } else {
    first = p->offsets[0];
    last = p->offsets[p->n];
    for (int64_t i = 0; i < p->n; ++i)
      if (p->offsets[i + 1] - p->offsets[i] > csr_max_len(p->metric))
        return fail(KNNG_ERR_INVALID_ARG, "set / string longer than %llu", (unsigned long long)csr_max_len(p->metric));
  }
  const int64_t nt = (int64_t)(last - first);
  if (tok0 + nt > *tok_cap) {
    const int64_t ncap = std::max<int64_t>(tok0 + nt, *tok_cap + *tok_cap / 2) + 1024;
    uint32_t *nb = nullptr;
    CK(cudaMalloc((void **)&nb, (size_t)ncap * 4));
    // zeroed slack: the set evaluator reads whole 16-byte chunks around a set's tokens
    CK(cudaMemsetAsync(nb + tok0, 0, (size_t)(ncap - tok0) * 4, g->stream));
    if (*tok_buf && tok0 > 0) CK(cudaMemcpyAsync(nb, *tok_buf, (size_t)tok0 * 4, cudaMemcpyDeviceToDevice, g->stream));
    CK(cudaStreamSynchronize(g->stream));
    if (*tok_buf) cudaFree(*tok_buf);
    *tok_buf = nb;
    *tok_cap = ncap;
  }
  if (nt > 0)
    CK(cudaMemcpyAsync(*tok_buf + tok0, (const uint32_t *)p->data + first, (size_t)nt * 4,
                       p->data_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, g->stream));
  // offsets rebased to tok0
  uint64_t *dst = *off_dst_base + row0;
  if (p->data_on_device) {
    k_rebase_offsets<<<(unsigned)((p->n + 256) / 256), 256, 0, g->stream>>>(p->offsets, p->n, (uint64_t)tok0, dst);
    CK(cudaGetLastError());
  } else {
    std::vector<uint64_t> h((size_t)p->n + 1);
    for (int64_t i = 0; i <= p->n; ++i) h[i] = (uint64_t)tok0 + (p->offsets[i] - first);
    CK(cudaMemcpyAsync(dst, h.data(), h.size() * 8, cudaMemcpyHostToDevice, g->stream));
    CK(cudaStreamSynchronize(g->stream));   // h is a local buffer
  }
  if (tok_max && nt > 0) {   // largest token: sizes the search's vocabulary bitmap
    unsigned m = 0;
    if (p->data_on_device) {
      unsigned *dm = nullptr;
      CK(cudaMalloc((void **)&dm, 4));
      CK(cudaMemsetAsync(dm, 0, 4, g->stream));
      k_token_max<<<256, 256, 0, g->stream>>>(*tok_buf + tok0, nt, dm);
      CK(cudaGetLastError());
      CK(cudaMemcpyAsync(&m, dm, 4, cudaMemcpyDeviceToHost, g->stream));
      CK(cudaStreamSynchronize(g->stream));
      cudaFree(dm);
    } else {
      const uint32_t *t = (const uint32_t *)p->data + first;
      for (int64_t i = 0; i < nt; ++i) m = std::max(m, t[i]);
    }
    *tok_max = std::max(*tok_max, (uint32_t)m);
  }
  *ntok_out = nt;
  return 0;
}

// store the batch's points at rows [row0, row0+n) of the graph's store
static int store_points(knng_graph *g, const knng_points *p, int64_t row0) {
  if (csr_points(g->metric)) {
    int64_t nt = 0;
    if (int r = append_sets(g, p, &g->off, &g->tok, &g->tok_cap, row0, g->tok_n, &nt, &g->tok_max)) return r;
    g->tok_n += nt;
    if (g->metric == KNNG_COSINE_2GRAM && p->n > 0) {
      k_str_norms<<<(unsigned)((p->n + 127) / 128), 128, 0, g->stream>>>(g->off, g->tok, row0, p->n, g->sn2);
      CK(cudaGetLastError());
    }
    return 0;
  }
  return copy_rows(g, g->vec + (size_t)row0 * g->geom.stride, p);
}

static void free_graph(knng_graph *g) {
  if (!g) return;
  cudaSetDevice(g->device);
  if (g->stream) cudaStreamSynchronize(g->stream);
  void *bufs[] = {g->vec, g->ids, g->keys, g->ncnt, g->nfill, g->noff, g->scan_tmp, g->part_of, g->local_idx, g->prow,
                  g->pvec, g->pset, g->members, g->member_cnt, g->medoids, g->off, g->tok, g->sn2};
  for (void *b : bufs)
    if (b) cudaFree(b);
  DBuf *ws[] = {&g->w_bits, &g->w_cand_i, &g->w_cand_k, &g->w_C_i, &g->w_C_k, &g->w_hash, &g->w_list, &g->w_props,
                &g->w_prop_cnt, &g->w_sorted, &g->w_stats, &g->w_target, &g->w_query, &g->w_starts, &g->w_route,
                &g->w_qoff, &g->w_qtok, &g->w_tprof, &g->w_ktm, &g->w_qn2};
  for (DBuf *b : ws) b->release();
  g->w_dense.part.release();
  g->w_dense.norm.release();
  for (auto &e : g->ev)
    if (e) cudaEventDestroy(e);
  if (g->ev_cnt) cudaEventDestroy(g->ev_cnt);
  if (g->h_cnt) cudaFreeHost(g->h_cnt);
  DBuf *dws[] = {&g->w_dci, &g->w_dck, &g->w_gci, &g->w_gck, &g->w_dprops, &g->w_dcnt, &g->w_dnid, &g->w_dnkey,
                 &g->w_gprops, &g->w_gcnt, &g->w_gnid, &g->w_gnkey, &g->w_dstats};
  for (DBuf *b : dws) b->release();
  if (g->comm) knng::nccl_comm_destroy(g->comm);
  if (g->own_stream && g->stream) cudaStreamDestroy(g->stream);
  delete g;
}

extern "C" {

const char *graph_last_error(void) { return knng_err_slot().c_str(); }

int graph_nccl_unique_id(void *id_out) {
  knng_err_slot().clear();
  if (!id_out) return fail(KNNG_ERR_INVALID_ARG, "graph_nccl_unique_id: null output");
  if (const char *m = knng::nccl_get_unique_id(id_out)) return fail(KNNG_ERR_NCCL, "%s", m);
  return KNNG_OK;
}

int32_t graph_world(const knng_graph *g) { return g ? g->world : -1; }

int64_t graph_size(const knng_graph *g) { return g ? g->n : -1; }
int32_t graph_degree(const knng_graph *g) { return g ? g->k : -1; }
void graph_free(knng_graph *g) { free_graph(g); }

int graph_init(const knng_points *pts, int32_t k, const knng_runtime *rt, knng_graph **out) {
  knng_err_slot().clear();
  if (!out) return fail(KNNG_ERR_INVALID_ARG, "graph_init: null out");
  *out = nullptr;
  if (int r = check_points(pts, "graph_init")) return r;
  if (k < 1 || k > 32) return fail(KNNG_ERR_INVALID_ARG, "graph_init: k=%d outside 1..32", k);
  if (pts->n <= k) return fail(KNNG_ERR_INSUFFICIENT, "graph_init: n=%lld <= k=%d", (long long)pts->n, k);
  if (pts->n >= (int64_t)1 << 31) return fail(KNNG_ERR_INVALID_ARG, "graph_init: n too large");
  knng_graph *g = new knng_graph();
  g->metric = pts->metric;
  g->dim = pts->dim;
  g->k = k;
  g->device = rt ? rt->device : 0;
  if (geom_for(g->metric, g->dim, &g->geom)) {
    delete g;
    return fail(KNNG_ERR_INVALID_ARG, "graph_init: vectors of %d dims are too wide", pts->dim);
  }
  int r = 0;
  auto bail = [&](int code) { free_graph(g); return code; };
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    delete g;
    return fail(KNNG_ERR_CUDA, "graph_init: no CUDA device");
  }
  if (cudaSetDevice(g->device) != cudaSuccess) {
    delete g;
    return fail(KNNG_ERR_CUDA, "graph_init: cudaSetDevice(%d) failed", rt ? rt->device : 0);
  }
  // multi-GPU: the library's own NCCL communicator (every rank calls graph_init with the same inputs and
  // the same 128-byte id from graph_nccl_unique_id on rank 0); a 1-rank communicator is allowed (tests)
  if (rt && (rt->world > 1 || rt->nccl_unique_id)) {
    if (rt->world < 1 || rt->rank < 0 || rt->rank >= rt->world || !rt->nccl_unique_id) {
      delete g;
      return fail(KNNG_ERR_INVALID_ARG, "graph_init: bad rank %d / world %d / id", rt->rank, rt->world);
    }
    g->rank = rt->rank;
    g->world = rt->world;
    if (const char *m = knng::nccl_comm_init(&g->comm, rt->world, rt->nccl_unique_id, rt->rank)) {
      delete g;
      return fail(KNNG_ERR_NCCL, "graph_init: %s", m);
    }
  }
  if (rt && rt->cuda_stream) {
    g->stream = (cudaStream_t)rt->cuda_stream;
  } else {
    if (cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking) != cudaSuccess) {
      free_graph(g);
      return fail(KNNG_ERR_CUDA, "graph_init: stream create failed");
    }
    g->own_stream = true;
  }
  g->n = pts->n;
  g->cap = (rt && rt->capacity > 0) ? rt->capacity : 2 * pts->n;
  if (g->cap < g->n) g->cap = g->n;
  const size_t cap = (size_t)g->cap;
#define A(ptr, bytes)                                             \
  do {                                                            \
    cudaError_t e_ = cudaMalloc((void **)&(ptr), (bytes));        \
    if (e_ != cudaSuccess) {                                      \
      fail(KNNG_ERR_OOM, "graph_init: cudaMalloc %zu B failed", (size_t)(bytes)); \
      return bail(KNNG_ERR_OOM);                                  \
    }                                                             \
  } while (0)
  if (csr_points(g->metric)) {
    A(g->off, (cap + 1) * 8);
    if (g->metric == KNNG_COSINE_2GRAM) A(g->sn2, cap * 4);
  } else {
    A(g->vec, cap * g->geom.stride);
  }
  A(g->ids, cap * k * 4);
  A(g->keys, cap * k * 4);
  A(g->ncnt, cap * 4);
  A(g->nfill, cap * 4);
  A(g->noff, cap * 4);
  A(g->scan_tmp, ((cap + 1023) / 1024 + 1) * 4);
#undef A
  for (auto &e : g->ev)
    if (cudaEventCreate(&e) != cudaSuccess) return bail(fail(KNNG_ERR_CUDA, "event create failed"));
  if ((g->vec && cudaMemsetAsync(g->vec, 0, cap * g->geom.stride, g->stream) != cudaSuccess) ||
      cudaMemsetAsync(g->ncnt, 0, cap * 4, g->stream) != cudaSuccess ||
      cudaMemsetAsync(g->nfill, 0, cap * 4, g->stream) != cudaSuccess)
    return bail(fail(KNNG_ERR_CUDA, "graph_init: memset failed"));
  if ((r = store_points(g, pts, 0))) return bail(r);
  cudaError_t e = launch_exact_build(g->geom, graph_store_view(g), g->n, k, g->ids, g->keys, &g->w_dense, g->stream);
  if (e != cudaSuccess) return bail(fail(KNNG_ERR_CUDA, "exact build launch: %s", cudaGetErrorString(e)));
  e = cudaStreamSynchronize(g->stream);
  if (e != cudaSuccess) return bail(fail(KNNG_ERR_CUDA, "exact build: %s", cudaGetErrorString(e)));
  *out = g;
  return KNNG_OK;
}

static int check_params(const knng_params *p) {
  if (!p) return fail(KNNG_ERR_INVALID_ARG, "null params");
  if (!(p->speedup >= 1.0)) return fail(KNNG_ERR_INVALID_ARG, "speedup < 1");
  if (p->expansion_den != 0 && p->expansion_num < p->expansion_den) return fail(KNNG_ERR_INVALID_ARG, "expansion < 1");
  if (p->expansion_num > 65535 || p->expansion_den > 65535)
    return fail(KNNG_ERR_INVALID_ARG, "expansion num/den must be <= 65535");
  return 0;
}

// K1 launch shape: one warp per (query, partition) task, WPC warps per CTA, as many CTAs as fit;
// each resident warp owns a slot of E / X bit planes sized for the largest pool.  Knobs
// KNNG_LANE_EVAL / KNNG_WIN_PREFETCH override it (measurement and tests only: results do not depend
// on them).
static int plan_k1(knng_graph *g, SearchArgs &a, int64_t tasks, int64_t mmax) {
  a.de_words = (((mmax + 15) / 16) + 3) & ~3ll;
  a.lane_eval = 1;
  if (const char *e = getenv("KNNG_LANE_EVAL")) a.lane_eval = atoi(e);
  // staged rows: the lane-form widths with nchunks % 8 == 0 are stored swizzled (no bank-conflict pad)
  const bool sets = csr_points(g->metric);
  const bool lform = search_lane_form(g->geom, a.lane_eval);
  a.swz = lform && g->geom.nchunks % 8 == 0;
  // sets: a lane's slot holds SETCH aligned 16-byte token chunks (longer sets are read from global memory);
  // KNNG_SET_SLOTCH overrides (measurement)
  int setch = 16;
  if (const char *e = getenv("KNNG_SET_SLOTCH")) setch = std::max(1, std::min(64, atoi(e)));
  a.pitch = sets ? setch * 16 + 16 : (int)g->geom.stride + (a.swz ? 0 : 16);

  // walk steps copy the rows of all of cur's neighbours with their vectors when the vectors dominate the
  // step's bytes anyway (measured: C2's 384-byte rows gain 6%, the 128-byte rows of C1/C3/C4 lose 12-17%)
  a.row_pf = !sets && g->geom.stride >= 256;
  if (const char *e = getenv("KNNG_ROW_PF")) a.row_pf = atoi(e) != 0;
  a.win_prefetch = 1;
  if (const char *e = getenv("KNNG_WIN_PREFETCH")) a.win_prefetch = atoi(e) != 0;
  if (a.srows) a.win_prefetch = 0;   // rows already in shared memory (the prefetch copies from global)
  // latency-bound launches (every task resident at once): the E bitmap (and, if it fits too, the X
  // bitmap) in shared memory and two chunk stages, if that plan still holds every task; else the E / X
  // bits in the per-slot global words and one stage
  int64_t warps = 0;
  a.e_smem = 0;
  a.x_smem = 0;
  a.ns2 = 0;
  a.e_bytes = 0;
  const int64_t eb = (((mmax + 31) / 32) * 4 + 15) & ~15ll;   // one bitmap
  int es_mode = -1;   // -1: automatic
  if (const char *e = getenv("KNNG_ESMEM")) es_mode = atoi(e);
  if (a.kt) {   // the key table's launch: E and X in shared memory, no chunk stages in flight
    a.e_smem = 1;
    a.x_smem = 1;
    a.e_bytes = (int)eb;
  } else if (!sets && es_mode != 0 && eb <= 64 * 1024) {
    for (int xs = 1; xs >= 0 && !a.e_smem; --xs) {
      SearchArgs t = a;
      t.e_smem = 1;
      t.x_smem = xs;
      t.ns2 = 1;
      t.e_bytes = (int)eb;
      if (const char *e = getenv("KNNG_NS2")) t.ns2 = atoi(e) != 0;
      if (const char *e = getenv("KNNG_XSMEM")) t.x_smem = atoi(e) != 0;
      int64_t w2 = 0;
      if (search_resident_warps(g->geom, t, &w2) == cudaSuccess && w2 > 0 && (es_mode == 1 || w2 >= tasks)) {
        a.e_smem = 1;
        a.x_smem = t.x_smem;
        a.ns2 = t.ns2;
        a.e_bytes = t.e_bytes;
      }
    }
  }
  // global E words: draws set no E bits and read their words only when the warp's W filter hits (perm_e;
  // KNNG_PERM_E=0 restores E bits for every evaluation -- same results, measurement and tests)
  // (vectors only: the set evaluators are ALU-bound and smem-limited, where the filter's 4 KB per warp and the
  // pi^-1 per walk neighbour cost more than the E traffic saved -- C4 at 500k 24.1 vs 19.9 ms)
  a.perm_e = !a.e_smem && !a.kt && a.starts == nullptr && !sets;
  if (const char *e = getenv("KNNG_PERM_E")) a.perm_e = a.perm_e && atoi(e) != 0;
  // one-stage plans of the lane-form widths: the rows are gathered by the TMA engine (one bulk copy per row
  // on the warp's mbarrier instead of 16-byte cp.async per lane; measured C2 -3%, C3 at 2M -4.5%, C3 at 8M
  // equal: profiles/round2/k1_ab_bulk.txt); KNNG_BULK=0 restores the cp.async gathers (measurement, tests)
  a.bulk = 0;
  if (lform && !a.ns2 && !a.kt) {
    a.bulk = 1;
    if (const char *e = getenv("KNNG_BULK")) a.bulk = atoi(e) != 0;
  }
  if (a.bulk) {
    a.swz = 0;
    a.pitch = (int)g->geom.stride + 16;
  }
  CK(search_resident_warps(g->geom, a, &warps));
  a.gslots = std::min<int64_t>(warps, (tasks + 3) / 4 * 4);
  return 0;
}

// Largest partition pool (sizes the search's workspaces; the kernel reads the exact sizes on the
// device).  An upper bound kept on the host -- exact after the asynchronous read-back that follows
// every placement, else the last exact value plus the points placed since -- so no search waits on
// the device for it.
static int max_pool(knng_graph *g, int64_t *out) {
  if (g->P == 0) { *out = g->n; return 0; }
  if (!g->h_cnt) CK(cudaMallocHost((void **)&g->h_cnt, 256 * sizeof(int64_t)));
  if (!g->ev_cnt) CK(cudaEventCreateWithFlags(&g->ev_cnt, cudaEventDisableTiming));
  if (g->cnt_pending && cudaEventQuery(g->ev_cnt) == cudaSuccess) {
    int64_t m = 0;
    for (int p = 0; p < g->P; ++p) m = std::max(m, g->h_cnt[p]);
    g->pool_bound = m + (g->n - g->cnt_n);   // + the points placed since the read-back was issued
    g->cnt_pending = false;
  }
  if (g->pool_bound <= 0) {   // first search after partitioning: one synchronous read
    CK(cudaMemcpyAsync(g->h_cnt, g->member_cnt, sizeof(int64_t) * g->P, cudaMemcpyDeviceToHost, g->stream));
    CK(cudaStreamSynchronize(g->stream));
    int64_t m = 0;
    for (int p = 0; p < g->P; ++p) m = std::max(m, g->h_cnt[p]);
    g->pool_bound = m;
  }
  *out = g->pool_bound;
  return 0;
}

// K1 over partitions [part_lo, part_hi) (unpartitioned: [0, 1)): raw per-partition candidates
// [nq][part_hi-part_lo][kr] into out_i / out_k.
static int run_search_phase(knng_graph *g, const StoreView &qs, int64_t qrow0, int64_t nq, int64_t pid_base, int kr,
                            const knng_params *p, const int32_t *d_starts, int nstarts, int part_lo, int part_hi,
                            int32_t *out_i, uint32_t *out_k, int *nl) {
  int64_t mmax = 0;
  if (int r = max_pool(g, &mmax)) return r;
  if (g->P > 0 && mmax == 0) return fail(KNNG_ERR_EMPTY, "all partitions are empty");
  // routing variant (reading Q18): one task per query, on the partition of its nearest medoid
  const bool routed = p->route && g->P > 0;
  if (routed) {
    CK(g->w_route.ensure((size_t)std::max<int64_t>(nq, 1) * 4));
    CK(launch_route_target(g->geom, qs, qrow0, nq, graph_store_view(g), g->P, g->medoids, g->w_route.as<int32_t>(),
                           g->stream));
    ++*nl;
    part_lo = 0;
    part_hi = 1;
  }
  const int pc = part_hi - part_lo;
  SearchArgs a;
  memset(&a, 0, sizeof a);
  a.metric = g->metric;
  a.st = graph_store_view(g);
  a.qs = qs;
  a.qrow0 = qrow0;
  a.rows = g->ids;
  a.k = g->k;
  a.n_t = g->n;
  a.nq = nq;
  a.pid_base = pid_base;
  a.P = g->P;
  a.part_lo = part_lo;
  a.part_cnt = pc;
  a.members = g->members;
  a.member_cap = g->cap;
  a.member_cnt = g->member_cnt;
  a.part_of = g->part_of;
  a.local_idx = g->local_idx;
  a.prow = g->prow;
  a.pvec = g->pvec;
  a.pset = g->pset;
  a.speedup = p->speedup;
  a.e_num = p->expansion_num;
  a.e_den = p->expansion_den;
  a.seed = p->seed;
  a.kr = kr;
  a.starts = d_starts;
  a.nstarts = nstarts;
  a.full_scan = p->full_scan != 0;
  a.route = routed ? g->w_route.as<int32_t>() : nullptr;
  a.out_ids = out_i;
  a.out_keys = out_k;
  a.stats = g->w_stats.as<unsigned long long>();
  a.prof = getenv("KNNG_PROFILE") ? a.stats + 16 : nullptr;  // cycle counters -> stats[16..31]
  if (a.prof) g->tprof_n = nq * pc;
  a.task_ctr = a.stats + 14;
  if (g->fuse_b1) {
    a.fuse = 1;
    a.nseq = (int)g->fuse_nseq;
    a.ub = *g->fuse_b1;
    a.ub.st = graph_store_view(g);   // after the ingest: a set / string store may have grown (moved) since
    mmax = g->n + g->fuse_nseq;   // the pool of the last insert of the sequence
    // small graphs: the sequence's keys against the whole pool, computed densely by one launch and
    // staged per insert in shared memory (<= 32 KB) for the search and the update
    a.kt = mmax <= 8192 && !getenv("KNNG_NO_KT");
    // the rows too when they fit (<= 160 KB): the walks' and the update's row reads become shared-memory reads
    a.srows = a.kt && mmax * g->k * 4 <= 160 * 1024 && !getenv("KNNG_NO_SROWS");
    if (a.kt) {
      a.ktm_ld = (mmax + 3) & ~3ll;
      CK(g->w_ktm.ensure((size_t)g->fuse_nseq * a.ktm_ld * 4));
      a.ktm = g->w_ktm.as<uint32_t>();
      CK(launch_keymat(g->metric, qs, qrow0, g->n, g->fuse_nseq, a.ktm_ld, g->w_ktm.as<uint32_t>(), g->stream));
      ++*nl;
    }
  }
  if (int r = plan_k1(g, a, nq * pc, mmax)) return r;
  CK(g->w_bits.ensure((size_t)a.gslots * a.de_words * 4));
  a.gbits = g->w_bits.as<uint32_t>();
  cudaError_t e = launch_search(g->geom, a, g->stream, nl);
  if (e != cudaSuccess) return fail(KNNG_ERR_CUDA, "search launch: %s", cudaGetErrorString(e));
  return 0;
}

static void fill_stats(knng_graph *g, knng_stats *st, const unsigned long long *h, int nl, int nev) {
  if (!st) return;
  memset(st, 0, sizeof *st);
  st->search_evals = (int64_t)h[0];
  st->search_starts = (int64_t)h[1];
  st->search_skipped = (int64_t)h[2];
  st->search_expansions = (int64_t)h[3];
  st->ball_nodes = (int64_t)h[4];
  st->proposals = (int64_t)h[5];
  st->allpair_pairs = (int64_t)h[6];
  st->kernel_launches = nl;
  float ms = 0;
  if (nev >= 2) { cudaEventElapsedTime(&ms, g->ev[0], g->ev[1]); st->ms_search = ms; }
  if (nev >= 3) { cudaEventElapsedTime(&ms, g->ev[1], g->ev[2]); st->ms_allpairs = ms; }
  if (nev >= 4) { cudaEventElapsedTime(&ms, g->ev[2], g->ev[3]); st->ms_update = ms; }
  if (nev >= 5) { cudaEventElapsedTime(&ms, g->ev[3], g->ev[4]); st->ms_merge = ms; }
  if (nev >= 2) { cudaEventElapsedTime(&ms, g->ev[0], g->ev[nev - 1]); st->ms_total = ms; }
}

// ---------------------------------------------------------------------------------------------
// graph_insert_batch in three stages.  One GPU runs them back to back; the multi-GPU driver
// (paper_1602_06819_b200/dist.py) runs them on every rank with two all-gathers in between:
//   search : ingest the batch (rows n_t..), K1 over this rank's partitions   -> candidates
//   update : K2 merge of all ranks' candidates, K3 all-pairs (all B), K4 balls of this rank's
//            query shard                                                      -> proposals
//   commit : K5 merge of all ranks' proposals, K6 placement, n_t += B  (identical on every rank)
// ---------------------------------------------------------------------------------------------
static int64_t ball_bound(int64_t n_t, int k, int depth) {   // k + k^2 + ... + k^DEPTH, <= n_t
  int64_t ballmax = 0, pw = 1;
  for (int d = 1; d <= depth && ballmax < n_t; ++d) {
    pw *= k;
    ballmax += pw;
  }
  return ballmax > n_t ? n_t : ballmax;
}

static int stage_search(knng_graph *g, const knng_points *pts, const knng_params *p, int part_lo, int part_hi,
                        int64_t q_lo, int64_t q_hi, int32_t *ci, uint32_t *ck, int *nl) {
  if (int r = check_points(pts, "insert")) return r;
  if (int r = check_params(p)) return r;
  if (pts->metric != g->metric || (!csr_points(g->metric) && pts->dim != g->dim))
    return fail(KNNG_ERR_INVALID_ARG, "insert: metric/dim mismatch");
  if (p->depth < 1 || p->depth > 10) return fail(KNNG_ERR_INVALID_ARG, "depth %d outside 1..10", p->depth);
  const int Pn = g->P > 0 ? g->P : 1;
  if (part_lo < 0 || part_hi > Pn || part_lo >= part_hi) return fail(KNNG_ERR_INVALID_ARG, "bad partition range");
  const int64_t B = pts->n, n_t = g->n;
  if (n_t + B > g->cap)
    return fail(KNNG_ERR_CAPACITY_EXCEEDED, "capacity %lld exceeded (n=%lld, B=%lld)", (long long)g->cap,
                (long long)n_t, (long long)B);
  if (q_lo < 0) q_hi = B, q_lo = 0;          // all queries
  if (q_hi > B || q_lo > q_hi) return fail(KNNG_ERR_INVALID_ARG, "bad query range");
  g->pend_B = B;
  g->pend_parts = part_hi - part_lo;
  g->pend_route = p->route && g->P > 0;
  if (B == 0) return 0;
  // A1: batch ingest into the store tail (ids n_t .. n_t+B-1)
  if (int r = store_points(g, pts, n_t)) return r;
  // A2-A3: iGNNS per (point, partition) on the snapshot, for queries [q_lo, q_hi)
  if (q_hi == q_lo) return 0;
  if (p->full_scan) return fail(KNNG_ERR_INVALID_ARG, "insert: full_scan (the GNNS baseline) is a graph_search mode");
  return run_search_phase(g, graph_store_view(g), n_t + q_lo, q_hi - q_lo, n_t + q_lo, g->k, p, nullptr, 0, part_lo,
                          part_hi, ci, ck, nl);
}

static int stage_update(knng_graph *g, const knng_params *p, int world, const int32_t *ci_all, const uint32_t *ck_all,
                        int64_t q_lo, int64_t q_hi, int2 *props, int32_t *prop_cnt, int32_t *new_ids,
                        uint32_t *new_keys, int *nl, bool timed) {
  const int64_t B = g->pend_B, n_t = g->n;
  const int k = g->k;
  if (B == 0) return 0;
  const StoreView sv = graph_store_view(g);
  // A4: keep the k best of the P*k per-partition candidates (all-gathered, rank-major)
  int32_t *Ci = (int32_t *)ci_all;
  uint32_t *Ck = (uint32_t *)ck_all;
  if (g->P > 0 && !g->pend_route) {
    if (g->P % world) return fail(KNNG_ERR_INVALID_ARG, "P=%d not divisible by world=%d", g->P, world);
    if (g->pend_parts * world != g->P)   // the gathered candidates must cover every partition
      return fail(KNNG_ERR_INVALID_ARG, "stage_update: %d ranks x %d searched partitions != P=%d", world, g->pend_parts,
                  g->P);
    CK(g->w_C_i.ensure((size_t)B * k * 4));
    CK(g->w_C_k.ensure((size_t)B * k * 4));
    Ci = g->w_C_i.as<int32_t>();
    Ck = g->w_C_k.as<uint32_t>();
    CK(launch_merge_parts(g->metric, ci_all, ck_all, B, g->P, world, k, Ci, Ck, g->stream));
    ++*nl;
  }
  if (timed) CK(cudaEventRecord(g->ev[1], g->stream));
  // A5: intra-batch all-pairs -> new rows of queries [q_lo, q_hi) (into the graph, or into new_ids/new_keys
  // for the all-gather of a multi-GPU job)
  int32_t *oi = new_ids ? new_ids : g->ids + (size_t)(n_t + q_lo) * k;
  uint32_t *ok = new_keys ? new_keys : g->keys + (size_t)(n_t + q_lo) * k;
  CK(launch_allpairs(g->geom, sv, n_t, B, q_lo, q_hi - q_lo, k, Ci + (size_t)q_lo * k, Ck + (size_t)q_lo * k, oi, ok,
                     &g->w_dense, g->stream));
  ++*nl;
  if (timed) CK(cudaEventRecord(g->ev[2], g->stream));
  // A6: update balls of queries [q_lo, q_hi) over the snapshot -> proposals
  const int64_t ballmax = ball_bound(n_t, k, p->depth);
  int hcap = 64;
  while (hcap < 2 * ballmax) hcap <<= 1;
  const int64_t nqb = q_hi - q_lo;
  const int64_t bslots = std::max<int64_t>(1, std::min<int64_t>((nqb + 3) / 4, 148 * 8)) * 4;
  CK(g->w_hash.ensure((size_t)bslots * hcap * 4));
  CK(g->w_list.ensure((size_t)bslots * ballmax * 4));
  BallArgs ba;
  memset(&ba, 0, sizeof ba);
  ba.st = sv;
  ba.ids = g->ids;
  ba.keys = g->keys;
  ba.k = k;
  ba.n_t = n_t;
  ba.B = B;
  ba.q0 = q_lo;
  ba.nqb = nqb;
  ba.depth = p->depth;
  ba.C = Ci;
  ba.hash = g->w_hash.as<int32_t>();
  ba.hcap = hcap;
  ba.list = g->w_list.as<int32_t>();
  ba.ballmax = (int)ballmax;
  // small balls (depth 2, k <= 16: <= 4 KB of hash + list per warp) keep their sets in shared memory
  // (JW: 24 KB of the 48 KB static budget hold the per-lane character pointers)
  ba.smem_ball = (size_t)4 * (hcap + ballmax) * 4 <= (g->metric == KNNG_JARO_WINKLER ? 16 : 24) * 1024 ? 1 : 0;
  if (const char *e = getenv("KNNG_SMEM_BALL")) ba.smem_ball = atoi(e) != 0 && ba.smem_ball;
  ba.props = props;
  ba.prop_cnt = prop_cnt;
  ba.stats = g->w_stats.as<unsigned long long>();
  CK(launch_ball(g->geom, ba, bslots, g->stream));
  ++*nl;
  return 0;
}

static int stage_commit(knng_graph *g, const knng_params *p, int64_t nq_slots, const int2 *props_all,
                        const int32_t *prop_cnt_all, const int32_t *new_ids_all, const uint32_t *new_keys_all,
                        int *nl) {
  const int64_t B = g->pend_B, n_t = g->n;
  if (B == 0) return 0;
  if (new_ids_all) {   // the all-gathered new rows (slot b = query b)
    CK(cudaMemcpyAsync(g->ids + (size_t)n_t * g->k, new_ids_all, (size_t)B * g->k * 4, cudaMemcpyDeviceToDevice,
                       g->stream));
    CK(cudaMemcpyAsync(g->keys + (size_t)n_t * g->k, new_keys_all, (size_t)B * g->k * 4, cudaMemcpyDeviceToDevice,
                       g->stream));
  }
  const int64_t ballmax = ball_bound(n_t, g->k, p->depth);
  CK(g->w_sorted.ensure((size_t)nq_slots * ballmax * 8));
  // A8: placement at the nearest medoid.  It reads only the new points and the medoids, and the
  // search of this batch is complete, so it runs before the merge: the merged rows' partition-local
  // copies (prow) then see the new ids' partitions.
  if (g->P > 0) {
    CK(g->w_target.ensure((size_t)B * 4));
    CK(launch_place(g->geom, graph_store_view(g), n_t, B, g->P, g->medoids, g->members, g->cap, g->member_cnt,
                    g->part_of, g->local_idx, g->w_target.as<int32_t>(), g->stream));
    *nl += 2;
  }
  // A7: row_v = top-k(row_v u proposals), proposal (slot b) carries the new id n_t + b
  CK(launch_merge_props(g->metric, g->ids, g->keys, g->k, n_t, nq_slots, props_all, prop_cnt_all, (int)ballmax,
                        g->ncnt, g->nfill, g->noff, g->scan_tmp, g->w_sorted.as<int2>(), g->stream, nl,
                        g->P > 0 ? g->prow : nullptr, g->cap, g->part_of, g->local_idx));
  if (g->P > 0) {   // the new nodes' partition-local store (rows, vectors / token ranges)
    CK(launch_local_store(graph_store_view(g), g->ids, g->k, n_t, B, g->part_of, g->local_idx, graph_local_store(g),
                          g->stream));
    *nl += 2;
    // partition sizes: bound now, exact once the read-back lands
    if (g->pool_bound > 0) g->pool_bound += B;
    if (g->h_cnt && g->ev_cnt && !g->cnt_pending) {
      CK(cudaMemcpyAsync(g->h_cnt, g->member_cnt, sizeof(int64_t) * g->P, cudaMemcpyDeviceToHost, g->stream));
      CK(cudaEventRecord(g->ev_cnt, g->stream));
      g->cnt_pending = true;
      g->cnt_n = n_t + B;
    }
  }
  g->n = n_t + B;
  g->pend_B = 0;
  return 0;
}

static void print_profile(knng_graph *g, const unsigned long long *h, int64_t B) {
  if (!getenv("KNNG_PROFILE") || B <= 0 || !h[16]) return;
  const double T = (double)g->tprof_n > 0 ? (double)g->tprof_n : (double)B;
  fprintf(stderr, "KNNG_PROFILE per task (%.0f tasks): %.0f cyc, walks %.0f | chunks %.1f (fast %.1f, windows %.1f) | "
          "walk steps %.1f\n", T, h[16] / T, h[18] / T, h[25] / T, h[24] / T, h[21] / T, h[22] / T);
  if (h[22])
    fprintf(stderr, "KNNG_PROFILE walk step: %.0f cyc = row %.0f + copies/keys %.0f + commit %.0f (+ move)\n",
            (double)h[18] / h[22], (double)h[26] / h[22], (double)h[27] / h[22], (double)h[28] / h[22]);
  if (h[25])
    fprintf(stderr, "KNNG_PROFILE chunk: draw+gather+keys %.0f cyc; fast chunks: decision %.0f + commit %.0f cyc\n",
            (double)h[29] / h[25], h[24] ? (double)h[30] / h[24] : 0.0, h[24] ? (double)h[31] / h[24] : 0.0);
}

static int finish_stats(knng_graph *g, knng_stats *st, int nl, int nev, int64_t B) {
  unsigned long long h[32];
  CK(cudaMemcpyAsync(h, g->w_stats.p, 32 * 8, cudaMemcpyDeviceToHost, g->stream));
  CK(cudaStreamSynchronize(g->stream));
  h[6] = (unsigned long long)(B * (B - 1));
  print_profile(g, h, B);
  fill_stats(g, st, h, nl, nev);
  return 0;
}

static int insert_batch_dist(knng_graph *g, const knng_points *pts, const knng_params *p, knng_stats *st);

// Sequential inserts on an unpartitioned single-GPU graph -- the paper's sequential algorithm (Alg. 1 +
// Alg. 2 per point): ingest all n points (rows n_t.., invisible to the searches until their
// turn), then ONE launch in which a warp searches (K1, one task) and runs the update (new row = C,
// ball, proposals applied in place) point after point, and one synchronisation for the stats.
static int insert_seq(knng_graph *g, const knng_points *pts, const knng_params *p, knng_stats *st) {
  int nl = 0;
  const int64_t n_t = g->n, B = pts->n;
  const int64_t ballmax = ball_bound(n_t + B - 1, g->k, p->depth);
  int hcap = 64;
  while (hcap < 2 * ballmax) hcap <<= 1;
  CK(g->w_stats.ensure(32 * 8));
  CK(g->w_cand_i.ensure((size_t)g->k * 4));
  CK(g->w_cand_k.ensure((size_t)g->k * 4));
  if (getenv("KNNG_PROFILE")) CK(cudaMemsetAsync(g->w_stats.p, 0, 32 * 8, g->stream));   // cycle counters add up
  BallArgs ba;
  memset(&ba, 0, sizeof ba);
  ba.st = graph_store_view(g);
  ba.ids = g->ids;
  ba.keys = g->keys;
  ba.k = g->k;
  ba.n_t = n_t;
  ba.B = 1;
  ba.depth = p->depth;
  ba.C = g->w_cand_i.as<int32_t>();
  ba.hcap = hcap;
  ba.ballmax = (int)ballmax;
  ba.stats = g->w_stats.as<unsigned long long>();
  CK(cudaEventRecord(g->ev[0], g->stream));
  g->fuse_b1 = &ba;
  g->fuse_nseq = B;
  const int r = stage_search(g, pts, p, 0, 1, 0, 1, g->w_cand_i.as<int32_t>(), g->w_cand_k.as<uint32_t>(), &nl);
  g->fuse_b1 = nullptr;
  g->fuse_nseq = 0;
  if (r) {
    g->pend_B = 0;
    return r;
  }
  CK(cudaEventRecord(g->ev[1], g->stream));
  g->n = n_t + B;
  g->pend_B = 0;
  g->tprof_n = B;
  const int rc = finish_stats(g, st, nl, 2, 1);
  g->tprof_n = 0;
  if (st) st->allpair_pairs = 0;
  return rc;
}

static bool seq_fusable(const knng_graph *g, const knng_points *pts, const knng_params *p) {
  return pts && pts->n >= 1 && g->P == 0 && !g->comm && p && p->depth >= 1 && p->depth <= 10 &&
         !getenv("KNNG_NO_B1") && g->n + pts->n <= g->cap && ball_bound(g->n + pts->n - 1, g->k, p->depth) <= 4096;
}

int graph_insert_batch(knng_graph *g, const knng_points *pts, const knng_params *p, int64_t *first_id_out,
                       knng_stats *st) {
  knng_err_slot().clear();
  if (!g) return fail(KNNG_ERR_INVALID_ARG, "graph_insert_batch: null graph");
  if (g->pend_B) return fail(KNNG_ERR_INVALID_ARG, "graph_insert_batch: a staged batch is pending");
  if (first_id_out) *first_id_out = g->n;
  CK(cudaSetDevice(g->device));
  if (g->comm) return insert_batch_dist(g, pts, p, st);
  // the sequential algorithm's fast path (the ball of a B = 1 insert fits one warp's shared memory)
  if (pts && pts->n == 1 && seq_fusable(g, pts, p)) return insert_seq(g, pts, p, st);
  CK(g->w_stats.ensure(32 * 8));
  CK(cudaMemsetAsync(g->w_stats.p, 0, 32 * 8, g->stream));
  const int64_t B = pts ? pts->n : 0, k = g->k;
  const int Pn = g->P > 0 ? g->P : 1;
  CK(g->w_cand_i.ensure((size_t)std::max<int64_t>(B, 1) * Pn * k * 4));
  CK(g->w_cand_k.ensure((size_t)std::max<int64_t>(B, 1) * Pn * k * 4));
  int nl = 0;
  CK(cudaEventRecord(g->ev[0], g->stream));
  if (int r = stage_search(g, pts, p, 0, Pn, -1, -1, g->w_cand_i.as<int32_t>(), g->w_cand_k.as<uint32_t>(), &nl)) {
    g->pend_B = 0;   // a failed batch leaves the graph as it was (its points are past n)
    return r;
  }
  if (B == 0) {
    g->pend_B = 0;
    return finish_stats(g, st, 0, 0, 0);
  }
  const int64_t ballmax = ball_bound(g->n, g->k, p->depth);
  CK(g->w_props.ensure((size_t)B * ballmax * 8));
  CK(g->w_prop_cnt.ensure((size_t)B * 4));
  if (int r = stage_update(g, p, 1, g->w_cand_i.as<int32_t>(), g->w_cand_k.as<uint32_t>(), 0, B,
                           g->w_props.as<int2>(), g->w_prop_cnt.as<int32_t>(), nullptr, nullptr, &nl, true)) {
    g->pend_B = 0;
    return r;
  }
  CK(cudaEventRecord(g->ev[3], g->stream));
  if (int r = stage_commit(g, p, B, g->w_props.as<int2>(), g->w_prop_cnt.as<int32_t>(), nullptr, nullptr, &nl)) {
    g->pend_B = 0;
    return r;
  }
  CK(cudaEventRecord(g->ev[4], g->stream));
  return finish_stats(g, st, nl, 5, B);
}

int graph_insert_sequential(knng_graph *g, const knng_points *pts, const knng_params *p, int64_t *first_id_out,
                            knng_stats *st) {
  knng_err_slot().clear();
  if (!g) return fail(KNNG_ERR_INVALID_ARG, "graph_insert_sequential: null graph");
  if (g->pend_B) return fail(KNNG_ERR_INVALID_ARG, "graph_insert_sequential: a staged batch is pending");
  if (first_id_out) *first_id_out = g->n;
  if (int r = check_points(pts, "insert")) return r;
  if (st) memset(st, 0, sizeof *st);
  if (pts->n == 0) return 0;
  CK(cudaSetDevice(g->device));
  if (seq_fusable(g, pts, p)) return insert_seq(g, pts, p, st);
  // otherwise one graph_insert_batch of one point after another (views into the caller's points)
  std::vector<uint64_t> hoff;
  if (csr_points(pts->metric)) {
    hoff.resize((size_t)pts->n + 1);
    if (pts->data_on_device)
      CK(cudaMemcpy(hoff.data(), pts->offsets, hoff.size() * 8, cudaMemcpyDeviceToHost));
    else
      memcpy(hoff.data(), pts->offsets, hoff.size() * 8);
  }
  uint64_t *doff = nullptr;   // 2-entry offsets of a one-set view, in the caller's memory space
  if (csr_points(pts->metric) && pts->data_on_device) CK(cudaMalloc(&doff, 16));
  knng_stats acc;
  memset(&acc, 0, sizeof acc);
  int rc = 0;
  for (int64_t i = 0; i < pts->n && rc == 0; ++i) {
    knng_points one = *pts;
    one.n = 1;
    uint64_t ho[2];
    if (csr_points(pts->metric)) {
      ho[0] = 0;
      ho[1] = hoff[i + 1] - hoff[i];
      one.data = (const uint32_t *)pts->data + hoff[i];
      if (doff) {
        if (cudaMemcpy(doff, ho, 16, cudaMemcpyHostToDevice) != cudaSuccess) { rc = fail(KNNG_ERR_CUDA, "offsets"); break; }
        one.offsets = doff;
      } else {
        one.offsets = ho;
      }
    } else {
      one.data = (const uint8_t *)pts->data + (size_t)i * pts->dim * (pts->metric == KNNG_L2SQ_U8 ? 1 : 4);
    }
    knng_stats s1;
    rc = graph_insert_batch(g, &one, p, nullptr, &s1);
    if (rc == 0) {
      acc.search_evals += s1.search_evals;
      acc.search_starts += s1.search_starts;
      acc.search_skipped += s1.search_skipped;
      acc.search_expansions += s1.search_expansions;
      acc.ball_nodes += s1.ball_nodes;
      acc.proposals += s1.proposals;
      acc.kernel_launches += s1.kernel_launches;
      acc.ms_search += s1.ms_search;
      acc.ms_allpairs += s1.ms_allpairs;
      acc.ms_update += s1.ms_update;
      acc.ms_merge += s1.ms_merge;
      acc.ms_total += s1.ms_total;
    }
  }
  if (doff) cudaFree(doff);
  if (st) *st = acc;
  return rc;
}

// ---------------------------------------------------------------------------------------------
// graph_insert_batch on G ranks (Alg. 3 + Alg. 5 across GPUs): every rank
// holds a full replica and makes the same call with the same batch; everything is stream-ordered on
// the handle's stream, with the library's NCCL all-gathers between the stages and no host sync:
//   search   partitioned: this rank's partitions [r P/G, (r+1) P/G) for all B points -> cand [B][P/G][k]
//            unpartitioned: all partitions for the query shard [r S, r S + S)         -> cand [S][1][k]
//   all-gather cand ("the compute nodes send the k.p candidates")
//   update   K2 merge (identical on every rank), new rows + balls of the query shard [r S, r S + S)
//   all-gather new rows, proposals and their counts (S slots per rank)
//   commit   write the new rows, apply every proposal, place the points (identical on every rank)
// The counters are summed over the ranks (one more all-reduce), so every rank reports the job's.
// ---------------------------------------------------------------------------------------------
static int nccl_ck(const char *m) { return m ? fail(KNNG_ERR_NCCL, "%s", m) : 0; }

static int insert_batch_dist_(knng_graph *g, const knng_points *pts, const knng_params *p, knng_stats *st);
static int insert_batch_dist(knng_graph *g, const knng_points *pts, const knng_params *p, knng_stats *st) {
  const int rc = insert_batch_dist_(g, pts, p, st);
  if (rc) g->pend_B = 0;
  return rc;
}
static int insert_batch_dist_(knng_graph *g, const knng_points *pts, const knng_params *p, knng_stats *st) {
  const int G = g->world, r = g->rank, k = g->k;
  const int64_t B = pts ? pts->n : 0, n_t = g->n;
  const int P = g->P;
  if (P > 0 && P % G) return fail(KNNG_ERR_INVALID_ARG, "P=%d is not a multiple of the world size %d", P, G);
  if (p && p->route) return fail(KNNG_ERR_INVALID_ARG, "route: single-GPU handles only");
  const int64_t S = (B + G - 1) / G;                     // query slots per rank (balls, new rows)
  const int64_t qlo = std::min<int64_t>(r * S, B), qhi = std::min<int64_t>(qlo + S, B);
  if (p && (p->depth < 1 || p->depth > 10)) return fail(KNNG_ERR_INVALID_ARG, "depth %d outside 1..10", p->depth);
  const int64_t ballmax = p ? ball_bound(n_t, k, p->depth) : 0;
  const int pown = P > 0 ? P / G : 1;
  const int64_t cand_rows = P > 0 ? B : S;               // rows of this rank's candidate buffer
  const size_t cand_n = (size_t)std::max<int64_t>(cand_rows, 1) * pown * k;
  CK(g->w_dci.ensure(cand_n * 4));
  CK(g->w_dck.ensure(cand_n * 4));
  CK(g->w_gci.ensure(cand_n * G * 4));
  CK(g->w_gck.ensure(cand_n * G * 4));
  const size_t sl = (size_t)std::max<int64_t>(S, 1);
  CK(g->w_dprops.ensure(sl * std::max<int64_t>(ballmax, 1) * 8));
  CK(g->w_dcnt.ensure(sl * 4));
  CK(g->w_dnid.ensure(sl * k * 4));
  CK(g->w_dnkey.ensure(sl * k * 4));
  CK(g->w_gprops.ensure(sl * G * std::max<int64_t>(ballmax, 1) * 8));
  CK(g->w_gcnt.ensure(sl * G * 4));
  CK(g->w_gnid.ensure(sl * G * k * 4));
  CK(g->w_gnkey.ensure(sl * G * k * 4));
  CK(g->w_dstats.ensure(16 * 8));
  CK(g->w_stats.ensure(32 * 8));
  CK(cudaMemsetAsync(g->w_stats.p, 0, 32 * 8, g->stream));
  int nl = 0;
  CK(cudaEventRecord(g->ev[0], g->stream));
  // candidate slots this rank does not fill (short last shard) stay empty: -1 ids
  CK(cudaMemsetAsync(g->w_dci.p, 0xFF, cand_n * 4, g->stream));
  if (int rc = stage_search(g, pts, p, P > 0 ? r * pown : 0, P > 0 ? (r + 1) * pown : 1, P > 0 ? -1 : qlo,
                            P > 0 ? -1 : qhi, g->w_dci.as<int32_t>(), g->w_dck.as<uint32_t>(), &nl)) {
    g->pend_B = 0;
    return rc;
  }
  if (B == 0) {
    g->pend_B = 0;
    return finish_stats(g, st, nl, 0, 0);
  }
  if (int rc = nccl_ck(knng::nccl_allgather(g->w_dci.p, g->w_gci.p, cand_n, ncclInt32, g->comm, g->stream))) return rc;
  if (int rc = nccl_ck(knng::nccl_allgather(g->w_dck.p, g->w_gck.p, cand_n, ncclInt32, g->comm, g->stream))) return rc;
  CK(cudaEventRecord(g->ev[1], g->stream));
  CK(cudaMemsetAsync(g->w_dcnt.p, 0, sl * 4, g->stream));
  CK(cudaMemsetAsync(g->w_dnid.p, 0xFF, sl * k * 4, g->stream));
  // the gathered candidates: partitioned [G][B][P/G][k] (rank-major, merged by K2 with world = G);
  // unpartitioned [G*S][1][k], row b = query b (world = 1)
  if (int rc = stage_update(g, p, P > 0 ? G : 1, g->w_gci.as<int32_t>(), g->w_gck.as<uint32_t>(), qlo, qhi,
                            g->w_dprops.as<int2>(), g->w_dcnt.as<int32_t>(), g->w_dnid.as<int32_t>(),
                            g->w_dnkey.as<uint32_t>(), &nl, false))
    return rc;
  CK(cudaEventRecord(g->ev[2], g->stream));
  if (int rc = nccl_ck(knng::nccl_group_start())) return rc;
  const char *m = knng::nccl_allgather(g->w_dprops.p, g->w_gprops.p, sl * std::max<int64_t>(ballmax, 1) * 2, ncclInt32,
                                       g->comm, g->stream);
  if (!m) m = knng::nccl_allgather(g->w_dcnt.p, g->w_gcnt.p, sl, ncclInt32, g->comm, g->stream);
  if (!m) m = knng::nccl_allgather(g->w_dnid.p, g->w_gnid.p, sl * k, ncclInt32, g->comm, g->stream);
  if (!m) m = knng::nccl_allgather(g->w_dnkey.p, g->w_gnkey.p, sl * k, ncclInt32, g->comm, g->stream);
  const char *m2 = knng::nccl_group_end();
  if (int rc = nccl_ck(m ? m : m2)) return rc;
  CK(cudaEventRecord(g->ev[3], g->stream));
  // the ball slots are ballmax wide on every rank (same n_t, k, depth)
  if (int rc = stage_commit(g, p, G * S, g->w_gprops.as<int2>(), g->w_gcnt.as<int32_t>(), g->w_gnid.as<int32_t>(),
                            g->w_gnkey.as<uint32_t>(), &nl))
    return rc;
  // job-wide counters
  if (int rc = nccl_ck(knng::nccl_allreduce_sum(g->w_stats.p, g->w_dstats.p, 8, ncclInt64, g->comm, g->stream)))
    return rc;
  CK(cudaMemcpyAsync(g->w_stats.p, g->w_dstats.p, 8 * 8, cudaMemcpyDeviceToDevice, g->stream));
  CK(cudaEventRecord(g->ev[4], g->stream));
  return finish_stats(g, st, nl, 5, B);
}

// ---- the stages as C-ABI calls (multi-GPU building blocks; device buffers) ----
int64_t graph_ball_bound(const knng_graph *g, int32_t depth) {
  if (!g || depth < 1) return -1;
  return ball_bound(g->n, g->k, depth);
}

int graph_insert_stage_search(knng_graph *g, const knng_points *pts, const knng_params *p, int32_t part_lo,
                              int32_t part_hi, int64_t q_lo, int64_t q_hi, int32_t *cand_ids, uint32_t *cand_keys,
                              knng_stats *st) {
  knng_err_slot().clear();
  if (!g) return fail(KNNG_ERR_INVALID_ARG, "stage_search: null graph");
  if (g->pend_B) return fail(KNNG_ERR_INVALID_ARG, "stage_search: a staged batch is pending");
  CK(cudaSetDevice(g->device));
  CK(g->w_stats.ensure(32 * 8));
  CK(cudaMemsetAsync(g->w_stats.p, 0, 32 * 8, g->stream));
  int nl = 0;
  CK(cudaEventRecord(g->ev[0], g->stream));
  if (int r = stage_search(g, pts, p, part_lo, part_hi, q_lo, q_hi, cand_ids, cand_keys, &nl)) {
    g->pend_B = 0;
    return r;
  }
  CK(cudaEventRecord(g->ev[1], g->stream));
  return finish_stats(g, st, nl, 2, 0);
}

int graph_insert_stage_update(knng_graph *g, const knng_params *p, int32_t world, const int32_t *cand_ids_all,
                              const uint32_t *cand_keys_all, int64_t q_lo, int64_t q_hi, int32_t *props,
                              int32_t *prop_cnt, int32_t *new_ids, uint32_t *new_keys, knng_stats *st) {
  knng_err_slot().clear();
  if (!g || !p) return fail(KNNG_ERR_INVALID_ARG, "stage_update: null argument");
  if (world < 1 || q_lo < 0 || q_hi < q_lo || q_hi > g->pend_B) return fail(KNNG_ERR_INVALID_ARG, "stage_update: bad range");
  CK(cudaSetDevice(g->device));
  CK(cudaMemsetAsync(g->w_stats.p, 0, 32 * 8, g->stream));
  int nl = 0;
  CK(cudaEventRecord(g->ev[0], g->stream));
  if (int r = stage_update(g, p, world, cand_ids_all, cand_keys_all, q_lo, q_hi, (int2 *)props, prop_cnt, new_ids,
                           new_keys, &nl, false))
    return r;
  CK(cudaEventRecord(g->ev[1], g->stream));
  return finish_stats(g, st, nl, 2, 0);
}

int graph_insert_stage_commit(knng_graph *g, const knng_params *p, int64_t nq_slots, const int32_t *props_all,
                              const int32_t *prop_cnt_all, const int32_t *new_ids_all, const uint32_t *new_keys_all,
                              knng_stats *st) {
  knng_err_slot().clear();
  if (!g || !p) return fail(KNNG_ERR_INVALID_ARG, "stage_commit: null argument");
  if (nq_slots < g->pend_B) return fail(KNNG_ERR_INVALID_ARG, "stage_commit: fewer query slots than the batch");
  CK(cudaSetDevice(g->device));
  CK(cudaMemsetAsync(g->w_stats.p, 0, 32 * 8, g->stream));
  int nl = 0;
  CK(cudaEventRecord(g->ev[0], g->stream));
  if (int r = stage_commit(g, p, nq_slots, (const int2 *)props_all, prop_cnt_all, new_ids_all, new_keys_all, &nl))
    return r;
  CK(cudaEventRecord(g->ev[1], g->stream));
  return finish_stats(g, st, nl, 2, 0);
}

int graph_search(knng_graph *g, const knng_points *q, int32_t kr, const knng_params *p, int32_t *ids_out,
                 uint32_t *keys_out, int32_t out_on_device, knng_stats *st) {
  knng_err_slot().clear();
  if (!g) return fail(KNNG_ERR_INVALID_ARG, "graph_search: null graph");
  if (int r = check_points(q, "graph_search")) return r;
  if (int r = check_params(p)) return r;
  if (q->metric != g->metric || q->dim != g->dim) return fail(KNNG_ERR_INVALID_ARG, "graph_search: metric/dim mismatch");
  if (kr < 1 || kr > 32) return fail(KNNG_ERR_INVALID_ARG, "graph_search: kr=%d outside 1..32", kr);
  if (q->n > 0 && (!ids_out || !keys_out)) return fail(KNNG_ERR_INVALID_ARG, "graph_search: null outputs");
  CK(cudaSetDevice(g->device));
  CK(g->w_stats.ensure(32 * 8));
  const int64_t nq = q->n;
  if (nq == 0) {
    fill_stats(g, st, (const unsigned long long[8]){0, 0, 0, 0, 0, 0, 0, 0}, 0, 0);
    return KNNG_OK;
  }
  int nl = 0;
  CK(cudaMemsetAsync(g->w_stats.p, 0, 32 * 8, g->stream));
  StoreView qs = graph_store_view(g);
  if (csr_points(g->metric)) {
    CK(g->w_qoff.ensure((size_t)(nq + 1) * 8));
    uint32_t *qt = g->w_qtok.as<uint32_t>();
    int64_t qcap = (int64_t)(g->w_qtok.bytes / 4), ntok = 0;
    uint64_t *qo = g->w_qoff.as<uint64_t>();
    if (int r = append_sets(g, q, &qo, &qt, &qcap, 0, 0, &ntok)) return r;
    if (qt != g->w_qtok.p) {   // append_sets reallocated the token buffer (and freed the old one)
      g->w_qtok.p = qt;
      g->w_qtok.bytes = (size_t)qcap * 4;
    }
    qs.off = g->w_qoff.as<uint64_t>();
    qs.tok = g->w_qtok.as<uint32_t>();
    if (g->metric == KNNG_COSINE_2GRAM) {   // the queries' own |q|^2 (a query is never another row's entry, but
                                           // the evaluator's layout is the store's)
      CK(g->w_qn2.ensure((size_t)nq * 4));
      k_str_norms<<<(unsigned)((nq + 127) / 128), 128, 0, g->stream>>>(qs.off, qs.tok, 0, nq, g->w_qn2.as<uint32_t>());
      CK(cudaGetLastError());
      qs.n2 = g->w_qn2.as<uint32_t>();
    }
  } else {
    CK(g->w_query.ensure((size_t)nq * g->geom.stride));
    CK(cudaMemsetAsync(g->w_query.p, 0, (size_t)nq * g->geom.stride, g->stream));
    if (int r = copy_rows(g, g->w_query.as<uint8_t>(), q)) return r;
    qs.vec = g->w_query.as<uint8_t>();
  }
  const int32_t *d_starts = nullptr;
  int nstarts = 0;
  if (p->start_override && p->start_override_len > 0) {
    if (g->P > 0) return fail(KNNG_ERR_INVALID_ARG, "graph_search: start_override needs an unpartitioned graph");
    for (int i = 0; i < p->start_override_len; ++i)
      if (p->start_override[i] < 0 || p->start_override[i] >= g->n)
        return fail(KNNG_ERR_INVALID_ARG, "graph_search: start_override[%d] = %d is not a node", i, p->start_override[i]);
    nstarts = p->start_override_len;
    CK(g->w_starts.ensure((size_t)nstarts * 4));
    CK(cudaMemcpyAsync(g->w_starts.p, p->start_override, (size_t)nstarts * 4, cudaMemcpyHostToDevice, g->stream));
    d_starts = g->w_starts.as<int32_t>();
  }
  int32_t *oi = ids_out;
  uint32_t *ok = keys_out;
  if (!out_on_device) {
    CK(g->w_C_i.ensure((size_t)nq * kr * 4));
    CK(g->w_C_k.ensure((size_t)nq * kr * 4));
    oi = g->w_C_i.as<int32_t>();
    ok = g->w_C_k.as<uint32_t>();
  }
  CK(cudaEventRecord(g->ev[0], g->stream));
  if (g->P > 0 && !p->route) {
    CK(g->w_cand_i.ensure((size_t)nq * g->P * kr * 4));
    CK(g->w_cand_k.ensure((size_t)nq * g->P * kr * 4));
    if (int r = run_search_phase(g, qs, 0, nq, 0, kr, p, d_starts, nstarts, 0, g->P, g->w_cand_i.as<int32_t>(),
                                 g->w_cand_k.as<uint32_t>(), &nl))
      return r;
    CK(launch_merge_parts(g->metric, g->w_cand_i.as<int32_t>(), g->w_cand_k.as<uint32_t>(), nq, g->P, 1, kr, oi, ok,
                          g->stream));
    ++nl;
  } else {
    if (int r = run_search_phase(g, qs, 0, nq, 0, kr, p, d_starts, nstarts, 0, 1, oi, ok, &nl)) return r;
  }
  CK(cudaEventRecord(g->ev[1], g->stream));
  if (!out_on_device) {
    CK(cudaMemcpyAsync(ids_out, oi, (size_t)nq * kr * 4, cudaMemcpyDeviceToHost, g->stream));
    CK(cudaMemcpyAsync(keys_out, ok, (size_t)nq * kr * 4, cudaMemcpyDeviceToHost, g->stream));
  }
  unsigned long long h[32];
  CK(cudaMemcpyAsync(h, g->w_stats.p, 32 * 8, cudaMemcpyDeviceToHost, g->stream));
  CK(cudaStreamSynchronize(g->stream));
  print_profile(g, h, nq);
  h[4] = h[5] = h[6] = 0;
  fill_stats(g, st, h, nl, 2);
  return KNNG_OK;
}

int graph_get_rows(const knng_graph *g, int64_t first, int64_t count, int32_t *ids, uint32_t *keys) {
  knng_err_slot().clear();
  if (!g) return fail(KNNG_ERR_INVALID_ARG, "graph_get_rows: null graph");
  if (first < 0 || count < 0 || first + count > g->n) return fail(KNNG_ERR_INVALID_ARG, "graph_get_rows: bad range");
  CK(cudaSetDevice(g->device));
  if (ids) CK(cudaMemcpyAsync(ids, g->ids + first * g->k, (size_t)count * g->k * 4, cudaMemcpyDeviceToHost, g->stream));
  if (keys)
    CK(cudaMemcpyAsync(keys, g->keys + first * g->k, (size_t)count * g->k * 4, cudaMemcpyDeviceToHost, g->stream));
  CK(cudaStreamSynchronize(g->stream));
  return KNNG_OK;
}

int graph_get_partition(const knng_graph *g, uint8_t *part, int32_t *medoids, int32_t *P_out) {
  knng_err_slot().clear();
  if (!g) return fail(KNNG_ERR_INVALID_ARG, "graph_get_partition: null graph");
  if (P_out) *P_out = g->P;
  if (g->P == 0) return KNNG_OK;
  CK(cudaSetDevice(g->device));
  if (part) CK(cudaMemcpyAsync(part, g->part_of, (size_t)g->n, cudaMemcpyDeviceToHost, g->stream));
  if (medoids) memcpy(medoids, g->h_medoids.data(), sizeof(int32_t) * g->P);
  CK(cudaStreamSynchronize(g->stream));
  return KNNG_OK;
}

int partition_kmedoids(knng_graph *g, int32_t P, double imbalance, int32_t max_iter, uint64_t seed, uint8_t *part_out,
                       int32_t *medoids_out, int64_t *cost_out, const int32_t *init_medoids);

}  // extern "C"
