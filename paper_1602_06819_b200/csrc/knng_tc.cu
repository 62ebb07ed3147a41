// knng_tc.cu -- the dense steps on the 5th-generation tensor cores (tcgen05, sm_100a):
// K7 exact initial graph (A0, "brute force") and K3 intra-batch all-pairs (A5) for uint8
// vectors under squared L2.
//
//   D(i, j) = |x_i|^2 + |x_j|^2 - 2 <x_i, x_j>
//
// <x_i, x_j> is an exact u8 x u8 -> s32 contraction (tcgen05.mma kind::i8, accumulator in TMEM);
// every term fits int32 (d <= 256: 256 * 255^2 < 2^24), so the key is bit-identical to the SIMT
// and oracle sums.  The epilogue turns each TMEM row into keys and keeps a per-row top-k in
// registers.
//
// CTA = 8 warps, one 128-row tile of the rows, the columns streamed in tiles of 256: each column
// tile is staged in shared memory by cp.async in the canonical K-major no-swizzle layout (8-row x
// 16-byte core matrices), multiplied by one elected thread (K/32 MMAs of 128x256x32) into one of two
// TMEM accumulators, and the MMA of tile j+1 runs while the epilogue reads tile j.  Epilogue: warp w
// reads TMEM lanes 32(w%4).. (tile rows) and column half w/4 of every tile, so each row has two
// partial top-k lists (column halves), merged with the other column splits afterwards.
#include <stdint.h>

#include "knng_common.cuh"
#include "knng_internal.h"

namespace knng {

namespace tc {

constexpr int TM = 128;   // rows per CTA (MMA M)
constexpr int TN = 256;   // columns per tile (MMA N)

__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  // SmemDescriptor (sm_100): start >> 4 [0,14), LBO >> 4 [16,30), SBO >> 4 [32,46), version 1 [46,48),
  // base offset 0, legacy LBO mode, layout SWIZZLE_NONE [61,64) = 0
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}

// instruction descriptor, kind::i8: D s32, A u8, B u8, both K-major, N >> 3, M >> 4
constexpr uint32_t IDESC = (2u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(TN >> 3) << 17) | ((uint32_t)(TM >> 4) << 24);

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(IDESC), "r"(accum));
}
__device__ __forceinline__ void mma_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// 32 consecutive TMEM columns of this thread's lane
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tmem_ld64(uint32_t taddr, uint32_t (&v)[64]) {
  uint32_t(&a)[32] = *reinterpret_cast<uint32_t(*)[32]>(&v[0]);
  uint32_t(&b)[32] = *reinterpret_cast<uint32_t(*)[32]>(&v[32]);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3]), "=r"(a[4]), "=r"(a[5]), "=r"(a[6]), "=r"(a[7]), "=r"(a[8]),
        "=r"(a[9]), "=r"(a[10]), "=r"(a[11]), "=r"(a[12]), "=r"(a[13]), "=r"(a[14]), "=r"(a[15]), "=r"(a[16]),
        "=r"(a[17]), "=r"(a[18]), "=r"(a[19]), "=r"(a[20]), "=r"(a[21]), "=r"(a[22]), "=r"(a[23]), "=r"(a[24]),
        "=r"(a[25]), "=r"(a[26]), "=r"(a[27]), "=r"(a[28]), "=r"(a[29]), "=r"(a[30]), "=r"(a[31])
      : "r"(taddr));
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(b[0]), "=r"(b[1]), "=r"(b[2]), "=r"(b[3]), "=r"(b[4]), "=r"(b[5]), "=r"(b[6]), "=r"(b[7]), "=r"(b[8]),
        "=r"(b[9]), "=r"(b[10]), "=r"(b[11]), "=r"(b[12]), "=r"(b[13]), "=r"(b[14]), "=r"(b[15]), "=r"(b[16]),
        "=r"(b[17]), "=r"(b[18]), "=r"(b[19]), "=r"(b[20]), "=r"(b[21]), "=r"(b[22]), "=r"(b[23]), "=r"(b[24]),
        "=r"(b[25]), "=r"(b[26]), "=r"(b[27]), "=r"(b[28]), "=r"(b[29]), "=r"(b[30]), "=r"(b[31])
      : "r"(taddr + 32));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// one TMEM column of this thread's lane
__device__ __forceinline__ uint32_t tmem_ld1(uint32_t taddr) {
  uint32_t v;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  return v;
}

}  // namespace tc

__global__ void k_norms_u8(const uint8_t *vec, size_t stride, int nchunks, int64_t row0, int64_t n, uint32_t *norms) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint4 *r = (const uint4 *)(vec + (size_t)(row0 + i) * stride);
  uint32_t acc = 0;
  for (int c = 0; c < nchunks; ++c) {
    const uint4 v = ldg16(r + c);
    acc = __dp4a(v.x, v.x, acc);
    acc = __dp4a(v.y, v.y, acc);
    acc = __dp4a(v.z, v.z, acc);
    acc = __dp4a(v.w, v.w, acc);
  }
  norms[i] = acc;
}

// Rows [row0, row0+nrows) x columns [col0, col0+ncols) of split blockIdx.y (column range
// [c_lo, c_hi) of gridDim.y splits); row-local top-KM (KM >= k entries kept, sorted by edge order;
// column ids ascend within a split, so a later column never precedes an equal key).
// norms_r / norms_c: |x|^2 of the rows / columns.  out: [2 * gridDim.y][nrows][k] (column half h of
// split y -> partial 2y + h).
template <int KM>
__global__ void __launch_bounds__(256, 1)
    k_tc_topk_u8(const uint8_t *__restrict__ vec, size_t stride, int nchunks, int64_t row0, int64_t nrows, int64_t col0,
                 int64_t ncols, int k, const uint32_t *__restrict__ norms_r, const uint32_t *__restrict__ norms_c,
                 int32_t *out_ids, uint32_t *out_keys) {
  using namespace tc;
  extern __shared__ __align__(1024) uint8_t smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int NC = (nchunks + 1) & ~1;              // 16-byte K chunks, even (K step of an MMA = 32 B)
  const uint32_t sboA = NC * 128;                 // next 8-row core-matrix group
  uint8_t *sA = smem;                             // [TM/8][NC][8][16]
  uint8_t *sB = sA + TM * NC * 16;                // [2][TN/8][NC][8][16]
  uint32_t *sN = (uint32_t *)(sB + 2 * TN * NC * 16);   // [3][TN] column norms (tile t -> t % 3)
  uint64_t *bars = (uint64_t *)(sN + 3 * TN);     // [2] MMA-done barriers
  uint32_t *tslot = (uint32_t *)(bars + 2);

  // column split
  const int64_t per = ((ncols + gridDim.y - 1) / gridDim.y + TN - 1) / TN * TN;
  const int64_t c_lo = (int64_t)blockIdx.y * per;
  const int64_t c_hi = c_lo + per < ncols ? c_lo + per : ncols;
  const int64_t ntile = c_hi > c_lo ? (c_hi - c_lo + TN - 1) / TN : 0;
  const int64_t r0 = (int64_t)blockIdx.x * TM;

  if (warp == 0) {   // TMEM: two 128 x 256 s32 accumulators
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tslot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // A tile (rows), zero beyond nrows / beyond nchunks
  for (int i = tid; i < TM * NC; i += 256) {
    const int r = i / NC, c = i % NC;
    uint8_t *dst = sA + (r >> 3) * sboA + c * 128 + (r & 7) * 16;
    if (r0 + r < nrows && c < nchunks) cp_async16(dst, vec + (size_t)(row0 + r0 + r) * stride + (size_t)c * 16);
    else *(uint4 *)dst = make_uint4(0, 0, 0, 0);
  }
  auto load_b = [&](int64_t t, int buf) {
    uint8_t *b = sB + (size_t)buf * TN * NC * 16;
    const int64_t cb = c_lo + t * TN;
    for (int i = tid; i < TN * NC; i += 256) {
      const int r = i / NC, c = i % NC;
      uint8_t *dst = b + (r >> 3) * (NC * 128) + c * 128 + (r & 7) * 16;
      if (cb + r < c_hi && c < nchunks) cp_async16(dst, vec + (size_t)(col0 + cb + r) * stride + (size_t)c * 16);
      else *(uint4 *)dst = make_uint4(0, 0, 0, 0);
    }
    // padded columns: a norm no key can beat (keys stay < 2^24 for d <= 256)
    for (int r = tid; r < TN; r += 256) sN[(t % 3) * TN + r] = cb + r < c_hi ? norms_c[cb + r] : 0x3FFFFFFFu;
  };
  if (ntile > 0) load_b(0, 0);
  cp_async_commit();

  // per-row top-KM (sorted; empty = (UINT32_MAX, INT32_MAX))
  uint32_t wk[KM];
  int32_t wi[KM];
#pragma unroll
  for (int t = 0; t < KM; ++t) { wk[t] = 0xFFFFFFFFu; wi[t] = 0x7FFFFFFF; }
  const int quarter = warp & 3, half = warp >> 2;
  const int64_t myrow = r0 + quarter * 32 + lane;
  const uint32_t ni = myrow < nrows ? norms_r[myrow] : 0u;
  const int64_t mygid = row0 + myrow;             // global id of this row (self is excluded)

  cp_async_wait<0>();
  fence_async_smem();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tbase = *tslot;
  const uint32_t aaddr = smem_u32(sA), baddr0 = smem_u32(sB);
  const uint32_t bstride = TN * NC * 16;
  auto issue_mma = [&](int64_t t) {
    const int buf = (int)(t & 1);
    const uint32_t td = tbase + (uint32_t)(buf * TN);
    const uint32_t bb = baddr0 + buf * bstride;
    for (int kk = 0; kk < NC / 2; ++kk)
      mma_i8(td, smem_desc(aaddr + kk * 256, 128, sboA), smem_desc(bb + kk * 256, 128, NC * 128), kk > 0 ? 1u : 0u);
    mma_commit(&bars[buf]);
  };
  if (ntile > 0 && tid == 0) issue_mma(0);
  if (ntile > 1) load_b(1, 1);
  cp_async_commit();

  for (int64_t t = 0; t < ntile; ++t) {
    const int buf = (int)(t & 1);
    mbar_wait(&bars[buf], (unsigned)((t >> 1) & 1));   // MMA t done: TMEM buf ready, smem B buf free
    fence_after();
    cp_async_wait<0>();                                 // B tile t+1 staged
    fence_async_smem();
    fence_before();
    __syncthreads();
    fence_after();
    if (t + 1 < ntile && tid == 0) issue_mma(t + 1);
    if (t + 2 < ntile) load_b(t + 2, buf);
    cp_async_commit();
    // epilogue of tile t: this thread's row against its 128 columns, 64 per TMEM load.
    // Screening key' = |x_c|^2 - 2 <x_r, x_c> against thr' = worst - |x_r|^2 (int32: both sides exact);
    // padded columns carry a huge norm, the row itself (key 0) is dropped on the rare insert path.
    const int64_t cbase = c_lo + t * TN + half * (TN / 2);
    const uint32_t taddr = tbase + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(buf * TN + half * (TN / 2));
    const int *nc = (const int *)sN + (t % 3) * TN + half * (TN / 2);
    const int64_t selfc = mygid - (col0 + cbase);     // column index of the row itself (if in range)
#pragma unroll 1
    for (int q = 0; q < TN / 128; ++q) {
      uint32_t v[64];
      tmem_ld64(taddr + q * 64, v);
      // screen: bit e of pm set when column e may enter the row's top-KM
      const int thr = wk[KM - 1] == 0xFFFFFFFFu ? 0x7FFFFFFF : (int)(wk[KM - 1] - ni);
      uint32_t pm0 = 0, pm1 = 0;
#pragma unroll
      for (int e4 = 0; e4 < 16; ++e4) {
        const int4 n4 = *(const int4 *)(nc + q * 64 + 4 * e4);
        const uint32_t b = ((n4.x - 2 * (int)v[4 * e4 + 0]) < thr ? 1u : 0u) |
                           ((n4.y - 2 * (int)v[4 * e4 + 1]) < thr ? 2u : 0u) |
                           ((n4.z - 2 * (int)v[4 * e4 + 2]) < thr ? 4u : 0u) |
                           ((n4.w - 2 * (int)v[4 * e4 + 3]) < thr ? 8u : 0u);
        if (e4 < 8) pm0 |= b << (4 * e4);
        else pm1 |= b << (4 * (e4 - 8));
      }
      if (myrow >= nrows) pm0 = pm1 = 0;
      // insert the survivors: warp-uniform walk over the columns any lane kept; each step re-reads
      // that column from TMEM (a warp-collective load) and inserts it in the lanes that kept it
      uint32_t w0 = __reduce_or_sync(FULL, pm0), w1 = __reduce_or_sync(FULL, pm1);
      while (w0 | w1) {
        int e;
        if (w0) { e = __ffs(w0) - 1; w0 &= w0 - 1; }
        else { e = 32 + __ffs(w1) - 1; w1 &= w1 - 1; }
        const uint32_t ve = tmem_ld1(taddr + q * 64 + e);
        const bool mine = ((e < 32 ? pm0 >> e : pm1 >> (e - 32)) & 1u) != 0;
        const int c = q * 64 + e;
        const uint32_t key = (uint32_t)(nc[c] - 2 * (int)ve) + ni;
        const bool ins = mine && key < wk[KM - 1] && c != selfc;
        uint32_t ck = ins ? key : 0xFFFFFFFFu;
        int32_t ci = ins ? (int32_t)(col0 + cbase + c) : 0x7FFFFFFF;
#pragma unroll
        for (int s2 = 0; s2 < KM; ++s2) {   // insertion by edge order (key, id); a no-op when !ins
          const bool sw = ck < wk[s2] || (ck == wk[s2] && ci < wi[s2]);
          const uint32_t tk = wk[s2];
          const int32_t ti = wi[s2];
          wk[s2] = sw ? ck : tk;
          wi[s2] = sw ? ci : ti;
          ck = sw ? tk : ck;
          ci = sw ? ti : ci;
        }
      }
    }
    fence_before();
  }
  if (myrow < nrows) {
    const size_t part = (size_t)blockIdx.y * 2 + half;
    int32_t *oi = out_ids + (part * nrows + myrow) * k;
    uint32_t *ok = out_keys + (part * nrows + myrow) * k;
#pragma unroll
    for (int s = 0; s < KM; ++s)
      if (s < k) {
        oi[s] = wi[s] == 0x7FFFFFFF ? -1 : wi[s];
        ok[s] = wi[s] == 0x7FFFFFFF ? 0u : wk[s];
      }
  }
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase) : "memory");
}

template <int KM>
static cudaError_t run_tc(const uint8_t *vec, size_t stride, int nchunks, int64_t row0, int64_t nrows, int64_t col0,
                          int64_t ncols, int k, const uint32_t *nr, const uint32_t *ncn, int64_t ny, int32_t *pi,
                          uint32_t *pk, cudaStream_t s) {
  const int NC = (nchunks + 1) & ~1;
  // operands + norms + barriers; >= 116 KB keeps one CTA per SM (its 512 TMEM columns)
  size_t smem = (size_t)tc::TM * NC * 16 + 2 * (size_t)tc::TN * NC * 16 + 3 * tc::TN * 4 + 64;
  if (smem < 116 * 1024) smem = 116 * 1024;
  cudaError_t e = cudaFuncSetAttribute(k_tc_topk_u8<KM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const dim3 grid((unsigned)((nrows + tc::TM - 1) / tc::TM), (unsigned)ny);
  k_tc_topk_u8<KM><<<grid, 256, smem, s>>>(vec, stride, nchunks, row0, nrows, col0, ncols, k, nr, ncn, pi, pk);
  return cudaGetLastError();
}

static uint32_t *g_norm_buf = nullptr;
static size_t g_norm_bytes = 0;

// tcgen05 form of launch_tile_topk for u8 rows (nchunks <= 16, k <= 32): partial rows per column
// split and half into pi/pk ([2 ny][nrows][k]).  Returns cudaErrorNotSupported when the shape is
// not covered.
cudaError_t launch_tc_topk_u8(const VecGeom &g, const uint8_t *vec, int64_t row0, int64_t nrows, int64_t col0,
                              int64_t ncols, int k, int64_t ny, int32_t *pi, uint32_t *pk, cudaStream_t s) {
  if (g.metric != M_U8 || g.nchunks > 16 || k > 32) return cudaErrorNotSupported;
  const size_t need = (size_t)(nrows + ncols) * 4;
  if (need > g_norm_bytes) {
    if (g_norm_buf) cudaFree(g_norm_buf);
    cudaError_t e = cudaMalloc((void **)&g_norm_buf, need);
    if (e != cudaSuccess) { g_norm_buf = nullptr; g_norm_bytes = 0; return e; }
    g_norm_bytes = need;
  }
  uint32_t *nr = g_norm_buf, *ncn = g_norm_buf + nrows;
  k_norms_u8<<<(unsigned)((nrows + 255) / 256), 256, 0, s>>>(vec, g.stride, g.nchunks, row0, nrows, nr);
  k_norms_u8<<<(unsigned)((ncols + 255) / 256), 256, 0, s>>>(vec, g.stride, g.nchunks, col0, ncols, ncn);
  if (k <= 10) return run_tc<10>(vec, g.stride, g.nchunks, row0, nrows, col0, ncols, k, nr, ncn, ny, pi, pk, s);
  if (k <= 16) return run_tc<16>(vec, g.stride, g.nchunks, row0, nrows, col0, ncols, k, nr, ncn, ny, pi, pk, s);
  return run_tc<32>(vec, g.stride, g.nchunks, row0, nrows, col0, ncols, k, nr, ncn, ny, pi, pk, s);
}

}  // namespace knng
