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
                 const int32_t *seed_ids, const uint32_t *seed_keys, int32_t *out_ids, uint32_t *out_keys) {
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
  // seeded rows (A5: C_i): columns beyond the seeds' k-th key cannot reach the merged row
  uint32_t seedk = 0xFFFFFFFFu;
  if (seed_ids && myrow < nrows && seed_ids[(size_t)myrow * k + k - 1] >= 0) seedk = seed_keys[(size_t)myrow * k + k - 1];

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
      const uint32_t tk = min(wk[KM - 1], seedk);
      const int thr = tk == 0xFFFFFFFFu ? 0x7FFFFFFF : (int)(tk - ni);
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
        const bool ins = mine && key < wk[KM - 1] && key < seedk && c != selfc;
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
                          int64_t ncols, int k, const uint32_t *nr, const uint32_t *ncn, const int32_t *sid,
                          const uint32_t *skey, int64_t ny, int32_t *pi, uint32_t *pk, cudaStream_t s) {
  const int NC = (nchunks + 1) & ~1;
  // operands + norms + barriers; >= 116 KB keeps one CTA per SM (its 512 TMEM columns)
  size_t smem = (size_t)tc::TM * NC * 16 + 2 * (size_t)tc::TN * NC * 16 + 3 * tc::TN * 4 + 64;
  if (smem < 116 * 1024) smem = 116 * 1024;
  cudaError_t e = cudaFuncSetAttribute(k_tc_topk_u8<KM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const dim3 grid((unsigned)((nrows + tc::TM - 1) / tc::TM), (unsigned)ny);
  k_tc_topk_u8<KM><<<grid, 256, smem, s>>>(vec, stride, nchunks, row0, nrows, col0, ncols, k, nr, ncn, sid, skey, pi, pk);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// fp32 rows (A0 / A5 for the F32 metric).  The exact key is the canonical fp32 sum of Q24, which a
// tensor core cannot reproduce; the tensor core screens instead.  3xTF32: x = hi + lo with hi =
// x with its 13 low mantissa bits cleared (exact in tf32) and lo = x - hi, and
//   <a, b> ~ hi_a.hi_b + hi_a.lo_b + lo_a.hi_b          (kind::tf32 MMAs, fp32 accumulation)
// whose error is below EPS * |a| |b| (dropped lo.lo term 2^-20, truncation of lo to tf32 2^-20 per
// cross term, fp32 accumulation of 3 x 96 products; EPS = 6.1e-5 is 2x the sum of these bounds at
// d <= 128).  A column survives the screen when its lower bound
//   |a|^2 + |b|^2 - 2 <a,b>~ - 2 EPS |a||b| - GUARD (|a|^2 + |b|^2)
// is below the row's exact k-th key; every survivor's key is then computed exactly in the canonical
// order (thread_dist) and inserted.  A column that fails the screen cannot enter, so the rows are
// bit-identical to the SIMT build's.
// ---------------------------------------------------------------------------------------------
namespace tc {
constexpr int TNF = 64;    // columns per tile (MMA N) for fp32
constexpr uint32_t IDESC_TF32 =
    (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(TNF >> 3) << 17) | ((uint32_t)(TM >> 4) << 24);
constexpr float EPS3 = 6.1e-5f, GUARD = 2.0e-5f;
__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(IDESC_TF32), "r"(accum));
}
__device__ __forceinline__ void split_tf32(const uint4 &x, uint4 &hi, uint4 &lo) {
  hi = make_uint4(x.x & 0xFFFFE000u, x.y & 0xFFFFE000u, x.z & 0xFFFFE000u, x.w & 0xFFFFE000u);
  lo = make_uint4(__float_as_uint(__fsub_rn(__uint_as_float(x.x), __uint_as_float(hi.x))),
                  __float_as_uint(__fsub_rn(__uint_as_float(x.y), __uint_as_float(hi.y))),
                  __float_as_uint(__fsub_rn(__uint_as_float(x.z), __uint_as_float(hi.z))),
                  __float_as_uint(__fsub_rn(__uint_as_float(x.w), __uint_as_float(hi.w))));
}
}  // namespace tc

__global__ void k_norms_f32(const uint8_t *vec, size_t stride, int nchunks, int64_t row0, int64_t n, float *norms,
                            float *roots) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint4 *r = (const uint4 *)(vec + (size_t)(row0 + i) * stride);
  float acc = 0.0f;
  for (int c = 0; c < nchunks; ++c) {
    const uint4 v = ldg16(r + c);
    acc = fmaf(__uint_as_float(v.x), __uint_as_float(v.x), acc);
    acc = fmaf(__uint_as_float(v.y), __uint_as_float(v.y), acc);
    acc = fmaf(__uint_as_float(v.z), __uint_as_float(v.z), acc);
    acc = fmaf(__uint_as_float(v.w), __uint_as_float(v.w), acc);
  }
  norms[i] = acc;
  roots[i] = sqrtf(acc);
}

// Same tiling and outputs as k_tc_topk_u8 with 64-column tiles: A (hi, lo) resident, B (hi, lo)
// double-buffered through registers (the split needs the values), two 64-column TMEM accumulators.
template <int KM>
__global__ void __launch_bounds__(256, 1)
    k_tc_topk_f32(const uint8_t *__restrict__ vec, size_t stride, int nchunks, int64_t row0, int64_t nrows,
                  int64_t col0, int64_t ncols, int k, const float *__restrict__ norms_r, const float *__restrict__ roots_r,
                  const float *__restrict__ norms_c, const float *__restrict__ roots_c, const int32_t *seed_ids,
                  const uint32_t *seed_keys, int32_t *out_ids, uint32_t *out_keys) {
  using namespace tc;
  constexpr int TN = TNF;
  extern __shared__ __align__(1024) uint8_t smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int NC = (nchunks + 1) & ~1;
  const uint32_t sboA = NC * 128, sboB = NC * 128;
  uint8_t *sAh = smem;                            // [TM/8][NC][8][16]
  uint8_t *sAl = sAh + TM * NC * 16;
  uint8_t *sB = sAl + TM * NC * 16;               // [2 buf][hi, lo][TN/8][NC][8][16]
  const uint32_t bpart = TN * NC * 16;            // one B operand (hi or lo) of one buffer
  float *sN = (float *)(sB + 4 * bpart);          // [3][TN] column norms (x (1 - GUARD)) and roots
  float *sR = sN + 3 * TN;
  uint64_t *bars = (uint64_t *)(sR + 3 * TN);
  uint32_t *tslot = (uint32_t *)(bars + 2);

  const int64_t per = ((ncols + gridDim.y - 1) / gridDim.y + TN - 1) / TN * TN;
  const int64_t c_lo = (int64_t)blockIdx.y * per;
  const int64_t c_hi = c_lo + per < ncols ? c_lo + per : ncols;
  const int64_t ntile = c_hi > c_lo ? (c_hi - c_lo + TN - 1) / TN : 0;
  const int64_t r0 = (int64_t)blockIdx.x * TM;

  if (warp == 0) {   // TMEM: two 128 x 64 fp32 accumulators
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(tslot)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = tid; i < TM * NC; i += 256) {      // A: rows split into hi / lo
    const int r = i / NC, c = i % NC;
    const uint32_t o = (r >> 3) * sboA + c * 128 + (r & 7) * 16;
    uint4 x = make_uint4(0, 0, 0, 0), hi, lo;
    if (r0 + r < nrows && c < nchunks) x = ldg16(vec + (size_t)(row0 + r0 + r) * stride + (size_t)c * 16);
    split_tf32(x, hi, lo);
    *(uint4 *)(sAh + o) = hi;
    *(uint4 *)(sAl + o) = lo;
  }
  // B tile loads: TN x NC chunks, at most 8 per thread (NC <= 32), staged in registers
  constexpr int BPT = (TN * 32 + 255) / 256;
  uint4 breg[BPT];
  auto load_regs = [&](int64_t t) {
    const int64_t cb = c_lo + t * TN;
#pragma unroll
    for (int j = 0; j < BPT; ++j) {
      const int i = tid + 256 * j;
      const int r = i / NC, c = i % NC;
      breg[j] = make_uint4(0, 0, 0, 0);
      if (i < TN * NC && cb + r < c_hi && c < nchunks)
        breg[j] = ldg16(vec + (size_t)(col0 + cb + r) * stride + (size_t)c * 16);
    }
  };
  auto store_b = [&](int64_t t, int buf) {
    const int64_t cb = c_lo + t * TN;
    uint8_t *bh = sB + (size_t)(2 * buf) * bpart, *bl = bh + bpart;
#pragma unroll
    for (int j = 0; j < BPT; ++j) {
      const int i = tid + 256 * j;
      if (i < TN * NC) {
        const int r = i / NC, c = i % NC;
        const uint32_t o = (r >> 3) * sboB + c * 128 + (r & 7) * 16;
        uint4 hi, lo;
        split_tf32(breg[j], hi, lo);
        *(uint4 *)(bh + o) = hi;
        *(uint4 *)(bl + o) = lo;
      }
    }
    for (int r = tid; r < TN; r += 256) {
      const bool ok = cb + r < c_hi;
      sN[(t % 3) * TN + r] = ok ? norms_c[cb + r] * (1.0f - GUARD) : __int_as_float(0x7F800000);
      sR[(t % 3) * TN + r] = ok ? roots_c[cb + r] : 0.0f;
    }
  };

  uint32_t wk[KM];   // exact keys (fp32 bits; non-negative, so integer order = float order)
  int32_t wi[KM];
#pragma unroll
  for (int t = 0; t < KM; ++t) { wk[t] = 0x7F800000u; wi[t] = 0x7FFFFFFF; }
  const int quarter = warp & 3, half = warp >> 2;
  const int64_t myrow = r0 + quarter * 32 + lane;
  const float nrow = myrow < nrows ? norms_r[myrow] : 0.0f;
  const float arow = myrow < nrows ? 2.0f * EPS3 * roots_r[myrow] : 0.0f;
  const int64_t mygid = row0 + myrow;
  const uint8_t *rowp = vec + (size_t)(myrow < nrows ? row0 + myrow : row0) * stride;
  // seeded rows (A5: C_i): no column beyond the seeds' k-th key can reach the merged row, and every
  // column id exceeds every seed id, so equal keys lose too
  uint32_t seedk = 0x7F800000u;
  if (seed_ids && myrow < nrows && seed_ids[(size_t)myrow * k + k - 1] >= 0) seedk = seed_keys[(size_t)myrow * k + k - 1];

  if (ntile > 0) { load_regs(0); store_b(0, 0); }
  fence_async_smem();
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tbase = *tslot;
  const uint32_t ah = smem_u32(sAh), al = smem_u32(sAl), b0 = smem_u32(sB);
  auto issue_mma = [&](int64_t t) {
    const int buf = (int)(t & 1);
    const uint32_t td = tbase + (uint32_t)(buf * TN);
    const uint32_t bh = b0 + 2 * buf * bpart, bl = bh + bpart;
    for (int kk = 0; kk < NC / 2; ++kk) {
      const uint64_t dah = smem_desc(ah + kk * 256, 128, sboA), dal = smem_desc(al + kk * 256, 128, sboA);
      const uint64_t dbh = smem_desc(bh + kk * 256, 128, sboB), dbl = smem_desc(bl + kk * 256, 128, sboB);
      mma_tf32(td, dah, dbh, kk > 0 ? 1u : 0u);
      mma_tf32(td, dah, dbl, 1u);
      mma_tf32(td, dal, dbh, 1u);
    }
    mma_commit(&bars[buf]);
  };
  if (ntile > 0 && tid == 0) issue_mma(0);
  if (ntile > 1) load_regs(1);

  for (int64_t t = 0; t < ntile; ++t) {
    const int buf = (int)(t & 1);
    mbar_wait(&bars[buf], (unsigned)((t >> 1) & 1));   // MMA t done: TMEM buf ready, B buf free
    fence_after();
    if (t + 1 < ntile) store_b(t + 1, buf ^ 1);         // B buf^1 was read by MMA t-1 (done)
    fence_async_smem();
    fence_before();
    __syncthreads();
    fence_after();
    if (t + 1 < ntile && tid == 0) issue_mma(t + 1);
    if (t + 2 < ntile) load_regs(t + 2);                // in flight during the epilogue
    // epilogue of tile t: this thread's row against its 32 columns
    const int64_t cbase = c_lo + t * TN + half * (TN / 2);
    const uint32_t taddr = tbase + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(buf * TN + half * (TN / 2));
    const float *nc = sN + (t % 3) * TN + half * (TN / 2);
    const float *rc = sR + (t % 3) * TN + half * (TN / 2);
    const int64_t selfc = mygid - (col0 + cbase);
    uint32_t v[32];
    tmem_ld32(taddr, v);
    // screen: lower bound of the key below the exact k-th key (its fp32 value; +inf while empty)
    const float rhs = __uint_as_float(min(wk[KM - 1], seedk)) - nrow * (1.0f - GUARD);
    uint32_t pm = 0;
#pragma unroll
    for (int e = 0; e < 32; ++e) {
      const float x = fmaf(-2.0f, __uint_as_float(v[e]), nc[e]);
      const float lb = fmaf(-arow, rc[e], x);
      pm |= (lb < rhs ? 1u : 0u) << e;
    }
    if (myrow >= nrows) pm = 0;
    while (pm) {                                   // exact keys of this lane's survivors
      const int e = __ffs(pm) - 1;
      pm &= pm - 1;
      if (e != selfc) {
        const int64_t gc = col0 + cbase + e;
        const uint32_t key = thread_dist<M_F32>((const uint4 *)rowp, (const uint4 *)(vec + (size_t)gc * stride), nchunks);
        if (key < wk[KM - 1] && key < seedk) {
          uint32_t ck = key;
          int32_t ci = (int32_t)gc;
#pragma unroll
          for (int s2 = 0; s2 < KM; ++s2) {
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
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tbase) : "memory");
}

template <int KM>
static cudaError_t run_tc_f32(const uint8_t *vec, size_t stride, int nchunks, int64_t row0, int64_t nrows,
                              int64_t col0, int64_t ncols, int k, const float *nr, const float *rr, const float *ncn,
                              const float *rcn, const int32_t *sid, const uint32_t *skey, int64_t ny, int32_t *pi,
                              uint32_t *pk, cudaStream_t s) {
  const int NC = (nchunks + 1) & ~1;
  size_t smem = 2 * (size_t)tc::TM * NC * 16 + 4 * (size_t)tc::TNF * NC * 16 + 6 * tc::TNF * 4 + 64;
  if (smem < 116 * 1024) smem = 116 * 1024;   // one CTA per SM
  cudaError_t e = cudaFuncSetAttribute(k_tc_topk_f32<KM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const dim3 grid((unsigned)((nrows + tc::TM - 1) / tc::TM), (unsigned)ny);
  k_tc_topk_f32<KM><<<grid, 256, smem, s>>>(vec, stride, nchunks, row0, nrows, col0, ncols, k, nr, rr, ncn, rcn, sid,
                                            skey, pi, pk);
  return cudaGetLastError();
}

// tcgen05 (3xTF32 screen + exact canonical rerank) form of launch_tile_topk for fp32 rows
// (nchunks <= 24, k <= 32): partial rows per column split and half into pi/pk ([2 ny][nrows][k]).
cudaError_t launch_tc_topk_f32(const VecGeom &g, const uint8_t *vec, int64_t row0, int64_t nrows, int64_t col0,
                               int64_t ncols, int k, const int32_t *sid, const uint32_t *skey, int64_t ny, int32_t *pi,
                               uint32_t *pk, Scratch *norm, cudaStream_t s) {
  if (g.metric != M_F32 || g.nchunks > 24 || k > 32) return cudaErrorNotSupported;
  if (cudaError_t e = norm->ensure((size_t)(nrows + ncols) * 8)) return e;
  float *nr = (float *)norm->p, *rr = nr + nrows, *ncn = rr + nrows, *rcn = ncn + ncols;
  k_norms_f32<<<(unsigned)((nrows + 255) / 256), 256, 0, s>>>(vec, g.stride, g.nchunks, row0, nrows, nr, rr);
  k_norms_f32<<<(unsigned)((ncols + 255) / 256), 256, 0, s>>>(vec, g.stride, g.nchunks, col0, ncols, ncn, rcn);
  if (k <= 10)
    return run_tc_f32<10>(vec, g.stride, g.nchunks, row0, nrows, col0, ncols, k, nr, rr, ncn, rcn, sid, skey, ny, pi, pk, s);
  if (k <= 20)
    return run_tc_f32<20>(vec, g.stride, g.nchunks, row0, nrows, col0, ncols, k, nr, rr, ncn, rcn, sid, skey, ny, pi, pk, s);
  return run_tc_f32<32>(vec, g.stride, g.nchunks, row0, nrows, col0, ncols, k, nr, rr, ncn, rcn, sid, skey, ny, pi, pk, s);
}

// tcgen05 form of launch_tile_topk for u8 rows (nchunks <= 16, k <= 32): partial rows per column
// split and half into pi/pk ([2 ny][nrows][k]).  Returns cudaErrorNotSupported when the shape is
// not covered.
cudaError_t launch_tc_topk_u8(const VecGeom &g, const uint8_t *vec, int64_t row0, int64_t nrows, int64_t col0,
                              int64_t ncols, int k, const int32_t *sid, const uint32_t *skey, int64_t ny, int32_t *pi,
                              uint32_t *pk, Scratch *norm, cudaStream_t s) {
  if (g.metric != M_U8 || g.nchunks > 16 || k > 32) return cudaErrorNotSupported;
  if (cudaError_t e = norm->ensure((size_t)(nrows + ncols) * 4)) return e;
  uint32_t *nr = (uint32_t *)norm->p, *ncn = nr + nrows;
  k_norms_u8<<<(unsigned)((nrows + 255) / 256), 256, 0, s>>>(vec, g.stride, g.nchunks, row0, nrows, nr);
  k_norms_u8<<<(unsigned)((ncols + 255) / 256), 256, 0, s>>>(vec, g.stride, g.nchunks, col0, ncols, ncn);
  if (k <= 10) return run_tc<10>(vec, g.stride, g.nchunks, row0, nrows, col0, ncols, k, nr, ncn, sid, skey, ny, pi, pk, s);
  if (k <= 16) return run_tc<16>(vec, g.stride, g.nchunks, row0, nrows, col0, ncols, k, nr, ncn, sid, skey, ny, pi, pk, s);
  return run_tc<32>(vec, g.stride, g.nchunks, row0, nrows, col0, ncols, k, nr, ncn, sid, skey, ny, pi, pk, s);
}

}  // namespace knng
