// Random-row gather bandwidth of the B200's HBM (measurement for the K1 roofline discussion):
// every thread reads R-byte rows at pseudo-random row indices of a buffer much larger than L2, with
// 16-byte vector loads, and folds them into a checksum.  Prints GB/s per row size.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a gather_bw.cu -o gather_bw
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

template <int R>
__global__ void gather(const uint4 *__restrict__ buf, uint64_t nrows, int per_thread, unsigned *out) {
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned acc = 0;
  for (int i = 0; i < per_thread; ++i) {
    const uint64_t r = __umul64hi(mix(t * 1000003ull + i), nrows);
    const uint4 *p = buf + r * (R / 16);
    uint4 v[R / 16];
#pragma unroll
    for (int c = 0; c < R / 16; ++c) v[c] = __ldg(p + c);
#pragma unroll
    for (int c = 0; c < R / 16; ++c) acc += v[c].x ^ v[c].y ^ v[c].z ^ v[c].w;
  }
  if (acc == 0x12345678u) out[0] = acc;
}

// warp-cooperative: R/16 lanes per row, each lane one 16-byte chunk (rows read as contiguous segments)
template <int R>
__global__ void gather_coop(const uint4 *__restrict__ buf, uint64_t nrows, int per_thread, unsigned *out) {
  constexpr int LPR = R / 16 < 32 ? R / 16 : 32, RPW = 32 / LPR, CPL = R / 16 / LPR;
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  unsigned acc = 0;
  for (int i = 0; i < per_thread; ++i) {
    const uint64_t r = __umul64hi(mix((t / LPR) * 1000003ull + i), nrows);
    const uint4 *p = buf + r * (R / 16) + (lane % LPR);
    uint4 v[CPL];
#pragma unroll
    for (int c = 0; c < CPL; ++c) v[c] = __ldg(p + c * LPR);
#pragma unroll
    for (int c = 0; c < CPL; ++c) acc += v[c].x ^ v[c].y ^ v[c].z ^ v[c].w;
  }
  (void)RPW;
  if (acc == 0x12345678u) out[0] = acc;
}

template <int R>
void run_coop(const uint4 *buf, size_t bytes, unsigned *out, int blocks, int threads) {
  const uint64_t nrows = bytes / R;
  const int per = 64;
  constexpr int LPR = R / 16 < 32 ? R / 16 : 32;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  gather_coop<R><<<blocks, threads>>>(buf, nrows, per, out);
  cudaEventRecord(a);
  for (int it = 0; it < 5; ++it) gather_coop<R><<<blocks, threads>>>(buf, nrows, per, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double moved = 5.0 * blocks * threads / LPR * per * R;
  printf("coop rows of %4d B, %6d blocks x %4d threads: %8.1f GB/s\n", R, blocks, threads, moved / (ms / 1e3) / 1e9);
}

template <int R>
void run(const uint4 *buf, size_t bytes, unsigned *out, int blocks, int threads) {
  const uint64_t nrows = bytes / R;
  const int per = 64;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  gather<R><<<blocks, threads>>>(buf, nrows, per, out);
  cudaEventRecord(a);
  for (int it = 0; it < 5; ++it) gather<R><<<blocks, threads>>>(buf, nrows, per, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double moved = 5.0 * blocks * threads * per * R;
  printf("rows of %4d B, %6d blocks x %4d threads: %8.1f GB/s\n", R, blocks, threads, moved / (ms / 1e3) / 1e9);
}

int main() {
  const size_t bytes = (size_t)4 << 30;
  uint4 *buf;
  unsigned *out;
  cudaMalloc(&buf, bytes);
  cudaMalloc(&out, 4);
  cudaMemset(buf, 1, bytes);
  for (int blocks : {148 * 4, 148 * 16, 148 * 64}) {
    run<32>(buf, bytes, out, blocks, 256);
    run<64>(buf, bytes, out, blocks, 256);
    run<128>(buf, bytes, out, blocks, 256);
    run<384>(buf, bytes, out, blocks, 256);
    run_coop<64>(buf, bytes, out, blocks, 256);
    run_coop<128>(buf, bytes, out, blocks, 256);
    run_coop<384>(buf, bytes, out, blocks, 256);
  }
  return 0;
}
