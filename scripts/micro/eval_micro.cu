// Microbenchmark (not product code): cost of evaluating chunks of 32 random u8 d=128 vectors per
// warp with the warp evaluator, as a function of warps per SM and lanes per vector.
#include <cstdio>
#include <cstdint>
#include "../../paper_1602_06819_b200/csrc/knng_common.cuh"
using namespace knng;

template <int L, int CPL>
__global__ void k_micro(StoreView st, int64_t n, int iters, uint32_t *out, long long *cyc) {
  const int lane = threadIdx.x & 31;
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  VecQuery<M_U8, L, CPL> Q;
  Q.load(st, gw % n, nullptr);
  uint32_t acc = 0;
  uint64_t h = rng_prefix(1, gw, 0);
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int32_t node = (int32_t)rng_index(h, (uint64_t)(it * 32 + lane), (uint64_t)n);
    acc += Q.eval(st, node, 32);
  }
  const long long t1 = clock64();
  out[gw * 32 + lane] = acc;
  if (lane == 0) cyc[gw] = t1 - t0;
}

int main() {
  const int64_t n = 100000;
  const int stride = 128;
  uint8_t *vec;
  cudaMalloc(&vec, n * stride);
  cudaMemset(vec, 7, n * stride);
  StoreView st{vec, (size_t)stride, 8, nullptr, nullptr};
  uint32_t *out;
  long long *cyc;
  cudaMalloc(&out, 148 * 64 * 32 * 4 * 4);
  cudaMalloc(&cyc, 148 * 64 * 8 * 4);
  const int iters = 400;
  for (int wps : {2, 4, 8, 16, 32, 48}) {
    for (int variant = 0; variant < 3; ++variant) {
      const int blocks = 148 * wps / 2;   // 2 warps per block
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0); cudaEventCreate(&e1);
      auto launch = [&]() {
        if (variant == 0) k_micro<8, 1><<<blocks, 64>>>(st, n, iters, out, cyc);
        if (variant == 1) k_micro<1, 8><<<blocks, 64>>>(st, n, iters, out, cyc);
        if (variant == 2) k_micro<4, 2><<<blocks, 64>>>(st, n, iters, out, cyc);
      };
      launch();
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      long long h[148 * 64];
      const int nw = blocks * 2;
      cudaMemcpy(h, cyc, nw * 8, cudaMemcpyDeviceToHost);
      double avg = 0;
      for (int i = 0; i < nw; ++i) avg += h[i];
      avg /= nw;
      const double chunks = (double)nw * iters;
      printf("warps/SM %2d  L=%d  kernel %.3f ms  cycles/chunk/warp %.0f  chunks/us %.0f  GB/s %.0f\n", wps,
             variant == 0 ? 8 : variant == 1 ? 1 : 4, ms, avg / iters, chunks / (ms * 1e3),
             chunks * 32 * 128 / (ms * 1e-3) / 1e9);
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
