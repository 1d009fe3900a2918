// Throughput of a single claim counter: every warp's lane 0 claims items with
// atomicAdd on ONE global address until n items are taken (the k_lower_xr
// claim pattern), vs 8 counters (warp % 8) and CTA-local shared chunks.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_claim1(unsigned* ctr, unsigned n, unsigned* sink) {
  const int lane = threadIdx.x & 31;
  unsigned acc = 0;
  while (true) {
    unsigned i = 0;
    if (lane == 0) i = atomicAdd(ctr, 1u);
    i = __shfl_sync(0xffffffffu, i, 0);
    if (i >= n) break;
    acc += i;
  }
  if (acc == 0xdeadbeef) *sink = acc;
}
__global__ void k_claim8(unsigned* ctr, unsigned n, unsigned* sink) {
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  unsigned acc = 0;
  unsigned* c = ctr + 32 * (w & 7);
  while (true) {
    unsigned i = 0;
    if (lane == 0) i = atomicAdd(c, 1u);
    i = __shfl_sync(0xffffffffu, i, 0);
    if (i >= n / 8) break;
    acc += i;
  }
  if (acc == 0xdeadbeef) *sink = acc;
}
int main() {
  unsigned *ctr, *sink;
  cudaMalloc(&ctr, 4096);
  cudaMalloc(&sink, 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (unsigned n : {25000u, 100000u}) {
    for (int grid : {148, 296, 592}) {
      for (int v = 0; v < 2; ++v) {
        float best = 1e9;
        for (int r = 0; r < 5; ++r) {
          cudaMemset(ctr, 0, 4096);
          cudaEventRecord(a);
          if (v == 0) k_claim1<<<grid, 256>>>(ctr, n, sink);
          else k_claim8<<<grid, 256>>>(ctr, n, sink);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          best = ms < best ? ms : best;
        }
        printf("%s n=%u grid=%d: %.1f us (%.2f ns/claim)\n", v ? "8 counters" : "1 counter ", n, grid,
               best * 1e3, best * 1e6 / n);
      }
    }
  }
  return 0;
}
