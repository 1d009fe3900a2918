// H2D of one 640x480 float depth image: DMA (cudaMemcpyAsync) vs a kernel
// reading mapped pinned host memory (GPU-initiated PCIe reads).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_pull(const float4* __restrict__ src, float4* __restrict__ dst, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) dst[i] = src[i];
}
int main() {
  const size_t bytes = 640 * 480 * 4;
  float *h, *d;
  cudaHostAlloc(&h, bytes, cudaHostAllocMapped);
  for (size_t i = 0; i < bytes / 4; ++i) h[i] = float(i);
  cudaMalloc(&d, bytes);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float* hd;
  cudaHostGetDevicePointer(&hd, h, 0);
  for (int grid : {0, 148, 296, 592, 1184}) {
    float best = 1e9;
    for (int r = 0; r < 20; ++r) {
      cudaStreamSynchronize(s);
      cudaEventRecord(a, s);
      if (grid == 0) cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s);
      else k_pull<<<grid, 256, 0, s>>>((const float4*)hd, (float4*)d, int(bytes / 16));
      cudaEventRecord(b, s);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    std::printf("%s grid %d: %.1f us (%.1f GB/s)\n", grid ? "pull kernel" : "memcpy", grid, best * 1e3,
                bytes / (best * 1e-3) / 1e9);
  }
  // first DMA from each of 24 freshly pinned buffers vs the same buffers again
  const int NB = 24;
  float* hb[NB];
  for (int i = 0; i < NB; ++i) {
    cudaHostAlloc(&hb[i], bytes, cudaHostAllocDefault);
    for (size_t j = 0; j < bytes / 4; ++j) hb[i][j] = float(j + i);
  }
  for (int pass = 0; pass < 2; ++pass) {
    float sum = 0, mx = 0;
    for (int i = 0; i < NB; ++i) {
      cudaStreamSynchronize(s);
      cudaEventRecord(a, s);
      cudaMemcpyAsync(d, hb[i], bytes, cudaMemcpyHostToDevice, s);
      cudaEventRecord(b, s);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      sum += ms;
      if (ms > mx) mx = ms;
    }
    std::printf("pass %d over %d fresh pinned buffers: mean %.1f us, max %.1f us\n", pass, NB, sum / NB * 1e3, mx * 1e3);
  }
  return 0;
}
