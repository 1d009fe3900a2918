// Micro-benchmark: cycles per sweep pass / phase of the ESDF block sweep in
// isolation (one 64-thread group per CTA).  Build: make -C tools/micro
#include "esdf.cu"
#ifndef NOMASK
#define NOMASK 0
#endif
#include <cstdio>
#include <vector>
namespace vxm {
__global__ void k_sweep_micro(const uint32_t* src, Limits lim, long long* clk, int reps) {
  __shared__ GroupSmem G;
  const int t = threadIdx.x;
  RawBlock rb;
  bool any_site, fast;
  load_raw3(rb, src, t, 1, lim, false, &any_site, &fast);
  stage_block3(G, rb, t, 1, lim, fast);
  long long acc[4] = {0, 0, 0, 0};
  for (int r = 0; r < reps; ++r) {
    if (t == 0) {
      G.mask[0][0] = G.mask[1][0] = G.mask[2][0] = ~0ull;
      G.mask[0][1] = G.mask[1][1] = G.mask[2][1] = 0;
    }
    group_sync(1);
    long long c0 = clock64();
    uint32_t c = NOMASK ? sweep_line_fast<0>(G, t) : sweep_phase3<0>(G, t, 1, 0, lim);
    group_sync(1);
    long long c1 = clock64();
    c |= NOMASK ? sweep_line_fast<1>(G, t) : sweep_phase3<1>(G, t, 1, 0, lim);
    group_sync(1);
    long long c2 = clock64();
    c |= NOMASK ? sweep_line_fast<2>(G, t) : sweep_phase3<2>(G, t, 1, 0, lim);
    group_sync_or(1, c != 0);
    long long c3 = clock64();
    acc[0] += c1 - c0; acc[1] += c2 - c1; acc[2] += c3 - c2; acc[3] += c3 - c0;
  }
  if (t == 0)
    for (int i = 0; i < 4; ++i) clk[4 * blockIdx.x + i] = acc[i] / reps;
}
}  // namespace vxm

int main() {
  using namespace vxm;
  // block: observed everywhere, one site at the centre, the rest saturated
  std::vector<uint32_t> h(1536);
  for (int lin = 0; lin < 512; ++lin) {
    const bool site = lin == 4 + 8 * 4 + 64 * 4;
    h[3 * lin] = site ? 0 : 10000;
    h[3 * lin + 1] = 0;
    h[3 * lin + 2] = uint32_t(VXM_ESDF_OBSERVED | (site ? VXM_ESDF_SITE : 0)) << 16;
  }
  uint32_t* d;
  long long* dc;
  cudaMalloc(&d, 1536 * 4);
  cudaMalloc(&dc, 4 * 1184 * sizeof(long long));
  cudaMemcpy(d, h.data(), 1536 * 4, cudaMemcpyHostToDevice);
  Limits lim{10000, 16};
  for (int grid : {1, 148, 592, 1184}) {
    k_sweep_micro<<<grid, 64>>>(d, lim, dc, 200);
    cudaDeviceSynchronize();
    std::vector<long long> c(4 * grid);
    cudaMemcpy(c.data(), dc, c.size() * 8, cudaMemcpyDeviceToHost);
    double m[4] = {0, 0, 0, 0};
    for (int b = 0; b < grid; ++b)
      for (int i = 0; i < 4; ++i) m[i] += double(c[4 * b + i]) / grid;
    std::printf("grid %4d: cycles/pass %.0f (X %.0f, Y %.0f, Z+or %.0f)  %s\n", grid, m[3], m[0], m[1],
                m[2], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
