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


namespace vxm {
// Experimental: one warp per block, two lines per lane (lines q and q + 32).
template <int AXIS>
__device__ inline uint32_t sweep_line_fast2(GroupSmem& g, int q0) {
  constexpr int sh = AXIS == 0 ? 20 : (AXIS == 1 ? 10 : 0);
  constexpr uint32_t sb = 1u << sh;
  uint32_t th[2][8], tl[2][8], qm[2][8], ko[2][8];
  int po[2][8], idx[2][8];
#pragma unroll
  for (int L = 0; L < 2; ++L)
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      idx[L][k] = line_idx3<AXIS>(q0 + 32 * L, k);
      th[L][k] = g.a[0][idx[L][k]];
      tl[L][k] = g.a[1][idx[L][k]];
      const uint32_t key = g.a[2][idx[L][k]];
      const int pa = int((key >> sh) & 1023u) - int(kFastBias);
      qm[L][k] = g.a[3][idx[L][k]] - uint32_t(pa * pa);
      po[L][k] = pa - 1;
      ko[L][k] = key - sb;
    }
  uint32_t ch[2] = {0, 0};
#pragma unroll
  for (int k = 1; k < 8; ++k)
#pragma unroll
    for (int L = 0; L < 2; ++L) {
      const int j = k - 1;
      const uint32_t cm = uint32_t(po[L][j] * po[L][j]) + qm[L][j];
      const unsigned long long cv = (unsigned long long)cm << 32 | ko[L][j];
      const unsigned long long tv = (unsigned long long)th[L][k] << 32 | tl[L][k];
      if (cv < tv) {
        th[L][k] = cm; tl[L][k] = ko[L][j]; qm[L][k] = qm[L][j];
        po[L][k] = po[L][j] - 1; ko[L][k] = ko[L][j] - sb; ch[L] |= 1u << k;
      }
    }
#pragma unroll
  for (int L = 0; L < 2; ++L)
#pragma unroll
    for (int k = 0; k < 8; ++k) { po[L][k] += 2; ko[L][k] += 2u * sb; }
#pragma unroll
  for (int k = 6; k >= 0; --k)
#pragma unroll
    for (int L = 0; L < 2; ++L) {
      const int j = k + 1;
      const uint32_t cm = uint32_t(po[L][j] * po[L][j]) + qm[L][j];
      const unsigned long long cv = (unsigned long long)cm << 32 | ko[L][j];
      const unsigned long long tv = (unsigned long long)th[L][k] << 32 | tl[L][k];
      if (cv < tv) {
        th[L][k] = cm; tl[L][k] = ko[L][j]; qm[L][k] = qm[L][j];
        po[L][k] = po[L][j] + 1; ko[L][k] = ko[L][j] + sb; ch[L] |= 1u << k;
      }
    }
#pragma unroll
  for (int L = 0; L < 2; ++L)
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (ch[L] & (1u << k)) {
        g.a[0][idx[L][k]] = th[L][k]; g.a[1][idx[L][k]] = tl[L][k];
        g.a[2][idx[L][k]] = tl[L][k]; g.a[3][idx[L][k]] = th[L][k];
      }
  return ch[0] | (ch[1] << 8);
}

__global__ void k_sweep_micro2(const uint32_t* src, Limits lim, long long* clk, int reps) {
  __shared__ GroupSmem G;
  const int t = threadIdx.x;
  RawBlock rb;
  bool any_site, fast;
  load_raw3(rb, src, t, 1, lim, false, &any_site, &fast);
  stage_block3(G, rb, t, 1, lim, fast);
  if (t >= 32) return;
  long long acc[4] = {0, 0, 0, 0};
  for (int r = 0; r < reps; ++r) {
    __syncwarp();
    long long c0 = clock64();
    uint32_t c = sweep_line_fast2<0>(G, t);
    __syncwarp();
    long long c1 = clock64();
    c |= sweep_line_fast2<1>(G, t);
    __syncwarp();
    long long c2 = clock64();
    c |= sweep_line_fast2<2>(G, t);
    const bool any = __any_sync(0xffffffffu, c != 0);
    long long c3 = clock64();
    if (any && t == 99) clk[0] = 1;
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
  cudaMalloc(&dc, 4 * 2368 * sizeof(long long));
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
  for (int grid : {1, 148, 1184, 2368}) {
    k_sweep_micro2<<<grid, 64>>>(d, lim, dc, 200);
    cudaDeviceSynchronize();
    std::vector<long long> c(4 * grid);
    cudaMemcpy(c.data(), dc, c.size() * 8, cudaMemcpyDeviceToHost);
    double m[4] = {0, 0, 0, 0};
    for (int b = 0; b < grid; ++b)
      for (int i = 0; i < 4; ++i) m[i] += double(c[4 * b + i]) / grid;
    std::printf("2-line warp, grid %4d: cycles/pass %.0f (X %.0f, Y %.0f, Z+any %.0f)  %s\n", grid, m[3], m[0], m[1],
                m[2], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
