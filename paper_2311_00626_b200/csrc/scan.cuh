// Device-wide ordered compaction primitives: block scan of (a, b) count pairs
// plus single-pass decoupled look-back across tiles taken in ticket order.
// Every list the hot path produces (candidates, changed blocks, effective
// blocks, ESDF changed set) is emitted in sorted order this way, without a
// sort: inputs are already key-ordered and compaction preserves order.
#pragma once

#include "common.cuh"

namespace vxm {

// Inclusive warp scan of two counters.
__device__ inline void warp_scan2(uint32_t& a, uint32_t& b) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t na = __shfl_up_sync(0xffffffffu, a, o);
    const uint32_t nb = __shfl_up_sync(0xffffffffu, b, o);
    if (lane >= o) {
      a += na;
      b += nb;
    }
  }
}

// Block-wide exclusive scan of (a, b); returns block totals. smem: 64 uint32.
// Must be called by all threads of the block (blockDim.x multiple of 32).
__device__ inline void block_scan2(uint32_t a, uint32_t b, uint32_t& ea, uint32_t& eb,
                                   uint32_t& ta, uint32_t& tb, uint32_t* smem) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  uint32_t ia = a, ib = b;
  warp_scan2(ia, ib);
  if (lane == 31) {
    smem[warp] = ia;
    smem[32 + warp] = ib;
  }
  __syncthreads();
  if (warp == 0) {
    uint32_t va = lane < nwarps ? smem[lane] : 0u;
    uint32_t vb = lane < nwarps ? smem[32 + lane] : 0u;
    warp_scan2(va, vb);
    smem[lane] = va;
    smem[32 + lane] = vb;
  }
  __syncthreads();
  const uint32_t wa = warp ? smem[warp - 1] : 0u, wb = warp ? smem[32 + warp - 1] : 0u;
  ea = wa + ia - a;
  eb = wb + ib - b;
  ta = smem[nwarps - 1];
  tb = smem[32 + nwarps - 1];
  __syncthreads();
}

// Clears the other status buffer for the next pass and resets its ticket.
__device__ inline void scan_prepare_next(const ScanTiles& st) {
  const uint32_t gtid = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t gsz = gridDim.x * blockDim.x;
  for (uint32_t i = gtid; i < st.n_next; i += gsz) st.next[i] = 0ull;
  if (gtid == 0) *st.next_ticket = 0u;
}

// Takes the next tile ticket (thread 0) and broadcasts it.
__device__ inline uint32_t scan_take_tile(const ScanTiles& st, uint32_t* s_tile) {
  if (threadIdx.x == 0) *s_tile = atomicAdd(st.ticket, 1u);
  __syncthreads();
  const uint32_t t = *s_tile;
  __syncthreads();
  return t;
}

// Warp 0 (all 32 lanes): publish this tile's aggregate, look back for the
// exclusive prefix 32 predecessors at a time, publish the inclusive prefix.
// Returns the exclusive prefix (a, b) in every lane.
__device__ inline void scan_lookback(const ScanTiles& st, uint32_t tile, uint32_t agg_a,
                                     uint32_t agg_b, uint32_t& ex_a, uint32_t& ex_b) {
  const int lane = threadIdx.x & 31;
  volatile unsigned long long* status = st.status;
  if (tile == 0) {
    if (lane == 0) atomicExch(st.status, kFlagPre | pack_ab(agg_a, agg_b));
    ex_a = ex_b = 0;
    return;
  }
  if (lane == 0) atomicExch(st.status + tile, kFlagAgg | pack_ab(agg_a, agg_b));
  uint32_t a = 0, b = 0;
  int64_t base = int64_t(tile) - 1;
  while (true) {
    const int64_t j = base - lane;
    // tile 0 always publishes an inclusive prefix, so j >= 0 for every lane
    // that can matter; lanes beyond it read a zero prefix
    const unsigned long long v = j >= 0 ? status[j] : (2ull << 62);  // kFlagPre
    const unsigned long long f = v & (3ull << 62);
    const uint32_t pre = __ballot_sync(0xffffffffu, f == kFlagPre);
    const uint32_t zero = __ballot_sync(0xffffffffu, f == 0ull);
    const int first = pre ? __ffs(pre) - 1 : 32;  // nearest inclusive prefix
    const uint32_t need = first >= 31 ? 0xffffffffu : ((2u << first) - 1u);
    if (zero & need) continue;  // a predecessor has not published yet
    const bool use = (need >> lane) & 1u;
    a += __reduce_add_sync(0xffffffffu, use ? unpack_a(v) : 0u);
    b += __reduce_add_sync(0xffffffffu, use ? unpack_b(v) : 0u);
    if (first < 32) break;
    base -= 32;
  }
  if (lane == 0) atomicExch(st.status + tile, kFlagPre | pack_ab(a + agg_a, b + agg_b));
  ex_a = a;
  ex_b = b;
}

}  // namespace vxm
