// ESDF update.
//
// Reference: proj/src/esdf/integrator.cpp — relax (:58-88), sweep_block
// (:96-139), exchange_pair (:144-168), TsdfClassifier (:177-198), mark_impl
// (:268-348), reset_parented (:352-363), update_impl (:365-413),
// clear_invalid (:433-486), lower_esdf (:488-565).
//
// The reference's update is a full-map recompute whenever any site/side
// changed: reset every parented voxel to saturation, then lower from ALL
// blocks with its exact sweep/border schedule.  This file reproduces that
// schedule bit-for-bit on the GPU:
//   * mark: CTA per effective block (updated + allocated face neighbours).
//     The effective set is a 7-way rank merge of the sorted updated list and
//     its six axis-shifted copies (each shift preserves order), so it is
//     produced sorted without a sort.
//   * allocation: look-up + ordered slot assignment + hash insert in one
//     look-back pass; the sorted set of all ESDF blocks is maintained by a
//     rank merge (no sort); a 6-neighbour slot table serves the border phase.
//   * lowering: ONE cooperative persistent kernel runs every round.  Sweeps:
//     a 64-thread group per dirty block holds the block in shared memory
//     (bank-conflict-free swizzled SoA), each thread owns one line per
//     direction and runs the Gauss-Seidel X+/X- (Y, Z) passes in registers
//     until the block's fixed point.  Borders: a warp per (dirty block, side)
//     relaxes the 64 face pairs of each axis in turn (x, then y, then z), with
//     grid-wide barriers between phases exactly where the reference has them.
//     Round 1 reads the pre-update field and writes the other buffer (fused
//     reset_parented + snapshot), so the changed set is a block compare of the
//     two buffers — no O(map) snapshot copy.
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>

#include "runtime.cuh"
#include "scan.cuh"

namespace cg = cooperative_groups;

namespace vxm {

void launch_compact_keys(Context* ctx, const uint64_t* in, const uint8_t* flags,
                         const uint32_t* n_ptr, uint32_t n_cap, uint64_t* out, uint32_t* n_out,
                         const DevStatus* guard, const char* prof_name = "k_compact");

}  // namespace vxm

#include "esdf_lower.cuh"
#include "esdf_host.cuh"

namespace vxm {

__global__ void __launch_bounds__(kL3Threads, 2) k_lower3(LowerArgs a) {
  cg::grid_group grid = cg::this_grid();
  uint32_t tr = 0;
  auto stamp = [&]() {
    if (a.trace && blockIdx.x == 0 && threadIdx.x == 0 && tr < 127) {
      unsigned long long tm;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tm));
      a.trace[1 + tr++] = tm;
      a.trace[0] = tr;
    }
  };
  stamp();
  __shared__ GroupSmem s_grp[kL3Groups];
  const int g = threadIdx.x >> 6, t = threadIdx.x & 63, lane = threadIdx.x & 31;
  const int bar = 1 + g;
  GroupSmem& G = s_grp[g];
  const int wid = (blockIdx.x * kL3Threads + threadIdx.x) >> 5;
  const int nwarps = gridDim.x * (kL3Threads >> 5);
  const uint32_t n_blocks = a.meta->num_blocks;
  const uint32_t cur = a.meta->cur;
  const uint32_t base_epoch = a.meta->round_epoch;
  const bool failed = a.status->capacity_error || a.status->pool_overflow;
  const bool lower = !failed && (a.full ? a.status->any_update != 0 : true);
  uint32_t* const pcur = a.pool[cur];
  uint32_t* const pnxt = a.pool[cur ^ 1u];
  uint32_t* const work = a.full ? pnxt : pcur;
  const Limits lim = a.lim;
  if (!a.full && lower) {  // seeded mode: round-1 dirty list = seeds
    const uint32_t ns = *a.n_seeds;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < ns; i += gridDim.x * blockDim.x) {
      const int32_t s = a.seeds[i];
      a.list[1][i] = s;
      a.stamp_dirty[1][s] = base_epoch + 1;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) a.count[1] = ns;
  }
  // Dirty-list counts are triple-buffered by round (read r%3, append (r+1)%3,
  // reset (r+2)%3) because pair items of round r append while other CTAs may
  // still be starting round r; lists are double-buffered by parity.
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.count[2] = 0u;
    a.work_ctr[0] = a.work_ctr[1] = a.work_ctr[2] = a.work_ctr[3] = 0u;
  }
  // Round 1 of a full update splits the map: blocks that may hold sites go to
  // the 64-thread sweep groups (front of list[1]); site-free blocks are only
  // reset and copied, one warp each (back of list[1]).  Order is irrelevant:
  // round-1 sweeps are independent.  (a.r1 is zero on entry.)
  if (a.full && lower) {
    for (uint32_t b0 = blockIdx.x * kL3Threads + (threadIdx.x & ~31u); b0 < n_blocks;
         b0 += gridDim.x * kL3Threads) {
      const uint32_t b = b0 + lane;
      const bool in = b < n_blocks;
      const bool site = in && a.site_any[b] != 0;
      const uint32_t ms = __ballot_sync(0xffffffffu, site), mn = __ballot_sync(0xffffffffu, in && !site);
      uint32_t bs = 0, bn = 0;
      if (lane == 0) {
        if (ms) bs = atomicAdd(a.r1 + 0, __popc(ms));
        if (mn) bn = atomicAdd(a.r1 + 1, __popc(mn));
      }
      bs = __shfl_sync(0xffffffffu, bs, 0);
      bn = __shfl_sync(0xffffffffu, bn, 0);
      const uint32_t below = (1u << lane) - 1u;
      if (site) a.list[1][bs + __popc(ms & below)] = int32_t(b);
      else if (in) a.list[1][n_blocks - 1u - (bn + __popc(mn & below))] = int32_t(b);
    }
  }
  grid.sync();
  stamp();
  uint32_t r = 0;
  uint32_t n_pairs = 0, n_cmp = 0;
  const uint32_t n_first = a.full ? n_blocks : *((volatile uint32_t*)&a.count[1]);
  if (lower && n_first > 0) {  // while (!dirty.empty()) — esdf/integrator.cpp:506
    while (true) {
      ++r;
      const int cp = int(r & 1u), np = cp ^ 1;
      const uint32_t ep = base_epoch + r, ep_next = ep + 1;
      const bool r1_full = a.full && r == 1;
      if (a.trace && blockIdx.x == 0 && threadIdx.x == 0 && r < 16) {
        unsigned long long tm;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tm));
        a.trace[256 + 4 * r + 3] = tm;  // round start (block 0)
      }
      const uint32_t n_dirty = r1_full ? n_blocks : *((volatile uint32_t*)&a.count[r % 3u]);
      const int32_t* dirty = a.list[cp];
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        a.count[(r + 2u) % 3u] = 0;  // read in round r - 1, appended in round r + 1
        a.work_ctr[np] = 0u;      // counters of the previous round (finished at the
        a.work_ctr[2 + np] = 0u;  // last grid barrier) serve the next round
        if (r > 1 || !a.full) a.status->sum_dirty += n_dirty;
      }
      // ---- sweep phase (esdf/integrator.cpp:509-513)
      uint32_t* const ctr = r1_full ? a.r1 + 2 : a.work_ctr + cp;
      const uint32_t n_grp = r1_full ? *((volatile uint32_t*)(a.r1 + 0)) : n_dirty;
      while (true) {
        if (t == 0) G.bcast = atomicAdd(ctr, 1u);
        group_sync(bar);
        const uint32_t i = G.bcast;
        if (i >= n_grp) break;
        const int32_t s = __ldcg((r1_full ? a.list[1] : dirty) + i);
        unsigned long long tt0 = 0, tt1 = 0, tt2 = 0;
        if (a.trace && t == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt0));
        if (t == 0) {
          unsigned long long m0 = ~0ull, m1 = ~0ull, m2 = ~0ull;
          if (a.full && !r1_full) {  // lines through voxels changed by the last borders
            m0 = atomicExch(a.line_mask + 3 * size_t(s), 0ull);
            m1 = atomicExch(a.line_mask + 3 * size_t(s) + 1, 0ull);
            m2 = atomicExch(a.line_mask + 3 * size_t(s) + 2, 0ull);
          }
          G.mask[0][0] = m0;
          G.mask[1][0] = m1;
          G.mask[2][0] = m2;
          G.mask[0][1] = G.mask[1][1] = G.mask[2][1] = 0ull;
        }
        // (the mask writes are ordered by the barriers below)
        RawBlock rb;
        bool any_site, fast;
        load_raw3(rb, (r1_full ? pcur : work) + size_t(s) * 1536, t, bar, lim, r1_full, &any_site, &fast);
        bool changed = false;
        int passes = 0;
        if (!any_site) {  // round 1, no site: the reset block is already at its fixed point
          raw_store(rb, work + size_t(s) * 1536, t);
          if (a.trace && t == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt1));
          tt2 = tt1;
        } else {
          stage_block3(G, rb, t, bar, lim, fast);
          if (a.trace && t == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt1));
          changed = sweep_block3(G, t, bar, lim, &passes);
          if (a.trace && t == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt2));
          if (r1_full || changed) store_block3(G, work + size_t(s) * 1536, t);
        }
        if (changed && !a.full && t == 0) a.stamp_lchg[s] = a.lchg_tag;
        group_sync(bar);  // the group's stores before the release of its sweep stamp
        if (t == 0) st_release(a.stamp_swept + s, ep);
        if (a.trace && t == 0 && r < 16) {  // debug: per-block cost breakdown per round
          unsigned long long tt3;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt3));
          atomicMax(a.trace + 256 + 4 * r, tt3);  // last sweep end
          unsigned long long* d = a.trace + 128 + 8 * r;
          atomicAdd(d + 0, 1ull);                      // blocks
          atomicAdd(d + 1, tt1 - tt0);                 // load
          atomicAdd(d + 2, tt2 - tt1);                 // sweep
          atomicAdd(d + 3, tt3 - tt2);                 // store
          atomicMax(d + 4, tt3 - tt0);                 // max block total
          atomicMax(d + 5, tt2 - tt1);                 // max sweep
          atomicAdd(d + 6, (unsigned long long)passes);  // passes
          atomicMax(d + 7, (unsigned long long)passes);  // max passes
        }
      }
      if (r1_full) {  // site-free blocks: reset + copy, one warp each
        const uint32_t n_ns = *((volatile uint32_t*)(a.r1 + 1));
        constexpr uint32_t kCopyChunk = 2;
        uint32_t j = 0, j_end = 0;
        while (true) {
          if (j == j_end) {
            if (lane == 0) j = atomicAdd(a.r1 + 3, kCopyChunk);
            j = __shfl_sync(0xffffffffu, j, 0);
            j_end = j + kCopyChunk;
          }
          if (j >= n_ns) break;
          const int32_t s = __ldcg(a.list[1] + (n_blocks - 1u - j));
          ++j;
          warp_reset_copy(pcur + size_t(s) * 1536, work + size_t(s) * 1536, lane, lim);
          __syncwarp();  // the warp's stores before the release of the sweep stamp
          if (lane == 0) st_release(a.stamp_swept + s, ep);
          if (a.trace && lane == 0 && r < 16) {
            unsigned long long tm;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tm));
            atomicMax(a.trace + 256 + 4 * r + 2, tm);  // last copy end
          }
        }
      }
      // ---- border phase (esdf/integrator.cpp:517-559) as a dataflow: pair items
      // are taken in axis order (all x, then y, then z) after every sweep was
      // taken, and each waits only for what the reference's phase order makes
      // it depend on: the sweeps of its two blocks, and for y (z) the x (x, y)
      // pairs touching its two blocks.  The graph is acyclic and every producer
      // is already running when a consumer waits, so no grid barrier is needed
      // until the round's end.
      auto is_dirty = [&](int32_t b) {
        return r1_full || __ldcg(a.stamp_dirty[cp] + b) == ep;
      };
      uint32_t* const pctr = a.work_ctr + 2 + cp;
      // items per axis: (dirty block, side); in round 1 of a full update every
      // block is dirty, so each pair is its lower block's side-0 item
      const uint32_t sides = r1_full ? 1u : 2u;
      const uint32_t per_axis = sides * n_dirty;
      // one pair item (warp-uniform); `wait` enables the dataflow dependencies
      auto do_item = [&](uint32_t w, bool wait) {
        {
          const int axis = int(w / per_axis);
          const uint32_t rest = w - uint32_t(axis) * per_axis;
          const uint32_t i = r1_full ? rest : rest >> 1;
          const int side = r1_full ? 0 : int(rest & 1u);
          const int32_t d = r1_full ? int32_t(i) : __ldcg(dirty + i);
          int32_t lo, hi;
          if (side == 0) {
            hi = __ldg(a.nbr + size_t(d) * 6 + 2 * axis);  // d + axis
            lo = d;
            if (hi < 0) return;
          } else {
            lo = __ldg(a.nbr + size_t(d) * 6 + 2 * axis + 1);  // d - axis
            hi = d;
            if (lo < 0) return;
            // pair (lo, d) is handled by lo's side-0 item when lo is dirty
            if (r1_full || __ldcg(a.stamp_dirty[cp] + lo) == ep) return;
          }
          // dependencies, one lane each: sweeps of lo/hi (lanes 0-1); pairs of
          // lower axes touching lo or hi (lanes 2-5: axis 0, 6-9: axis 1)
          bool dep_chg = false;  // the lane's earlier pair changed its block
          if (lane < 2 + 4 * axis && (wait || r1_full)) {
            if (lane < 2) {
              const int32_t b = lane == 0 ? lo : hi;
              if (wait && is_dirty(b)) wait_stamp(a.stamp_swept + b, ep, &a.status->watchdog, 10u + axis, b);
            } else {
              const int q = (lane - 2) >> 2;               // the earlier axis
              const int32_t b = ((lane - 2) & 2) ? hi : lo;
              const bool b_is_hi = ((lane - 2) & 1) == 0;  // pair (b - q, b), else (b, b + q)
              int32_t c = b;
              if (b_is_hi) c = __ldg(a.nbr + size_t(b) * 6 + 2 * q + 1);  // b - q
              if (c >= 0) {
                const int32_t n = __ldg(a.nbr + size_t(c) * 6 + 2 * q);
                if (n >= 0 && (is_dirty(c) || is_dirty(n))) {
                  const uint32_t v = wait ? wait_stamp(a.stamp_pair[q] + c, ep, &a.status->watchdog,
                                                       20u + 10u * q + axis, c)
                                          : ld_acquire(a.stamp_pair[q] + c);
                  dep_chg = (v & (b_is_hi ? kStampHiChg : kStampLoChg)) != 0u;
                }
              }
            }
          }
          const uint32_t chg_mask = __ballot_sync(0xffffffffu, dep_chg);
          __syncwarp();
          if (r1_full) {
            // After reset_parented only sites give, and a pair can only give to
            // a face through a giver on the other face: a block gives here if
            // it holds a site or an earlier pair of this round changed it (for a
            // y (z) pair: the x (x, y) pairs through its faces, whose stamps
            // were just read).  A pair with no giver on either side is the
            // identity: skip it.
            // lanes 2 + 4q + {0, 1} watch lo's pairs, 2 + 4q + {2, 3} hi's
            constexpr uint32_t lo_lanes = 0x0ccu, hi_lanes = 0x330u;
            const bool g_lo = a.site_any[lo] != 0 || (chg_mask & lo_lanes) != 0u;
            const bool g_hi = a.site_any[hi] != 0 || (chg_mask & hi_lanes) != 0u;
            if (!g_lo && !g_hi) {
              if (lane == 0) st_release(a.stamp_pair[axis] + lo, ep);
              return;
            }
          }
          const int dx = axis == 0, dy = axis == 1, dz = axis == 2;
          bool ac = false, bc = false;
          unsigned long long mlo[3] = {0, 0, 0}, mhi[3] = {0, 0, 0};
#pragma unroll
          for (int k = 0; k < 2; ++k) {
            const int f = lane + 32 * k, i0 = f & 7, j0 = f >> 3;
            int ax, ay, az, bx, by, bz;
            if (axis == 0) { ax = 7; ay = i0; az = j0; bx = 0; by = i0; bz = j0; }
            else if (axis == 1) { ax = i0; ay = 7; az = j0; bx = i0; by = 0; bz = j0; }
            else { ax = i0; ay = j0; az = 7; bx = i0; by = j0; bz = 0; }
            const int la = ax + 8 * ay + 64 * az, lb = bx + 8 * by + 64 * bz;
            EV va = load_voxel(work, lo, la), vb = load_voxel(work, hi, lb);
            const bool cb = relax(vb, va, dx, dy, dz, lim);     // exchange_pair :158
            const bool ca = relax(va, vb, -dx, -dy, -dz, lim);  // :159
            if (cb) {
              store_voxel(work, hi, lb, vb);
              line_bits(bx, by, bz, mhi);
            }
            if (ca) {
              store_voxel(work, lo, la, va);
              line_bits(ax, ay, az, mlo);
            }
            ac |= ca;
            bc |= cb;
          }
          ac = __any_sync(0xffffffffu, ac);
          bc = __any_sync(0xffffffffu, bc);
          ++n_pairs;
          __syncwarp();  // the warp's voxel stores before the release of the pair stamp
          if (lane == 0)
            st_release(a.stamp_pair[axis] + lo, ep | (ac ? kStampLoChg : 0u) | (bc ? kStampHiChg : 0u));
          if (a.trace && lane == 0 && r < 16) {
            unsigned long long tm;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tm));
            atomicMax(a.trace + 256 + 4 * r + 1, tm);  // last pair end
            if (r == 1 || r == 3) atomicMax(a.trace + 320 + 4 * r + axis, tm);  // per axis
          }
          const int32_t who[2] = {lo, hi};
          const bool chg[2] = {ac, bc};
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            if (!chg[q]) continue;
            if (a.full) {
              unsigned long long* m = q == 0 ? mlo : mhi;
              const unsigned long long r0 = warp_or64(m[0]), r1 = warp_or64(m[1]), r2 = warp_or64(m[2]);
              if (lane == 0) {
                atomicOr(a.line_mask + 3 * size_t(who[q]), r0);
                atomicOr(a.line_mask + 3 * size_t(who[q]) + 1, r1);
                atomicOr(a.line_mask + 3 * size_t(who[q]) + 2, r2);
              }
            }
            if (lane == 0) {
              if (!a.full) a.stamp_lchg[who[q]] = a.lchg_tag;
              if (atomicMax(a.stamp_dirty[np] + who[q], ep_next) < ep_next) {
                const uint32_t slot = atomicAdd(a.count + (r + 1u) % 3u, 1u);
                a.list[np][slot] = who[q];
              }
            }
          }
        }
      };
      if (a.dataflow) {
        // one item per claim: a warp blocked on a dependency must not hold
        // later items (claiming chunks serialises the chains measurably)
        const uint32_t n_items = 3u * per_axis;
        while (true) {
          uint32_t w = 0;
          if (lane == 0) w = atomicAdd(pctr, 1u);
          w = __shfl_sync(0xffffffffu, w, 0);
          if (w >= n_items) break;
          do_item(w, true);
        }
      } else {  // phased: a grid barrier before each axis group, as the reference
        for (int axis = 0; axis < 3; ++axis) {
          grid.sync();
          stamp();
          for (uint32_t w = uint32_t(axis) * per_axis + wid; w < uint32_t(axis + 1) * per_axis;
               w += nwarps)
            do_item(w, false);
        }
      }
      grid.sync();
      stamp();
      if (*((volatile uint32_t*)&a.count[(r + 1u) % 3u]) == 0) break;
    }
  }
  // ---- changed set of update_esdf (esdf/integrator.cpp:403-411) -------------
  if (a.full) {
    for (uint32_t k = wid; k < n_blocks; k += nwarps) {
      const int32_t s = a.sorted_slots[k];
      bool ch = a.stamp_new[s] == a.call_epoch || a.stamp_mark[s] == a.call_epoch;
      if (!ch && lower) {
        const uint4* p0 = reinterpret_cast<const uint4*>(pcur + size_t(s) * 1536);
        const uint4* p1 = reinterpret_cast<const uint4*>(pnxt + size_t(s) * 1536);
        bool diff = false;
#pragma unroll 4
        for (int q = lane; q < 384; q += 32) {
          const uint4 x = __ldcg(p0 + q), y = __ldcg(p1 + q);
          diff |= (x.x != y.x) | (x.y != y.y) | (x.z != y.z) | (x.w != y.w);
        }
        ch = __any_sync(0xffffffffu, diff);
        ++n_cmp;
      }
      if (lane == 0) a.out_flags[k] = uint8_t(ch);
    }
  }
  if (lane == 0 && (n_pairs | n_cmp)) {
    atomicAdd(&a.status->sum_pairs, n_pairs);
    atomicAdd(&a.status->cmp_blocks, n_cmp);
  }
  grid.sync();
  stamp();
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.r1[0] = a.r1[1] = a.r1[2] = a.r1[3] = 0u;  // zero for the next launch
    a.status->rounds = r;
    a.status->n_esdf_blocks = n_blocks;
    a.meta->round_epoch = base_epoch + r + 2;
    if (a.full && lower) a.meta->cur = cur ^ 1u;
  }
}

// ---- effective set: 7-way rank merge -------------------------------------------
__device__ inline uint32_t lower_bound_u64(const uint64_t* a, uint32_t n, uint64_t k) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (a[mid] < k) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}
__device__ inline uint32_t upper_bound_u64(const uint64_t* a, uint32_t n, uint64_t k) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (a[mid] <= k) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}
// shift j: 0 identity, 1 +x, 2 -x, 3 +y, 4 -y, 5 +z, 6 -z (mark_impl :279-285)
__device__ inline uint64_t shift7(uint64_t k, int j, int sign) {
  if (j == 0) return k;
  const int axis = (j - 1) >> 1;
  const int s = ((j - 1) & 1) ? -1 : 1;
  return key_shift(k, axis, s * sign);
}

__global__ void k_merge7(const uint64_t* __restrict__ upd, const uint32_t* n_ptr,
                         uint64_t* __restrict__ merged) {
  pdl_wait();  // see launch_pdl
  pdl_trigger();
  const uint32_t n = *n_ptr;
  const uint32_t total = 7u * n;
  for (uint32_t it = blockIdx.x * blockDim.x + threadIdx.x; it < total;
       it += gridDim.x * blockDim.x) {
    const int j = int(it / n);
    const uint32_t i = it - uint32_t(j) * n;
    const uint64_t key = shift7(upd[i], j, 1);
    uint32_t rank = i;
    for (int q = 0; q < 7; ++q) {
      if (q == j) continue;
      const uint64_t probe = shift7(key, q, -1);
      rank += q < j ? upper_bound_u64(upd, n, probe) : lower_bound_u64(upd, n, probe);
    }
    merged[rank] = key;
  }
}

// ---- get_or_allocate over a sorted key list --------------------------------------
struct AllocListArgs {
  const uint64_t* keys;
  const uint32_t* n_ptr;
  HashView hash;
  uint64_t* slot_keys;
  LayerMeta* meta;
  uint32_t capacity;
  uint64_t max_blocks;
  int32_t* slots_out;      // per key: slot, or -1 when capacity was exhausted
  uint64_t* new_keys;      // sorted new keys
  int32_t* new_slots;
  uint32_t* n_new_out;
  uint32_t* n_old_out;     // num_blocks before this allocation
  uint32_t* stamp_new;     // may be null
  uint32_t call_epoch;
  DevStatus* status;
};

__global__ void __launch_bounds__(256) k_alloc_list(AllocListArgs a, ScanTiles st) {
  __shared__ uint32_t s_tile, s_scan[64], s_pre[2], s_base;
  scan_prepare_next(st);
  const uint32_t n = *a.n_ptr;
  const uint32_t tiles = (n + blockDim.x - 1) / blockDim.x;
  if (tiles == 0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      *a.n_new_out = 0;
      *a.n_old_out = a.meta->num_blocks;
    }
    return;
  }
  const uint64_t limit = a.capacity < a.max_blocks ? uint64_t(a.capacity) : a.max_blocks;
  while (true) {
    const uint32_t tile = scan_take_tile(st, &s_tile);
    if (tile >= tiles) break;
    if (threadIdx.x == 0) s_base = a.meta->num_blocks;
    const uint32_t i = tile * blockDim.x + threadIdx.x;
    uint64_t k = 0;
    int32_t found = -1;
    bool is_new = false;
    if (i < n) {
      k = a.keys[i];
      found = hash_find_rw(a.hash, k);
      is_new = found < 0;
    }
    uint32_t ea, eb, ta, tb;
    block_scan2(is_new ? 1u : 0u, 0u, ea, eb, ta, tb, s_scan);
    if (threadIdx.x < 32) {  // warp 0: look-back
      uint32_t pa, pb;
      scan_lookback(st, tile, ta, 0u, pa, pb);
      if (threadIdx.x == 0) {
        s_pre[0] = pa;
      }
    }
    __syncthreads();
    const uint32_t base = s_base;
    if (i < n) {
      int32_t slot = found;
      if (is_new) {
        const uint32_t r = s_pre[0] + ea;
        const uint64_t s = uint64_t(base) + r;
        if (s < limit) {
          hash_insert(a.hash, k, int32_t(s));
          a.slot_keys[s] = k;
          slot = int32_t(s);
          a.new_keys[r] = k;
          a.new_slots[r] = slot;
          if (a.stamp_new) a.stamp_new[s] = a.call_epoch;
        } else {
          slot = -1;
        }
      }
      a.slots_out[i] = slot;
    }
    if (threadIdx.x == 0 && tile == tiles - 1) {
      const uint32_t total = s_pre[0] + ta;
      const uint64_t want = uint64_t(base) + total;
      const uint64_t got = want < limit ? want : limit;
      *a.n_new_out = uint32_t(got - base);
      *a.n_old_out = base;
      if (want > a.capacity && a.capacity < a.max_blocks) a.status->pool_overflow = 1u;
      if (want > a.max_blocks) a.status->capacity_error = 1u;
      a.meta->num_blocks = uint32_t(got);
    }
    __syncthreads();
  }
}

// 6-neighbour table of new ESDF blocks (both directions).
__global__ void k_nbr_update(const uint64_t* __restrict__ new_keys,
                             const int32_t* __restrict__ new_slots, const uint32_t* n_ptr,
                             HashView h, int32_t* nbr) {
  const uint32_t n = *n_ptr;
  for (uint32_t it = blockIdx.x * blockDim.x + threadIdx.x; it < 6u * n;
       it += gridDim.x * blockDim.x) {
    const uint32_t i = it / 6;
    const int d = int(it - i * 6);
    const int axis = d >> 1, s = (d & 1) ? -1 : 1;
    const int32_t me = new_slots[i];
    const int32_t nb = hash_find(h, key_shift(new_keys[i], axis, s));
    nbr[size_t(me) * 6 + d] = nb;
    if (nb >= 0) nbr[size_t(nb) * 6 + (d ^ 1)] = me;
  }
}

// Sorted set of all blocks += new (sorted, disjoint) by rank merge.
__global__ void k_merge_sorted(const uint64_t* __restrict__ ok, const int32_t* __restrict__ os,
                               const uint32_t* n_old_ptr, const uint64_t* __restrict__ nk,
                               const int32_t* __restrict__ ns, const uint32_t* n_new_ptr,
                               uint64_t* __restrict__ out_k, int32_t* __restrict__ out_s) {
  const uint32_t n_old = *n_old_ptr, n_new = *n_new_ptr;
  for (uint32_t it = blockIdx.x * blockDim.x + threadIdx.x; it < n_old + n_new;
       it += gridDim.x * blockDim.x) {
    if (it < n_old) {
      const uint64_t k = ok[it];
      const uint32_t r = it + lower_bound_u64(nk, n_new, k);
      out_k[r] = k;
      out_s[r] = os[it];
    } else {
      const uint32_t j = it - n_old;
      const uint64_t k = nk[j];
      const uint32_t r = j + lower_bound_u64(ok, n_old, k);
      out_k[r] = k;
      out_s[r] = ns[j];
    }
  }
}

// unique + has_block(TSDF) + ESDF get_or_allocate in one ordered pass
// (mark_impl :279-295): per merged element one thread; tiles publish the
// (effective, new) count pair through one look-back; new blocks get slots
// num_blocks + rank(new) in key order, as the reference's sorted loop does.
__global__ void __launch_bounds__(256) k_effective_alloc(const uint64_t* __restrict__ merged,
                                                         const uint32_t* n_upd, HashView tsdf,
                                                         uint64_t* __restrict__ eff_keys,
                                                         int32_t* __restrict__ eff_tslot,
                                                         uint32_t* n_eff, AllocListArgs a,
                                                         ScanTiles st) {
  pdl_wait();  // see launch_pdl
  pdl_trigger();
  __shared__ uint32_t s_tile, s_scan[64], s_pre[2], s_base;
  scan_prepare_next(st);
  const uint32_t n = 7u * (*n_upd);
  const uint32_t tiles = (n + blockDim.x - 1) / blockDim.x;
  if (tiles == 0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      *n_eff = 0;
      *a.n_new_out = 0;
      *a.n_old_out = a.meta->num_blocks;
    }
    return;
  }
  const uint64_t limit = a.capacity < a.max_blocks ? uint64_t(a.capacity) : a.max_blocks;
  while (true) {
    const uint32_t tile = scan_take_tile(st, &s_tile);
    if (tile >= tiles) break;
    if (threadIdx.x == 0) s_base = a.meta->num_blocks;
    const uint32_t r = tile * blockDim.x + threadIdx.x;
    bool keep = false, is_new = false;
    int32_t ts = -1, found = -1;
    uint64_t k = 0;
    if (r < n) {
      k = merged[r];
      if (r == 0 || merged[r - 1] != k) {
        ts = hash_find(tsdf, k);
        keep = ts >= 0;
        if (keep) {
          found = hash_find_rw(a.hash, k);
          is_new = found < 0;
        }
      }
    }
    uint32_t ea, eb, ta, tb;
    block_scan2(keep ? 1u : 0u, is_new ? 1u : 0u, ea, eb, ta, tb, s_scan);
    if (threadIdx.x < 32) {  // warp 0: look-back
      uint32_t pa, pb;
      scan_lookback(st, tile, ta, tb, pa, pb);
      if (threadIdx.x == 0) {
        s_pre[0] = pa;
        s_pre[1] = pb;
      }
    }
    __syncthreads();
    const uint32_t base = s_base;
    if (keep) {
      const uint32_t e = s_pre[0] + ea;
      int32_t slot = found;
      if (is_new) {
        const uint32_t q = s_pre[1] + eb;
        const uint64_t sl = uint64_t(base) + q;
        if (sl < limit) {
          hash_insert(a.hash, k, int32_t(sl));
          a.slot_keys[sl] = k;
          slot = int32_t(sl);
          a.new_keys[q] = k;
          a.new_slots[q] = slot;
          if (a.stamp_new) a.stamp_new[sl] = a.call_epoch;
        } else {
          slot = -1;
        }
      }
      eff_keys[e] = k;
      eff_tslot[e] = ts;
      a.slots_out[e] = slot;
    }
    if (threadIdx.x == 0 && tile == tiles - 1) {
      *n_eff = s_pre[0] + ta;
      const uint64_t want = uint64_t(base) + s_pre[1] + tb;
      const uint64_t got = want < limit ? want : limit;
      *a.n_new_out = uint32_t(got - base);
      *a.n_old_out = base;
      if (want > a.capacity && a.capacity < a.max_blocks) a.status->pool_overflow = 1u;
      if (want > a.max_blocks) a.status->capacity_error = 1u;
      a.meta->num_blocks = uint32_t(got);
    }
    __syncthreads();
  }
}

// Side structures of the new blocks (neighbour table, sorted set), done by
// k_mark's CTAs after their marking: neither depends on the other.
struct PostAllocArgs {
  const uint64_t* new_keys;
  const int32_t* new_slots;
  const uint32_t* n_new;
  const uint32_t* n_old;
  HashView hash;
  int32_t* nbr;
  const uint64_t* old_sorted_k;
  const int32_t* old_sorted_s;
  uint64_t* out_sorted_k;
  int32_t* out_sorted_s;
};
__device__ inline void post_alloc(const PostAllocArgs& p) {
  const uint32_t n_new = *p.n_new, n_old = *p.n_old;
  const uint32_t gsz = gridDim.x * blockDim.x;
  const uint32_t gtid = blockIdx.x * blockDim.x + threadIdx.x;
  for (uint32_t it = gtid; it < 6u * n_new; it += gsz) {  // k_nbr_update
    const uint32_t i = it / 6;
    const int d = int(it - i * 6);
    const int axis = d >> 1, s = (d & 1) ? -1 : 1;
    const int32_t me = p.new_slots[i];
    const int32_t nb = hash_find(p.hash, key_shift(p.new_keys[i], axis, s));
    p.nbr[size_t(me) * 6 + d] = nb;
    if (nb >= 0) p.nbr[size_t(nb) * 6 + (d ^ 1)] = me;
  }
  for (uint32_t it = gtid; it < n_old + n_new; it += gsz) {  // k_merge_sorted
    if (it < n_old) {
      const uint64_t k = p.old_sorted_k[it];
      const uint32_t r = it + lower_bound_u64(p.new_keys, n_new, k);
      p.out_sorted_k[r] = k;
      p.out_sorted_s[r] = p.old_sorted_s[it];
    } else {
      const uint32_t j = it - n_old;
      const uint64_t k = p.new_keys[j];
      const uint32_t r = j + lower_bound_u64(p.old_sorted_k, n_old, k);
      p.out_sorted_k[r] = k;
      p.out_sorted_s[r] = p.new_slots[j];
    }
  }
}

// ---- mark_sites — esdf/integrator.cpp:177-266 (classifiers), 268-348 ------------
struct MarkArgs {
  const uint64_t* eff_keys;
  const int32_t* eff_tslot;
  const int32_t* eff_eslot;
  const uint32_t* n_eff;
  const void* src_pool;  // TSDF (float2) or occupancy (float) blocks
  HashView src_hash;     // occupancy: the 6 face-neighbour blocks
  float occ_threshold;   // EsdfConfig::occupied_log_odds_threshold
  uint32_t* pools[2];
  const LayerMeta* meta;
  float site_threshold;
  Limits lim;
  uint32_t* stamp_mark;
  uint32_t call_epoch;
  uint8_t* flags;  // per effective block: 1 changed, 2 to_update, 4 to_clear
  DevStatus* status;
  uint8_t* site_any;  // per ESDF slot: the block holds a site after marking
  PostAllocArgs post;
  // mark skip (Layer::mark_stamp): null mark_stamp = off; skip_on = 0: the
  // stamps are only written (every stamp is below the floor anyway)
  uint32_t* mark_stamp;
  int skip_on;
  const uint32_t* src_stamp;  // the source's stamp_mod
  uint32_t skip_floor;        // stamps at or below it are not trusted
  uint32_t mark_now;          // this marking's tick
};

// OccupancyClassifier (esdf/integrator.cpp:200-266): observed = log_odds != 0;
// inside = occupied = observed && log_odds > threshold; a site is an occupied
// voxel with an observed-free 6-neighbour, looked up in the face-neighbour
// block across a border (absent neighbour block: no neighbour).
__device__ inline bool occ_free(float lo, float thr) { return lo != 0.0f && !(lo > thr); }

__device__ inline bool occ_has_free_neighbour(const float* src, int32_t self, const int32_t nb[6],
                                              int lin, float thr) {
  const int x = lin & 7, y = (lin >> 3) & 7, z = lin >> 6;
  const int c[3] = {x, y, z};
#pragma unroll
  for (int n = 0; n < 6; ++n) {  // {+x, -x, +y, -y, +z, -z} (:229-231)
    const int axis = n >> 1, step = (n & 1) ? -1 : 1;
    const int m = c[axis] + step;
    int32_t blk = self;
    int nl;
    if (m >= 0 && m < 8) {
      nl = lin + step * (axis == 0 ? 1 : axis == 1 ? 8 : 64);
    } else {
      blk = nb[n];
      nl = lin + step * (axis == 0 ? -7 : axis == 1 ? -56 : -448);  // wrap (N + m) % N
    }
    if (blk >= 0 && occ_free(__ldg(src + size_t(blk) * kVPB + nl), thr)) return true;
  }
  return false;
}

// One warp per effective block: lane l holds voxels 4 * (l + 32 h) + e
// (h = 0..3, e = 0..3), so the ESDF block (3 x 16-byte words per 4 voxels)
// and the source block (TSDF: 2, occupancy: 1 x 16-byte words per 4 voxels)
// load and store coalesced, all in flight at once; the block flags are warp
// ballots.
template <bool OCC, bool SKIP = false>
__global__ void __launch_bounds__(256) k_mark(MarkArgs a) {
  pdl_wait();  // see launch_pdl
  pdl_trigger();
  const uint32_t n = *a.n_eff;
  uint32_t* pool = a.pools[a.meta->cur];
  const int lane = threadIdx.x & 31;
  const uint32_t nwarps = gridDim.x * (blockDim.x >> 5);
  for (uint32_t e = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; e < n; e += nwarps) {
    const int32_t es = a.eff_eslot[e];
    if (es < 0) {  // capacity exhausted before this block (MapCapacityError)
      if (lane == 0) a.flags[e] = 0;
      continue;
    }
    const int32_t ts = a.eff_tslot[e];
    if (!OCC && SKIP) {  // unchanged source block since its last marking: same bytes
      // (lanes 0 / 1 load the two stamps side by side: one L2 trip)
      uint32_t st = 0;
      if (lane == 0) st = a.mark_stamp[es];
      else if (lane == 1) st = a.src_stamp[ts];
      const uint32_t ms = __shfl_sync(0xffffffffu, st, 0), sm = __shfl_sync(0xffffffffu, st, 1);
      if (ms > a.skip_floor && sm <= ms) {
        if (lane == 0) a.flags[e] = 0;
        continue;
      }
    }
    constexpr int kSrcWords = OCC ? 1 : 2;  // 16-byte source words per 4 voxels
    const uint4* t4 = reinterpret_cast<const uint4*>(
        static_cast<const unsigned char*>(a.src_pool) + size_t(ts) * kVPB * 4 * kSrcWords);
    uint4* e4 = reinterpret_cast<uint4*>(pool + size_t(es) * 1536);
    bool bch = false, bup = false, bcl = false, bsite = false;
    uint32_t w[48];
    float tv[16 * kSrcWords];
    int32_t nb[6];
    if (OCC) {  // BlockCtx::neighbors (:216-226): lanes 0..5 probe, then broadcast
      int32_t mine = -1;
      if (lane < 6) mine = hash_find(a.src_hash, key_shift(a.eff_keys[e], lane >> 1, (lane & 1) ? -1 : 1));
#pragma unroll
      for (int n = 0; n < 6; ++n) nb[n] = __shfl_sync(0xffffffffu, mine, n);
    }
#pragma unroll
    for (int h = 0; h < 4; ++h) {  // all loads in flight before any use
      const int q = lane + 32 * h;  // voxels 4q .. 4q + 3
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const uint4 v = __ldcg(e4 + 3 * q + j);
        w[12 * h + 4 * j] = v.x; w[12 * h + 4 * j + 1] = v.y;
        w[12 * h + 4 * j + 2] = v.z; w[12 * h + 4 * j + 3] = v.w;
      }
#pragma unroll
      for (int j = 0; j < kSrcWords; ++j) {
        const uint4 v = __ldcg(t4 + kSrcWords * q + j);
        const int o = 4 * kSrcWords * h + 4 * j;
        tv[o] = __uint_as_float(v.x); tv[o + 1] = __uint_as_float(v.y);
        tv[o + 2] = __uint_as_float(v.z); tv[o + 3] = __uint_as_float(v.w);
      }
    }
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      const int q = lane + 32 * h;
      bool ch = false;
#pragma unroll
      for (int v4 = 0; v4 < 4; ++v4) {
        const int v = 4 * h + v4;
        bool observed, site, inside;
        if (!OCC) {  // TsdfClassifier — :177-198
          const float dist = tv[2 * v], weight = tv[2 * v + 1];
          observed = weight > 0.0f;
          site = observed && fabsf(dist) <= a.site_threshold;
          inside = observed && dist < 0.0f;
        } else {     // OccupancyClassifier — :200-266
          const float lo = tv[v];
          observed = lo != 0.0f;
          inside = observed && lo > a.occ_threshold;
          site = inside && occ_has_free_neighbour(static_cast<const float*>(a.src_pool), ts, nb,
                                                  4 * q + v4, a.occ_threshold);
        }
        bsite |= site;
        const uint32_t o0 = w[3 * v], o1 = w[3 * v + 1], o2 = w[3 * v + 2];
        const EV ev = ev_unpack(o0, o1, o2);
        EV nv = ev;
        if (!observed) {
          if (ev.f & VXM_ESDF_SITE) bcl = true;
          nv = EV{0, 0, 0, 0, 0u, 0u};
        } else {
          nv.f = VXM_ESDF_OBSERVED | (site ? VXM_ESDF_SITE : 0) | (inside ? VXM_ESDF_INSIDE : 0);
          const bool was_obs = ev.f & VXM_ESDF_OBSERVED, was_site = ev.f & VXM_ESDF_SITE;
          if (site) {
            nv.sq = 0;
            nv.px = nv.py = nv.pz = 0;
            if (!was_obs || !was_site) bup = true;
          } else if (!was_obs) {
            reset_to_saturated(nv, a.lim);
            bup = true;
          } else if (was_site) {
            reset_to_saturated(nv, a.lim);
            bcl = true;
            bup = true;
          } else if (bool(ev.f & VXM_ESDF_INSIDE) != inside) {
            reset_to_saturated(nv, a.lim);
            bup = true;
          }
        }
        const uint32_t n0 = uint32_t(nv.sq), n1 = ev_w1(nv), n2 = ev_w2(nv);
        ch |= (n0 != o0) | (n1 != o1) | (n2 != o2);
        w[3 * v] = n0;
        w[3 * v + 1] = n1;
        w[3 * v + 2] = n2;
      }
      if (ch) {
#pragma unroll
        for (int j = 0; j < 3; ++j)
          __stcg(e4 + 3 * q + j, make_uint4(w[12 * h + 4 * j], w[12 * h + 4 * j + 1],
                                            w[12 * h + 4 * j + 2], w[12 * h + 4 * j + 3]));
      }
      bch |= ch;
    }
    bch = __any_sync(0xffffffffu, bch);
    bup = __any_sync(0xffffffffu, bup);
    bcl = __any_sync(0xffffffffu, bcl);
    bsite = __any_sync(0xffffffffu, bsite);
    if (lane == 0) {
      if (a.mark_stamp) a.mark_stamp[es] = a.mark_now;
      a.site_any[es] = bsite ? 1 : 0;
      a.flags[e] = uint8_t((bch ? 1 : 0) | (bup ? 2 : 0) | (bcl ? 4 : 0));
      if (bch) a.stamp_mark[es] = a.call_epoch;
      if (bup || bcl) atomicOr(&a.status->any_update, 1u);
    }
  }
  post_alloc(a.post);
}

// ---- clear_invalid — esdf/integrator.cpp:433-486 --------------------------------
struct ClearArgs {
  const uint64_t* sorted_keys;
  const int32_t* sorted_slots;
  uint32_t n_all;
  const uint64_t* clear_keys;
  uint32_t n_clear;
  int radius;
  HashView hash;
  uint32_t* pool;
  Limits lim;
  uint8_t* flags;  // per sorted index: 1 = cleared something
};

__device__ inline int64_t floor_div8(int64_t a) { return a >= 0 ? a / 8 : -((-a + 7) / 8); }

__global__ void __launch_bounds__(256) k_clear(ClearArgs a) {
  __shared__ int s_scan;
  for (uint32_t k = blockIdx.x; k < a.n_all; k += gridDim.x) {
    const uint64_t key = a.sorted_keys[k];
    const int32_t gx = key_x(key), gy = key_y(key), gz = key_z(key);
    if (threadIdx.x == 0) s_scan = 0;
    __syncthreads();
    for (uint32_t c = threadIdx.x; c < a.n_clear; c += blockDim.x) {
      const uint64_t ck = a.clear_keys[c];
      if (abs(gx - key_x(ck)) <= a.radius && abs(gy - key_y(ck)) <= a.radius &&
          abs(gz - key_z(ck)) <= a.radius)
        s_scan = 1;
    }
    __syncthreads();
    const bool scan = s_scan != 0;
    bool any = false;
    if (scan) {
      const int32_t s = a.sorted_slots[k];
      for (int q = 0; q < 2; ++q) {
        const int lin = threadIdx.x + 256 * q;
        uint32_t* p = a.pool + size_t(s) * 1536 + lin * 3;
        EV v = ev_unpack(p[0], p[1], p[2]);
        if (!ev_has_parent(v)) continue;
        const int64_t px = int64_t(gx) * 8 + (lin & 7) + v.px;
        const int64_t py = int64_t(gy) * 8 + ((lin >> 3) & 7) + v.py;
        const int64_t pz = int64_t(gz) * 8 + (lin >> 6) + v.pz;
        const int64_t bx = floor_div8(px), by = floor_div8(py), bz = floor_div8(pz);
        bool parent_site = false;
        if (coord_ok(bx) && coord_ok(by) && coord_ok(bz)) {
          const int32_t ps = hash_find(a.hash, pack_key(int32_t(bx), int32_t(by), int32_t(bz)));
          if (ps >= 0) {
            const int plin = int(px - bx * 8) + 8 * int(py - by * 8) + 64 * int(pz - bz * 8);
            const uint32_t w2 = a.pool[size_t(ps) * 1536 + plin * 3 + 2];
            parent_site = ((w2 >> 16) & VXM_ESDF_SITE) != 0;
          }
        }
        if (!parent_site) {
          // only clears parents; reads above only test site bits (never written)
          reset_to_saturated(v, a.lim);
          p[0] = uint32_t(v.sq);
          p[1] = ev_w1(v);
          p[2] = ev_w2(v);
          any = true;
        }
      }
    }
    any = __syncthreads_or(any);
    if (threadIdx.x == 0) a.flags[k] = uint8_t(any);
  }
}

// Flag blocks (in sorted order) whose lowering-change tag matches.
__global__ void k_flag_tag(const int32_t* sorted_slots, uint32_t n, const uint32_t* stamp,
                           uint32_t tag, uint8_t* flags) {
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x)
    flags[k] = uint8_t(stamp[sorted_slots[k]] == tag);
}

__global__ void k_lookup_slots(const uint64_t* keys, uint32_t n, HashView h, int32_t* out) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = hash_find(h, keys[i]);
}

// ---- host drivers -----------------------------------------------------------------
Limits limits_for(const vxm_esdf_config& cfg, double vs) {
  const double r = cfg.max_distance / vs;  // esdf/integrator.hpp:43-54
  Limits l;
  l.max_sq = int32_t(std::llround(r * r));
  l.cap_sq = l.max_sq < 16 ? l.max_sq : 16;
  return l;
}

// The limits of a call on layer E, noting the largest max_sq the layer's data
// may have been saturated with (k_lower_xr's compact-format rule).
static Limits esdf_limits(Layer* E, const vxm_esdf_config& cfg) {
  const Limits l = limits_for(cfg, E->vs);
  const int m = l.max_sq < 0 ? INT32_MAX : l.max_sq;
  if (m > E->esdf_max_sq_seen) E->esdf_max_sq_seen = m;
  return l;
}

uint32_t grid_for(Context* ctx, uint64_t n, int per_sm) {
  return uint32_t(std::max<uint64_t>(1, std::min<uint64_t>(ceil_div(std::max<uint64_t>(n, 1), 256),
                                                           uint64_t(ctx->sm_count) * per_sm)));
}


EsdfScratch esdf_scratch(Context* ctx, uint32_t n_upd_cap, uint32_t n_all_cap) {
  const uint64_t n7 = 7ull * std::max<uint32_t>(n_upd_cap, 1);
  const uint64_t nf = std::max<uint64_t>(n7, n_all_cap) + 16;
  ctx->tmp[0].ensure(sizeof(uint64_t) * n7);
  ctx->tmp[1].ensure(sizeof(uint64_t) * n7);
  ctx->tmp[2].ensure(sizeof(int32_t) * n7 * 2);
  ctx->tmp[3].ensure(sizeof(uint64_t) * n7);
  ctx->tmp[4].ensure(sizeof(int32_t) * n7 + nf);
  ctx->tmp[5].ensure(64 * sizeof(uint32_t));
  EsdfScratch s;
  s.merged = ctx->tmp[0].as<uint64_t>();
  s.eff_keys = ctx->tmp[1].as<uint64_t>();
  s.eff_tslot = ctx->tmp[2].as<int32_t>();
  s.eff_eslot = s.eff_tslot + n7;
  s.new_keys = ctx->tmp[3].as<uint64_t>();
  s.new_slots = ctx->tmp[4].as<int32_t>();
  s.flags = reinterpret_cast<uint8_t*>(s.new_slots + n7);
  s.counts = ctx->tmp[5].as<uint32_t>();
  return s;
}

// effective set + ESDF allocation + neighbour table + sorted-set merge + mark.
// `updated` must hold sorted unique keys (device).  Returns the upper bound of
// the effective count.
uint32_t esdf_mark_phase(Layer* E, Layer* T, BlockList* updated,
                                const vxm_esdf_config& cfg, EsdfScratch& s, uint32_t epoch, bool mark_skip) {
  Context* ctx = E->ctx;
  ++E->esdf_gen;
  const uint32_t nu_cap = std::max<uint32_t>(updated->count_hint, 1);
  const uint32_t n7 = 7u * nu_cap;
  const uint64_t* upd = updated->keys.as<uint64_t>();
  ctx->prof_begin("k_merge7");
  launch_pdl(ctx->stream, k_merge7, dim3(grid_for(ctx, n7)), dim3(256), 0, upd, updated->d_count, s.merged);
  ctx->prof_end();
  ctx->count_launch();
  {
    AllocListArgs al{};
    al.hash = E->hash;
    al.slot_keys = E->slot_keys;
    al.meta = E->meta;
    al.capacity = E->capacity;
    al.max_blocks = E->max_blocks;
    al.slots_out = s.eff_eslot;
    al.new_keys = s.new_keys;
    al.new_slots = s.new_slots;
    al.n_new_out = s.counts + 1;
    al.n_old_out = s.counts + 2;
    al.stamp_new = E->stamp_new;
    al.call_epoch = epoch;
    al.status = ctx->status_w();
    const ScanTiles st = ctx->next_scan(ceil_div(n7, 256));
    ctx->prof_begin("k_effective_alloc");
    launch_pdl(ctx->stream, k_effective_alloc, dim3(grid_for(ctx, n7, 4)), dim3(256), 0, 
        s.merged, updated->d_count, T->hash, s.eff_keys, s.eff_tslot, s.counts + 0, al, st);
    ctx->prof_end();
    ctx->count_launch();
  }
  const int sp = E->sorted_parity;
  PostAllocArgs pa{s.new_keys, s.new_slots, s.counts + 1, s.counts + 2, E->hash, E->nbr,
                   E->sorted_keys[sp], E->sorted_slots[sp], E->sorted_keys[1 - sp],
                   E->sorted_slots[1 - sp]};
  E->sorted_parity = 1 - sp;
  MarkArgs m{};
  m.eff_keys = s.eff_keys;
  m.eff_tslot = s.eff_tslot;
  m.eff_eslot = s.eff_eslot;
  m.n_eff = s.counts + 0;
  const bool occ = T->type == VXM_LAYER_OCCUPANCY;
  m.src_pool = T->pool[0];
  m.src_hash = T->hash;
  m.occ_threshold = cfg.occupied_log_odds_threshold;
  m.pools[0] = static_cast<uint32_t*>(E->pool[0]);
  m.pools[1] = static_cast<uint32_t*>(E->pool[1]);
  m.meta = E->meta;
  m.site_threshold = float(cfg.site_threshold);
  m.lim = esdf_limits(E, cfg);
  m.stamp_mark = E->stamp_mark;
  m.call_epoch = epoch;
  m.flags = s.flags;
  m.status = ctx->status_w();
  m.site_any = E->site_any;
  m.post = pa;
  if (mark_skip && !occ) {  // (the fused update decides whether the stamps are trustworthy)
    m.mark_stamp = E->mark_stamp;
    m.src_stamp = T->stamp_mod;
    m.skip_floor = std::max(E->mark_floor, T->mod_floor);
    m.mark_now = next_mod_tick();
    m.skip_on = E->mark_chain ? 1 : 0;
  }
  ctx->prof_begin("k_mark");
  // one wave of warps, each takes blocks until done
  const int mark_per_sm =
      ctx->resident_per_sm(occ ? (const void*)k_mark<true> : (const void*)k_mark<false>, 256);
  if (occ)
    launch_pdl(ctx->stream, k_mark<true>, dim3(ctx->sm_count * mark_per_sm), dim3(256), 0, m);
  else if (m.skip_on)  // (its own instantiation: the marking without the skip test is unchanged)
    launch_pdl(ctx->stream, k_mark<false, true>, dim3(ctx->sm_count * mark_per_sm), dim3(256), 0, m);
  else
    launch_pdl(ctx->stream, k_mark<false>, dim3(ctx->sm_count * mark_per_sm), dim3(256), 0, m);
  ctx->prof_end();
  ctx->count_launch();
  check_launch(ctx, "esdf mark phase");
  return n7;
}

static int lower_grid(Context* ctx) {
  return ctx->resident_per_sm((const void*)k_lower3, kL3Threads, 0, 4) * ctx->sm_count;
}

bool launch_lower_xr(Context* ctx, LowerArgs& la, uint32_t n_blocks_hint);  // lower_xr.cu: true when it compacted

// The cross-round kernel removes the per-round barrier and overlaps rounds:
// a win while rounds are latency-bound (maps of up to tens of thousands of
// blocks, e.g. C2: 0.26 -> 0.18 ms), and, with the current dataflow, also on
// the throughput-bound large maps (k_lower on C3 / C4 / C5: -1 / -2 / -2 %),
// so it is the default for every map (VXM_LOWER_XROUND=1 keeps the barrier
// schedule above kXrMaxBlocks, 0 always).
constexpr uint32_t kXrMaxBlocks = 48 * 1024;

// Returns whether the kernel also wrote the changed list (la.out_keys).
static bool launch_lower(Context* ctx, LowerArgs& la, uint32_t n_blocks_hint) {
  static const bool trace = std::getenv("VXM_TRACE_LOWER") != nullptr;
  static const int xround = [] {
    const char* e = std::getenv("VXM_LOWER_XROUND");  // 0 never, 1 by map size, 2 always
    return e ? std::atoi(e) : 2;
  }();
  if (la.full && la.dataflow && !trace &&  // (VXM_TRACE_LOWER traces k_lower3)
      (xround == 2 || (xround == 1 && n_blocks_hint <= kXrMaxBlocks))) {  // update_esdf
    return launch_lower_xr(ctx, la, n_blocks_hint);
  }
  static DevBuf trace_buf;
  if (trace) {
    trace_buf.ensure(512 * sizeof(unsigned long long));
    VXM_CUDA(cudaMemsetAsync(trace_buf.p, 0, 512 * sizeof(unsigned long long), ctx->stream));
    la.trace = trace_buf.as<unsigned long long>();
  }
  void* args[] = {&la};
  const int grid = lower_grid(ctx);
  ctx->prof_begin("k_lower");
  VXM_CUDA(cudaLaunchCooperativeKernel((const void*)k_lower3, dim3(grid), dim3(kL3Threads), args, 0,
                                       ctx->stream));
  ctx->prof_end();
  if (trace) {
    unsigned long long h[512];
    VXM_CUDA(cudaMemcpyAsync(h, trace_buf.p, sizeof h, cudaMemcpyDeviceToHost, ctx->stream));
    VXM_CUDA(cudaStreamSynchronize(ctx->stream));
    std::fprintf(stderr, "[k_lower grid=%d] phases(us):", grid);
    for (unsigned long long i = 2; i <= h[0] && i < 128; ++i)
      std::fprintf(stderr, " %.1f", (h[i] - h[i - 1]) * 1e-3);
    std::fprintf(stderr, " | total %.1f\n", h[0] > 1 ? (h[h[0]] - h[1]) * 1e-3 : 0.0);
    for (int r = 1; r < 16 && h[128 + 8 * r]; ++r) {
      const unsigned long long* d = h + 128 + 8 * r;
      std::fprintf(stderr,
                   "  r%d: %llu blocks, mean load %.2f sweep %.2f store %.2f us; max block %.1f, max "
                   "sweep %.1f us; passes mean %.2f max %llu\n",
                   r, d[0], d[1] * 1e-3 / d[0], d[2] * 1e-3 / d[0], d[3] * 1e-3 / d[0], d[4] * 1e-3,
                   d[5] * 1e-3, double(d[6]) / d[0], d[7]);
    }
    for (int r = 1; r < 16 && h[256 + 4 * r + 3]; ++r) {
      const unsigned long long* e = h + 256 + 4 * r;
      const double t0 = double(e[3]);
      const double nxt = (r + 1 < 16 && h[256 + 4 * (r + 1) + 3]) ? double(h[256 + 4 * (r + 1) + 3]) : 0.0;
      std::fprintf(stderr, "  r%d timeline (us from round start): last sweep %.1f, last copy %.1f, last pair %.1f, next round %.1f",
                   r, e[0] ? (e[0] - t0) * 1e-3 : 0.0, e[2] ? (e[2] - t0) * 1e-3 : 0.0,
                   e[1] ? (e[1] - t0) * 1e-3 : 0.0, nxt ? (nxt - t0) * 1e-3 : 0.0);
      if (r == 1 || r == 3)
        std::fprintf(stderr, "; pair axes x %.1f y %.1f z %.1f", (h[320 + 4 * r] - t0) * 1e-3,
                     (h[320 + 4 * r + 1] - t0) * 1e-3, (h[320 + 4 * r + 2] - t0) * 1e-3);
      std::fprintf(stderr, "\n");
    }
  }
  ctx->count_launch();
  return false;
}

LowerArgs lower_args(Layer* E, const vxm_esdf_config& cfg) {
  LowerArgs la{};
  la.pool[0] = static_cast<uint32_t*>(E->pool[0]);
  la.pool[1] = static_cast<uint32_t*>(E->pool[1]);
  la.meta = E->meta;
  la.nbr = E->nbr;
  la.stamp_dirty[0] = E->stamp_dirty[0];
  la.stamp_dirty[1] = E->stamp_dirty[1];
  la.stamp_lchg = E->stamp_lchg;
  la.list[0] = E->dirty_list[0];
  la.list[1] = E->dirty_list[1];
  la.count = E->dirty_count;
  la.work_ctr = E->dirty_count + 3;  // [0,1,2] list counts, [3..6] work counters
  la.line_mask = E->line_mask;
  la.stamp_swept = E->stamp_swept;
  la.site_any = E->site_any;
  la.site_near = E->site_near;
  la.r1_list = E->r1_list;
  la.r1 = E->dirty_count + 7;
  la.ring = E->dirty_count + kRingOffset;
  la.dlist[0] = E->dlist[0];
  la.dlist[1] = E->dlist[1];
  la.capacity = E->capacity;
  for (int i = 0; i < 3; ++i) la.pair_face[i] = E->pair_face[i];

  static const int dataflow = [] {
    const char* e = std::getenv("VXM_LOWER_DATAFLOW");
    return e ? std::atoi(e) : 1;
  }();
  la.dataflow = dataflow;
  for (int i = 0; i < 3; ++i) la.stamp_pair[i] = E->stamp_pair[i];
  la.stamp_r1same = E->stamp_r1same;
  la.stamp_quiet = E->stamp_quiet;
  la.quiet_epoch = 0;
  la.quiet_dense = 0;
  la.lim = esdf_limits(E, cfg);
  la.status = E->ctx->status_w();
  la.fast_only = !E->esdf_user_data && E->esdf_max_sq_seen <= kFastOff * kFastOff;
  return la;
}

void esdf_launch(Layer* E, Layer* T, BlockList* updated, const vxm_esdf_config& cfg,
                 BlockList* changed_out) {
  Context* ctx = E->ctx;
  const uint32_t epoch = ++ctx->call_epoch;
  // E->num_blocks is exact: every call that allocates adopts the meta at its end.
  const uint32_t n7 = 7u * std::max<uint32_t>(updated->count_hint, 1);
  // capacity for every effective block: at most 7 per updated block, and at
  // most one per TSDF block (effective blocks are allocated in the TSDF); when
  // the ESDF block set is known to be a subset of T's, T's pool bounds it
  E->note_esdf_source(T);
  uint64_t need = uint64_t(E->num_blocks) + std::min<uint64_t>(n7, T->capacity);
  if (E->bounded_by(T)) need = std::min<uint64_t>(need, T->capacity);
  E->ensure_capacity(std::min<uint64_t>(need, E->max_blocks));
  const uint32_t n_all_cap = E->capacity;
  EsdfScratch s = esdf_scratch(ctx, updated->count_hint, n_all_cap);
  // the quiet chain (Layer::stamp_quiet): unbroken since the last k_lower_xr
  // update (growth above breaks it), same limits
  const Limits qlim = esdf_limits(E, cfg);
  const uint32_t quiet_epoch = E->xr_gen == E->esdf_gen && E->xr_max_sq == qlim.max_sq &&
                               E->xr_cap_sq == qlim.cap_sq ? E->xr_epoch : 0u;
  // the mark skip's stamps hold while the quiet chain does and the source and
  // site threshold are the last update's; otherwise every stamp is dropped
  const bool occ_src = T->type == VXM_LAYER_OCCUPANCY;
  E->mark_chain = E->xr_gen == E->esdf_gen && E->mark_src_uid == T->uid &&
                  E->mark_site_threshold == float(cfg.site_threshold);
  if (!E->mark_chain) E->mark_floor = next_mod_tick();
  E->mark_src_uid = T->uid;
  E->mark_site_threshold = float(cfg.site_threshold);
  esdf_mark_phase(E, T, updated, cfg, s, epoch, !occ_src);
  LowerArgs la = lower_args(E, cfg);
  la.quiet_epoch = quiet_epoch;
  la.quiet_dense = quiet_epoch != 0u && uint64_t(E->xr_quiet) * 2u > E->num_blocks;
  la.full = 1;
  la.sorted_slots = E->sorted_slots[E->sorted_parity];
  la.stamp_new = E->stamp_new;
  la.stamp_mark = E->stamp_mark;
  la.call_epoch = epoch;
  la.out_flags = s.flags;
  changed_out->ensure(n_all_cap);
  la.sorted_keys = E->sorted_keys[E->sorted_parity];
  la.out_keys = changed_out->keys.as<uint64_t>();
  la.out_n = changed_out->d_count;
  if (!launch_lower(ctx, la, E->num_blocks)) {  // the cross-round kernel compacts in-kernel
    launch_compact_keys(ctx, E->sorted_keys[E->sorted_parity], s.flags, &E->meta->num_blocks,
                        n_all_cap, changed_out->keys.as<uint64_t>(), changed_out->d_count, nullptr,
                        "k_compact_esdf");
  } else {  // k_lower_xr: the chain continues from this update
    E->xr_gen = E->esdf_gen;
    E->xr_epoch = epoch;
    E->xr_max_sq = qlim.max_sq;
    E->xr_cap_sq = qlim.cap_sq;
  }
  check_launch(ctx, "k_lower");
  changed_out->host_valid = false;
  changed_out->host_pending = false;
  changed_out->count_hint = n_all_cap;
  if (changed_out->want_host) changed_out->enqueue_host();  // host result, same sync
  ctx->queue_copy(s.counts + 0, &ctx->d_status->n_effective, 2);  // n_effective, n_esdf_new
  ctx->queue_copy(changed_out->d_count, &ctx->d_status->n_out);
}

void esdf_finish(Layer* E, BlockList* changed_out) {
  Context* ctx = E->ctx;
  const DevStatus& st = *ctx->h_status;
  if (st.capacity_error || st.pool_overflow || st.watchdog) ++E->esdf_gen;  // (breaks the quiet chain)
  if (st.capacity_error || st.pool_overflow)
    throw Error(VXM_ERR_CAPACITY, "Layer: block capacity exhausted");
  if (st.watchdog)
    throw Error(VXM_ERR_INTERNAL, "ESDF lowering: dependency wait expired (code " +
                                      std::to_string(st.pad3[0]) + ", block " +
                                      std::to_string(st.pad3[1]) + ", epoch " +
                                      std::to_string(st.pad3[2]) + ")");
  changed_out->count_hint = std::min<uint32_t>(changed_out->count_hint, st.n_out);
  vxm_stats& w = ctx->stats;
  w.esdf_calls += 1;
  w.esdf_blocks += st.n_esdf_blocks;
  w.effective_blocks += st.n_effective;
  w.esdf_new_blocks += st.n_esdf_new;
  w.lower_rounds += st.rounds;
  w.dirty_blocks_after_round1 += st.sum_dirty;
  w.pair_exchanges += st.sum_pairs;
  w.compared_blocks += st.cmp_blocks;
  w.reserved[0] += st.n_out;  // ESDF changed blocks
  w.reserved[1] += st.quiet_blocks;  // round-1 blocks skipped by the quiet chain
  E->xr_quiet = st.quiet_blocks;
}

void run_update_esdf(Layer* E, Layer* T, BlockList* updated, const vxm_esdf_config& cfg,
                     BlockList* changed_out) {
  Context* ctx = E->ctx;
  ctx->reset_status();
  esdf_launch(E, T, updated, cfg, changed_out);
  E->stage_meta();
  host_trace_mark("launched");
  host_trace_dev(ctx, "kernels");
  ctx->sync_status(true);
  E->adopt_meta();
  esdf_finish(E, changed_out);
}

static void append_sorted_unique(std::vector<vxm_grid_index>& dst,
                                 const std::vector<vxm_grid_index>& add) {
  dst.insert(dst.end(), add.begin(), add.end());
  auto less = [](const vxm_grid_index& a, const vxm_grid_index& b) {
    return a.x != b.x ? a.x < b.x : (a.y != b.y ? a.y < b.y : a.z < b.z);
  };
  auto eq = [](const vxm_grid_index& a, const vxm_grid_index& b) {
    return a.x == b.x && a.y == b.y && a.z == b.z;
  };
  std::sort(dst.begin(), dst.end(), less);
  dst.erase(std::unique(dst.begin(), dst.end(), eq), dst.end());
}

static std::vector<vxm_grid_index> compact_to_host(Context* ctx, const uint64_t* keys,
                                                   const uint8_t* flags, const uint32_t* n_ptr,
                                                   uint32_t cap) {
  BlockList tmp;
  tmp.ctx = ctx;
  tmp.ensure(std::max<uint32_t>(cap, 1));
  launch_compact_keys(ctx, keys, flags, n_ptr, cap, tmp.keys.as<uint64_t>(), tmp.d_count, nullptr);
  tmp.host_valid = false;
  tmp.host_pending = false;
  return tmp.fetch();
}

__global__ void k_flags_bit(const uint8_t* in, const uint32_t* n_ptr, uint8_t bit, uint8_t* out) {
  const uint32_t n = *n_ptr;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = (in[i] & bit) ? 1 : 0;
}

void run_mark_sites(Layer* E, Layer* T, BlockList* updated, const vxm_esdf_config& cfg,
                    EsdfState* st, std::vector<vxm_grid_index>* changed) {
  Context* ctx = E->ctx;
  const uint32_t epoch = ++ctx->call_epoch;
  ctx->reset_status();
  E->refresh();
  E->note_esdf_source(T);
  E->ensure_capacity(std::min<uint64_t>(
      uint64_t(E->num_blocks) + 7ull * std::max<uint32_t>(updated->count_hint, 1), E->max_blocks));
  EsdfScratch s = esdf_scratch(ctx, updated->count_hint, 0);
  const uint32_t n7 = esdf_mark_phase(E, T, updated, cfg, s, epoch);
  DevBuf bits;
  bits.ensure(n7 + 16);
  const char* names[3] = {"changed", "to_update", "to_clear"};
  std::vector<vxm_grid_index> out[3];
  for (int b = 0; b < 3; ++b) {
    k_flags_bit<<<grid_for(ctx, n7), 256, 0, ctx->stream>>>(s.flags, s.counts + 0, uint8_t(1 << b),
                                                          bits.as<uint8_t>());
    ctx->count_launch();
    out[b] = compact_to_host(ctx, s.eff_keys, bits.as<uint8_t>(), s.counts + 0, n7);
    (void)names;
  }
  bits.release();
  ctx->sync_status();
  E->refresh();
  changed->insert(changed->end(), out[0].begin(), out[0].end());
  append_sorted_unique(st->lists[0], out[1]);
  append_sorted_unique(st->lists[1], out[2]);
  if (ctx->h_status->capacity_error || ctx->h_status->pool_overflow)
    throw Error(VXM_ERR_CAPACITY, "Layer: block capacity exhausted");
}

void esdf_sorted_export(Layer* E, std::vector<uint64_t>* keys, std::vector<int32_t>* slots) {
  Context* ctx = E->ctx;
  const uint32_t n = E->num_blocks;
  keys->resize(n);
  slots->resize(n);
  if (!n) return;
  VXM_CUDA(cudaMemcpyAsync(keys->data(), E->sorted_keys[E->sorted_parity], sizeof(uint64_t) * n,
                           cudaMemcpyDeviceToHost, ctx->stream));
  VXM_CUDA(cudaMemcpyAsync(slots->data(), E->sorted_slots[E->sorted_parity], sizeof(int32_t) * n,
                           cudaMemcpyDeviceToHost, ctx->stream));
  VXM_CUDA(cudaStreamSynchronize(ctx->stream));
}

void run_clear_invalid(Layer* E, const vxm_esdf_config& cfg, EsdfState* st,
                       std::vector<vxm_grid_index>* changed) {
  ++E->esdf_gen;  // k_clear writes blocks
  if (st->lists[1].empty()) return;  // esdf/integrator.cpp:435-437
  Context* ctx = E->ctx;
  E->refresh();
  const uint32_t n_all = E->num_blocks;
  std::vector<uint64_t> ck(st->lists[1].size());
  for (size_t i = 0; i < ck.size(); ++i)
    ck[i] = pack_key(st->lists[1][i].x, st->lists[1][i].y, st->lists[1][i].z);
  DevBuf dck, dflags, dn;
  dck.ensure(sizeof(uint64_t) * ck.size());
  dflags.ensure(n_all + 16);
  dn.ensure(sizeof(uint32_t));
  VXM_CUDA(cudaMemcpyAsync(dck.p, ck.data(), sizeof(uint64_t) * ck.size(), cudaMemcpyHostToDevice,
                           ctx->stream));
  VXM_CUDA(cudaMemcpyAsync(dn.p, &n_all, sizeof n_all, cudaMemcpyHostToDevice, ctx->stream));
  ClearArgs a{};
  a.sorted_keys = E->sorted_keys[E->sorted_parity];
  a.sorted_slots = E->sorted_slots[E->sorted_parity];
  a.n_all = n_all;
  a.clear_keys = dck.as<uint64_t>();
  a.n_clear = uint32_t(ck.size());
  a.radius = int(std::ceil(cfg.max_distance / E->vs / kVPS));
  a.hash = E->hash;
  a.pool = static_cast<uint32_t*>(E->pool[E->cur_host]);
  a.lim = esdf_limits(E, cfg);
  a.flags = dflags.as<uint8_t>();
  if (n_all) {
    k_clear<<<std::max<uint32_t>(1, std::min<uint32_t>(n_all, ctx->sm_count * 8)), 256, 0,
              ctx->stream>>>(a);
    ctx->count_launch();
    check_launch(ctx, "k_clear");
  }
  const auto cleared = compact_to_host(ctx, a.sorted_keys, a.flags, dn.as<uint32_t>(), n_all);
  changed->insert(changed->end(), cleared.begin(), cleared.end());
  append_sorted_unique(st->lists[2], cleared);
}

int run_lower_esdf(Layer* E, EsdfState* st, const vxm_esdf_config& cfg,
                   std::vector<vxm_grid_index>* changed) {
  Context* ctx = E->ctx;
  ctx->reset_status();
  E->refresh();
  // seeds = (to_update U cleared) n has_block — esdf/integrator.cpp:492-503
  std::vector<vxm_grid_index> seeds = st->lists[0];
  append_sorted_unique(seeds, st->lists[2]);
  std::vector<uint64_t> sk(seeds.size());
  for (size_t i = 0; i < seeds.size(); ++i) sk[i] = pack_key(seeds[i].x, seeds[i].y, seeds[i].z);
  const uint32_t ns = uint32_t(sk.size());
  DevBuf dk, dslots, dn;
  dk.ensure(sizeof(uint64_t) * (ns + 1));
  dslots.ensure(sizeof(int32_t) * (ns + 1));
  dn.ensure(sizeof(uint32_t) * 2);
  std::vector<int32_t> slots(ns);
  if (ns) {
    VXM_CUDA(cudaMemcpyAsync(dk.p, sk.data(), sizeof(uint64_t) * ns, cudaMemcpyHostToDevice,
                             ctx->stream));
    k_lookup_slots<<<grid_for(ctx, ns), 256, 0, ctx->stream>>>(dk.as<uint64_t>(), ns, E->hash,
                                                             dslots.as<int32_t>());
    ctx->count_launch();
    VXM_CUDA(cudaMemcpyAsync(slots.data(), dslots.p, sizeof(int32_t) * ns, cudaMemcpyDeviceToHost,
                             ctx->stream));
    VXM_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  std::vector<int32_t> live;
  for (int32_t s : slots)
    if (s >= 0) live.push_back(s);
  const uint32_t nl = uint32_t(live.size());
  if (nl) {
    VXM_CUDA(cudaMemcpyAsync(dslots.p, live.data(), sizeof(int32_t) * nl, cudaMemcpyHostToDevice,
                             ctx->stream));
  }
  VXM_CUDA(cudaMemcpyAsync(dn.p, &nl, sizeof nl, cudaMemcpyHostToDevice, ctx->stream));
  const uint32_t tag = ++ctx->call_epoch;
  ++E->esdf_gen;  // (a seeded lowering writes blocks)
  LowerArgs la = lower_args(E, cfg);
  la.full = 0;
  la.seeds = dslots.as<int32_t>();
  la.n_seeds = dn.as<uint32_t>();
  la.lchg_tag = tag;
  launch_lower(ctx, la, E->num_blocks);
  check_launch(ctx, "k_lower(seeded)");
  const uint32_t n_all = E->num_blocks;
  DevBuf dflags, dnall;
  dflags.ensure(n_all + 16);
  dnall.ensure(sizeof(uint32_t));
  VXM_CUDA(cudaMemcpyAsync(dnall.p, &n_all, sizeof n_all, cudaMemcpyHostToDevice, ctx->stream));
  if (n_all) {
    k_flag_tag<<<grid_for(ctx, n_all), 256, 0, ctx->stream>>>(
        E->sorted_slots[E->sorted_parity], n_all, E->stamp_lchg, tag, dflags.as<uint8_t>());
    ctx->count_launch();
  }
  const auto ch = compact_to_host(ctx, E->sorted_keys[E->sorted_parity], dflags.as<uint8_t>(),
                                  dnall.as<uint32_t>(), n_all);
  changed->insert(changed->end(), ch.begin(), ch.end());
  ctx->sync_status();
  E->refresh();
  return int(ctx->h_status->rounds);
}

// Allocation of an arbitrary key list (layer_write_blocks): sorted unique keys
// on device -> slots (new blocks registered in the ESDF side structures).
void alloc_key_list(Layer* L, BlockList* keys, int32_t* d_slots_out) {
  Context* ctx = L->ctx;
  const uint32_t n = std::max<uint32_t>(keys->count_hint, 1);
  L->ensure_capacity(std::min<uint64_t>(uint64_t(L->num_blocks) + n, L->max_blocks));
  EsdfScratch s = esdf_scratch(ctx, n, 0);
  AllocListArgs al{};
  al.keys = keys->keys.as<uint64_t>();
  al.n_ptr = keys->d_count;
  al.hash = L->hash;
  al.slot_keys = L->slot_keys;
  al.meta = L->meta;
  al.capacity = L->capacity;
  al.max_blocks = L->max_blocks;
  al.slots_out = d_slots_out;
  al.new_keys = s.new_keys;
  al.new_slots = s.new_slots;
  al.n_new_out = s.counts + 1;
  al.n_old_out = s.counts + 2;
  al.stamp_new = L->type == VXM_LAYER_ESDF ? L->stamp_new : nullptr;
  al.call_epoch = ++ctx->call_epoch;
  al.status = ctx->status_w();
  const ScanTiles st = ctx->next_scan(ceil_div(n, 256));
  k_alloc_list<<<grid_for(ctx, n, 4), 256, 0, ctx->stream>>>(al, st);
  ctx->count_launch();
  if (L->type == VXM_LAYER_ESDF) {
    k_nbr_update<<<grid_for(ctx, 6ull * n), 256, 0, ctx->stream>>>(s.new_keys, s.new_slots,
                                                                  s.counts + 1, L->hash, L->nbr);
    const int sp = L->sorted_parity;
    k_merge_sorted<<<grid_for(ctx, uint64_t(L->num_blocks) + n), 256, 0, ctx->stream>>>(
        L->sorted_keys[sp], L->sorted_slots[sp], s.counts + 2, s.new_keys, s.new_slots,
        s.counts + 1, L->sorted_keys[1 - sp], L->sorted_slots[1 - sp]);
    L->sorted_parity = 1 - sp;
    ctx->count_launch(2);
  }
  check_launch(ctx, "alloc_key_list");
}

}  // namespace vxm
