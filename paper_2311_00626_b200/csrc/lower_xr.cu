// Cross-round dataflow lowering for update_esdf (esdf/integrator.cpp:352-413,
// 488-565): the same schedule as k_lower3 (esdf.cu) without a grid barrier
// between rounds.
//
// k_lower3 ends every round with a grid barrier (the next dirty list must be
// complete).  Here a round's end is a counter: every pair item of round R
// increments done[R]; the item that completes the round zeroes the counters
// of round R + 2 and publishes last_done = R.  Meanwhile sweep groups already
// take round R + 1's dirty blocks as the pairs of round R append them (list
// entries carry their round's epoch, so a slot is read only once written);
// a block's sweep of round R + 1 waits only for the pairs of round R that
// touch it (the reference's order: those pairs are the only writers of the
// block since its last sweep).  Pair items of round R + 1 are taken once
// round R is complete (their enumeration needs the final dirty list).  Every
// wait is on an item some running warp has already claimed, and waits point
// from round R + 1 to round R or from one axis to a lower one, so there is no
// cycle.  The result is bit-identical to the barrier schedule.
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "esdf_lower.cuh"

namespace cg = cooperative_groups;

// Line masks (which lines a round's pairs touched, so a sweep skips idempotent
// lines): a pair stores the 64-bit masks of the face voxels it changed next to
// its stamp, before the stamp's release — plain stores ordered by the release
// it pays anyway, no atomics — and a sweep derives its lines from the faces of
// the pairs it waits for.

namespace vxm {

namespace {

constexpr int kRingCnt = 0, kRingSwc = 4, kRingPc = 8, kRingDone = 12, kRingLast = 16;
// Every ring counter sits on its own 256-byte line (kRingStride words): the
// counters are polled by every idle warp between rounds, and co-located
// counters would serialise the critical atomics behind those polls in one
// L2 slice.
__device__ __forceinline__ uint32_t* RG(uint32_t* ring, int i) { return ring + i * kRingStride; }

// Lines of a block through the voxels of one face (bit i0 + 8 j0 of F) that a
// pair along `axis` changed; `face` is the face's coordinate (0 or 7).  The
// same bits line_bits() sets voxel by voxel.
__device__ inline void face_lines(unsigned long long F, int axis, int face, unsigned long long m[3]) {
  uint32_t rows = 0, cols = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const uint32_t byte = uint32_t(F >> (8 * j)) & 0xffu;
    rows |= uint32_t(byte != 0u) << j;
    cols |= byte;
  }
  if (axis == 0) {         // (i0, j0) = (y, z), x = face
    m[0] |= F;
    m[1] |= spread8(rows) << face;
    m[2] |= spread8(cols) << face;
  } else if (axis == 1) {  // (i0, j0) = (x, z), y = face
    m[0] |= spread8(rows) << face;
    m[1] |= F;
    m[2] |= (unsigned long long)cols << (8 * face);
  } else {                 // (i0, j0) = (x, y), z = face
    m[0] |= (unsigned long long)rows << (8 * face);
    m[1] |= (unsigned long long)cols << (8 * face);
    m[2] |= F;
  }
}

// VXM_TRACE_XR phase stamps of round R < 24: trace[128 + 16 R + k], k = 0 first
// sweep claimed (min), 1 last sweep released, 2 first pair claimed (min),
// 3 / 4 / 5 last x / y / z pair released, 6 / 7 sum / count of sweep durations,
// 8 / 9 / 10 / 11 sums of the sweeps' dependency wait / load + stage / sweep /
// store + release, 12 / 13 / 14 sums of the x / y / z pairs' work after their
// waits, 15 count of non-identity pairs.
__device__ inline unsigned long long gtime() {
  unsigned long long tm;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tm));
  return tm;
}
__device__ inline void tr_max(unsigned long long* tr, uint32_t R, int k, unsigned long long v) {
  if (tr && R < 24) atomicMax(tr + 128 + 16 * R + k, v);
}
__device__ inline void tr_min(unsigned long long* tr, uint32_t R, int k, unsigned long long v) {
  if (tr && R < 24) atomicMax(tr + 128 + 16 * R + k, ~v);
}
__device__ inline void tr_add(unsigned long long* tr, uint32_t R, int k, unsigned long long v) {
  if (tr && R < 24) atomicAdd(tr + 128 + 16 * R + k, v);
}

// Round 1's compact pair lists (x, y, z), capacity entries each.
__device__ inline int32_t* r1_pairs(const LowerArgs& a, int axis) {
  return a.r1_list + size_t(axis) * a.capacity;
}

// Maps above this many blocks precompute round 1's pair lists
// (VXM_XR_R1_COMPACT_MIN overrides, for the variant tests).
constexpr uint32_t kR1CompactMin = 32 * 1024;

__device__ inline unsigned long long ld_relaxed64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// A FASTONLY kernel met a block outside the compact format: the host's
// eligibility rule (launch_lower_xr) was wrong — reported as an internal
// error (VXM_ERR_INTERNAL via the watchdog word), never a silent result.
__device__ inline void format_violation(const LowerArgs& a, int t) {
  if (t == 0 && atomicExch(&a.status->watchdog, 1u) == 0u) a.status->pad3[0] = 50u;
}

}  // namespace

// MINB resident CTAs per SM: 2 (124 registers, no spills) for latency-bound
// maps, 3 (80 registers, small spills, +50 % sweep groups) for throughput-bound
// large maps — measured: C2 -7 % with 3, C4 / C5 +9 % / +11 % with 3.
template <int MINB, bool TRACE, bool FASTONLY>
__global__ void __launch_bounds__(kL3Threads, MINB) k_lower_xr(LowerArgs a) {
  pdl_wait();  // see launch_pdl
  pdl_trigger();
  // VXM_TRACE_XR instrumentation only in the TRACE instantiations (the
  // production kernels carry none of it)
  unsigned long long* const trace = TRACE ? a.trace : nullptr;
  cg::grid_group grid = cg::this_grid();
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
  const bool lower = !failed && a.status->any_update != 0;
  uint32_t* const pcur = a.pool[cur];
  uint32_t* const pnxt = a.pool[cur ^ 1u];
  uint32_t* const work = pnxt;
  const Limits lim = a.lim;
  uint32_t* const ring = a.ring;
  // "round R complete": polled relaxed (an acquire per poll would invalidate L1
  // each time), then one acquire once seen
  const uint32_t* const last_rep = RG(ring, kRingLast);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    for (int q = 1; q <= 2; ++q) {  // rounds 1 and 2; later rounds are zeroed by round R - 2
      *RG(ring, kRingCnt + q) = 0u;
      *RG(ring, kRingSwc + q) = *RG(ring, kRingPc + q) = *RG(ring, kRingDone + q) = 0u;
    }
    *RG(ring, kRingLast) = 0u;
  }
  // round-1 split by site_any (as k_lower3), and each block's static "a site
  // nearby" bits for round 1's pairs: after reset_parented only sites give,
  // and a block can take parents in round 1's x phase only from its x
  // neighbours, in its y phase only from blocks whose x-neighbourhood holds a
  // site.  So a round-1 y pair is certainly the identity when neither block
  // has a site within +-x (bit 0), a z pair when neither has one in its 3 x 3
  // (x, y) neighbourhood (bit 1); such items are released without any wait.
  // (only on large maps: on a small one — C2, 9k blocks — the extra pass and
  // grid barrier cost more than the claims they save)
  // (the 2-CTA instantiation, for maps of at most kXrWideBlocks, never
  // plans: compiled out of it)
  const bool r1c = MINB == 3 && n_blocks > a.r1_compact_min;
  if (lower && r1c) {
    auto sa = [&](int32_t c) -> uint32_t { return c >= 0 ? uint32_t(a.site_any[c] != 0) : 0u; };
    auto near_x = [&](int32_t c) -> uint32_t {
      if (c < 0) return 0u;
      return sa(c) | sa(__ldg(a.nbr + size_t(c) * 6 + 0)) | sa(__ldg(a.nbr + size_t(c) * 6 + 1));
    };
    for (uint32_t b = blockIdx.x * kL3Threads + threadIdx.x; b < n_blocks; b += gridDim.x * kL3Threads) {
      const uint32_t nx = near_x(int32_t(b));
      const uint32_t nxy = nx | near_x(__ldg(a.nbr + size_t(b) * 6 + 2)) | near_x(__ldg(a.nbr + size_t(b) * 6 + 3));
      a.site_near[b] = uint8_t(nx | (nxy << 1));
    }
    grid.sync();
    // Round 1's pair items: the certainly-identity pairs (b, b + axis) are
    // released here, before any sweep (their readers see below); the others
    // go to one compact list per axis, so round 1 claims only those — on a
    // mostly site-free map (C5: 262k blocks, ~7k with sites) that removes
    // most of the 3 x N claims that would otherwise serialise on one counter.
    const uint32_t ep1 = base_epoch + 1u;
    for (uint32_t b0 = blockIdx.x * kL3Threads + (threadIdx.x & ~31u); b0 < n_blocks;
         b0 += gridDim.x * kL3Threads) {
      const uint32_t b = b0 + lane;
      const bool in = b < n_blocks;
#pragma unroll
      for (int axis = 0; axis < 3; ++axis) {
        const int32_t hi = in ? __ldg(a.nbr + size_t(b) * 6 + 2 * axis) : -1;
        bool keep = false;
        if (hi >= 0) {
          const bool ident = axis == 0 ? (a.site_any[b] == 0 && a.site_any[hi] == 0)
                                       : ((a.site_near[b] | a.site_near[hi]) & (axis == 1 ? 1u : 2u)) == 0u;
          if (ident) a.stamp_pair[axis][b] = ep1;
          keep = !ident;
        }
        const uint32_t mk = __ballot_sync(0xffffffffu, keep);
        uint32_t base = 0;
        if (lane == 0 && mk) base = atomicAdd(a.r1 + 5 + axis, __popc(mk));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (keep) r1_pairs(a, axis)[base + __popc(mk & ((1u << lane) - 1u))] = int32_t(b);
      }
    }
  }
  if (lower) {
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
  if (trace && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long tm;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tm));
    trace[0] = tm;
  }
  uint32_t n_pairs = 0, n_cmp = 0, rounds = 0, r1_mine = 0, n_quiet = 0;
  // One round of the loop; round 1 and the later rounds are separate
  // instantiations (r1 a compile-time constant in each), so the steady-state
  // loop carries none of round 1's code.  Returns false once the round's
  // dirty list is empty.
  auto round_body = [&](const uint32_t R, auto r1_tag) -> bool {
      constexpr bool r1 = decltype(r1_tag)::value;
      const uint32_t ep = base_epoch + R, ep_next = ep + 1;
      const int cp = int(R & 1u), np = cp ^ 1;
      const int q4 = int(R & 3u), q4n = int((R + 1u) & 3u);
      // ---- sweeps of round R (esdf/integrator.cpp:509-513) -------------------
      if (r1) {
        const uint32_t n_grp = *((volatile uint32_t*)(a.r1 + 0));
        while (true) {
          if (t == 0) G.bcast = atomicAdd(a.r1 + 2, 1u);
          group_sync(bar);
          const uint32_t i = G.bcast;
          if (i >= n_grp) break;
          const int32_t s = __ldcg(a.list[1] + i);
          if (t == 0) {
            G.mask[0][0] = G.mask[1][0] = G.mask[2][0] = ~0ull;
            G.mask[0][1] = G.mask[1][1] = G.mask[2][1] = 0ull;
          }
          RawBlock rb;
          bool any_site, fast;
          unsigned long long tm0 = 0, tm1 = 0;
          if (trace) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tm0));
          load_raw3(rb, pcur + size_t(s) * 1536, t, bar, lim, true, &any_site, &fast);
          if (FASTONLY && !fast) format_violation(a, t);
          if (!any_site) {
            raw_store(rb, work + size_t(s) * 1536, t);
          } else {
            stage_block3<FASTONLY>(G, rb, t, bar, lim, fast);
            int passes = 0;
            if (trace) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tm1));
            sweep_block3<FASTONLY>(G, t, bar, lim, &passes);
            if (trace && t == 0) {  // VXM_TRACE_XR: round-1 sweep statistics
              unsigned long long tm2;
              asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tm2));
              atomicAdd(trace + 54, tm1 - tm0);
              atomicAdd(trace + 55, tm2 - tm1);
              atomicAdd(trace + 56, (unsigned long long)passes);
              atomicAdd(trace + 57, 1ull);
            }
            store_block3<FASTONLY>(G, work + size_t(s) * 1536, t);
          }
          group_sync(bar);
          if (t == 0) {
            st_release(a.stamp_swept + s, ep);
            ++r1_mine;
          }
        }
        // round 1 completes only after every sweep / copy: counted per group
        if (t == 0 && r1_mine) {
          atom_add_release(a.r1 + 4, r1_mine);  // the group's block writes before the count
        }
        r1_mine = 0;
        const uint32_t n_ns = *((volatile uint32_t*)(a.r1 + 1));
        // site-free blocks: reset + copy, one warp each.  A quiet block
        // (Layer::stamp_quiet: the previous update left it untouched, its reset
        // the identity, the same bytes in both pools, and neither mark nor
        // allocation touched it since) is already its own round-1 result in
        // the work pool: no read, no copy.  On a large map with a quiet chain a
        // warp claims 32 blocks and its lanes decide them together when most
        // blocks were quiet in the previous update (C3's far field); otherwise
        // 2 at a time (the copies spread over all warps).
        const uint32_t chunk = (MINB >= 3 && a.quiet_dense != 0u) ? 32u : 2u;
        while (true) {
          uint32_t j0 = 0;
          if (lane == 0) j0 = atomicAdd(a.r1 + 3, chunk);
          j0 = __shfl_sync(0xffffffffu, j0, 0);
          if (j0 >= n_ns) break;
          const uint32_t jl = j0 + uint32_t(lane);
          const bool in = uint32_t(lane) < chunk && jl < n_ns;
          const int32_t s = in ? __ldcg(a.list[1] + (n_blocks - 1u - jl)) : 0;
          const bool quiet = in && a.quiet_epoch != 0u && a.stamp_quiet[s] == a.quiet_epoch &&
                             a.stamp_mark[s] != a.call_epoch && a.stamp_new[s] != a.call_epoch;
          if (quiet) {
            a.stamp_r1same[s] = a.call_epoch;
            st_release(a.stamp_swept + s, ep);
          }
          for (unsigned m = __ballot_sync(0xffffffffu, in && !quiet); m; m &= m - 1u) {
            const int32_t sc = __shfl_sync(0xffffffffu, s, __ffs(m) - 1);
            const bool reset_chg = warp_reset_copy(pcur + size_t(sc) * 1536, work + size_t(sc) * 1536, lane, lim);
            __syncwarp();
            if (lane == 0) {
              // unchanged by round 1: if no later round writes it, the changed-set
              // compare can skip it (every later writer marks it dirty)
              if (!reset_chg) a.stamp_r1same[sc] = a.call_epoch;
              st_release(a.stamp_swept + sc, ep);
            }
          }
          const uint32_t nq = __popc(__ballot_sync(0xffffffffu, quiet));
          const uint32_t nin = __popc(__ballot_sync(0xffffffffu, in));
          if (lane == 0) {
            n_quiet += nq;
            r1_mine += nin;
          }
        }
        __syncwarp();  // every lane's releases before the warp's count
        if (lane == 0 && r1_mine) {  // (per warp)
          atom_add_release(a.r1 + 4, r1_mine);
        }
        if (trace && lane == 0) {  // VXM_TRACE_XR: end of the round-1 sweeps / copies
          unsigned long long tm;
          asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tm));
          atomicMax(trace + 60, tm);
        }
      } else {
        const unsigned long long* dl = a.dlist[cp];
        while (true) {
          if (t == 0) {
            // claim the next dirty block of round R; its slot is written by the
            // round R - 1 pair that changed it (epoch-tagged), or the list ends
            // once round R - 1 is complete
            const uint32_t i = atomicAdd(RG(ring, kRingSwc + q4), 1u);
            int32_t s = -1;
            for (uint32_t it = 0; i < a.capacity; ++it) {  // (a round never lists more)
              const unsigned long long e = ld_relaxed64(dl + i);
              if (uint32_t(e >> 32) == ep) {
                s = int32_t(uint32_t(e));
                break;
              }
              if (ld_relaxed(last_rep) + 1u >= R && ld_acquire(last_rep) + 1u >= R &&
                  i >= *((volatile uint32_t*)(RG(ring, kRingCnt + q4)))) {
                const unsigned long long e2 = ld_relaxed64(dl + i);  // (written before the count)
                if (uint32_t(e2 >> 32) == ep) s = int32_t(uint32_t(e2));
                break;
              }
              if (it > (1u << 24)) {  // a lost producer is a bug, never a hang
                if (atomicExch(&a.status->watchdog, 1u) == 0u) a.status->pad3[0] = 40u;
                break;
              }
              __nanosleep(32);
            }
            G.bcast = uint32_t(s);
          }
          group_sync(bar);
          const int32_t s = int32_t(G.bcast);
          if (s < 0) break;
          unsigned long long tsw0 = 0;
          if (trace && t == 0) {
            tsw0 = gtime();
            tr_min(trace, R, 0, tsw0);
          }
          // the block's round R - 1 pairs (the reference's only writers of it since
          // its last sweep) must be complete: lanes 0-5 of the group's first warp
          // wait; then the block's load is issued first and the faces the pairs
          // changed (the lines to sweep first) are read while it is in flight
          uint32_t wv = 0;
          int32_t wlo = -1;
          if (t < 6) {
            const int q = t >> 1;
            const uint32_t epp = ep - 1;  // round R - 1
            const bool r1p = R - 1 == 1;
            const bool s_dirty = r1p || __ldcg(a.stamp_dirty[np] + s) == epp;
            const int32_t c = __ldg(a.nbr + size_t(s) * 6 + t);  // +q (even t) / -q (odd t)
            if (c >= 0 && (s_dirty || __ldcg(a.stamp_dirty[np] + c) == epp)) {
              const bool s_lo = (t & 1) == 0;  // pair (s, c) or (c, s)
              wlo = s_lo ? s : c;
              wv = wait_stamp(a.stamp_pair[q] + wlo, epp, &a.status->watchdog, 30u + q, wlo);
            }
          }
          group_sync(bar);  // every wait done before the voxels are read
          unsigned long long tsa = 0, tsb = 0, tsc = 0;
          if (trace && t == 0) tsa = gtime();
          RawBlock rb;
          raw_load(rb, work + size_t(s) * 1536, t);
          if (t < 32) {
            unsigned long long m[3] = {0, 0, 0};
            if (t < 6 && wlo >= 0) {
              const int q = t >> 1;
              const bool s_lo = (t & 1) == 0;
              if (wv & (s_lo ? kStampLoChg : kStampHiChg))
                face_lines(__ldcg(a.pair_face[q] + 2 * size_t(wlo) + (s_lo ? 0 : 1)), q, s_lo ? 7 : 0, m);
            }
            unsigned long long m0 = warp_or64(m[0]), m1 = warp_or64(m[1]), m2 = warp_or64(m[2]);
            if (t == 0) {
              G.mask[0][0] = m0;
              G.mask[1][0] = m1;
              G.mask[2][0] = m2;
              G.mask[0][1] = G.mask[1][1] = G.mask[2][1] = 0ull;
            }
          }
          bool any_site, fast;
          raw_check3(rb, t, bar, lim, false, &any_site, &fast);  // (its barriers publish the masks)
          if (FASTONLY && !fast) format_violation(a, t);
          stage_block3<FASTONLY>(G, rb, t, bar, lim, fast);
          if (trace && t == 0) tsb = gtime();
          const bool sw_chg = sweep_block3<FASTONLY>(G, t, bar, lim);
          if (trace && t == 0) tsc = gtime();
          if (sw_chg) store_block3<FASTONLY>(G, work + size_t(s) * 1536, t);
          group_sync(bar);  // the group's stores before the release of its sweep stamp
          if (t == 0) st_release(a.stamp_swept + s, ep);
          if (trace && t == 0) {
            const unsigned long long tsw1 = gtime();
            tr_max(trace, R, 1, tsw1);
            tr_add(trace, R, 6, tsw1 - tsw0);
            tr_add(trace, R, 7, 1ull);
            tr_add(trace, R, 8, tsa - tsw0);
            tr_add(trace, R, 9, tsb - tsa);
            tr_add(trace, R, 10, tsc - tsb);
            tr_add(trace, R, 11, tsw1 - tsc);
          }
        }
      }
      // ---- border phase of round R (esdf/integrator.cpp:517-559) ----------------
      if (!r1) {  // enumeration needs the final round-R list: round R - 1 complete
        for (uint32_t it = 0; ld_relaxed(last_rep) + 1u < R; ++it) {
          if (it > (1u << 24)) {
            if (atomicExch(&a.status->watchdog, 1u) == 0u) a.status->pad3[0] = 41u;
            break;
          }
          __nanosleep(32);
        }
      }
      if (!r1) (void)ld_acquire(last_rep);  // the round's list and counts are visible
      const uint32_t n_dirty = r1 ? n_blocks : *((volatile uint32_t*)(RG(ring, kRingCnt + q4)));
      if (n_dirty == 0) return false;  // while (!dirty.empty()) — esdf/integrator.cpp:506
      rounds = R;
      const unsigned long long* dl = a.dlist[cp];
      auto dirty_at = [&](uint32_t i) -> int32_t { return r1 ? int32_t(i) : int32_t(uint32_t(__ldcg(dl + i))); };
      auto is_dirty = [&](int32_t b) { return r1 || __ldcg(a.stamp_dirty[cp] + b) == ep; };
      const uint32_t sides = r1 ? 1u : 2u;
      const uint32_t per_axis = sides * n_dirty;
      // round 1 on a large map: the compact lists (x, y, z) of the pairs that
      // may change something
      const bool r1l = r1 && r1c;
      const uint32_t c1x = r1l ? *((volatile uint32_t*)(a.r1 + 5)) : 0u;
      const uint32_t c1y = r1l ? *((volatile uint32_t*)(a.r1 + 6)) : 0u;
      const uint32_t c1z = r1l ? *((volatile uint32_t*)(a.r1 + 7)) : 0u;
      const uint32_t n_items = r1l ? c1x + c1y + c1z : 3u * per_axis;
      uint32_t my_done = 0;
      // one item per claim: a warp blocked on a dependency must not hold later
      // items (measured on C2: chunks of 4 / 16 in round 1 cost 2 % / 34 %;
      // prefetching the next claim during the current item costs 4 %)
      while (true) {
        uint32_t wi = 0;
        if (lane == 0) wi = atomicAdd(RG(ring, kRingPc + q4), 1u);
        wi = __shfl_sync(0xffffffffu, wi, 0);
        if (wi >= n_items) break;
        if (trace && lane == 0 && wi == 0) tr_min(trace, R, 2, gtime());
        int axis;
        uint32_t rest;
        if (r1l) {
          axis = wi < c1x ? 0 : (wi < c1x + c1y ? 1 : 2);
          rest = wi - (axis == 0 ? 0u : (axis == 1 ? c1x : c1x + c1y));
        } else {
          axis = int(wi / per_axis);
          rest = wi - uint32_t(axis) * per_axis;
        }
        const uint32_t i = r1 ? rest : rest >> 1;
        const int side = r1 ? 0 : int(rest & 1u);
        const int32_t d = r1l ? __ldcg(r1_pairs(a, axis) + i) : dirty_at(i);
        int32_t lo = -1, hi = -1;
        if (side == 0) {
          hi = __ldg(a.nbr + size_t(d) * 6 + 2 * axis);  // d + axis
          lo = d;
        } else {
          lo = __ldg(a.nbr + size_t(d) * 6 + 2 * axis + 1);  // d - axis
          hi = d;
        }
        // round 1: whether a side can give is known before any wait (after the
        // reset only sites give); the loads are issued ahead of the waits
        const bool site_lo = r1 && lo >= 0 && a.site_any[lo] != 0;
        const bool site_hi = r1 && hi >= 0 && a.site_any[hi] != 0;
        // Round 1's certainly-identity pairs are released without waiting (on
        // a large map before the sweeps, from the static site bits; on a small
        // one the x pairs here).  Their readers: the pairs of later axes, which
        // also wait for the blocks' sweeps and their non-identity x / y pairs
        // — the only writers; round-2 sweeps, of blocks some non-identity pair
        // changed; round-2 pairs, which start once round 1 is complete — and
        // round 1 completes only after every round-1 sweep and copy.
        if (lo >= 0 && hi >= 0 && r1 && !r1c && axis == 0 && !site_lo && !site_hi) {
          if (lane == 0) st_release(a.stamp_pair[0] + lo, ep);
        } else if (lo >= 0 && hi >= 0) {
          // every lane's dirty-stamp / neighbour loads first, all in flight
          // together: lanes 0 / 1 the pair's blocks (their sweeps), lanes 2.. the
          // lower-axis pairs through its faces, lower block c, upper block n
          // (one neighbour look-up: the other block is the face's own)
          bool own_dirty = false;
          int32_t wc = -1;
          const int q = (lane - 2) >> 2;
          const bool b_is_hi = ((lane - 2) & 1) == 0;
          if (lane < 2) {
            own_dirty = is_dirty(lane == 0 ? lo : hi);
          } else if (lane < 2 + 4 * axis) {
            const int32_t b = ((lane - 2) & 2) ? hi : lo;
            const int32_t o = __ldg(a.nbr + size_t(b) * 6 + 2 * q + (b_is_hi ? 1 : 0));
            const int32_t c = b_is_hi ? o : b, n = b_is_hi ? b : o;
            if (o >= 0) {
              const bool dc = is_dirty(c), dn = is_dirty(n);
              if (dc || dn) wc = c;
            }
          }
          // side 1 with a dirty lower block: lo's side-0 item has this pair
          const bool dup = side == 1 && __shfl_sync(0xffffffffu, own_dirty, 0);
          if (!dup) {
            bool dep_chg = false;
            if (lane < 2) {
              const int32_t b = lane == 0 ? lo : hi;
              if (own_dirty) wait_stamp(a.stamp_swept + b, ep, &a.status->watchdog, 10u + axis, b);
            } else if (wc >= 0) {
              const uint32_t v = wait_stamp(a.stamp_pair[q] + wc, ep, &a.status->watchdog, 20u + 10u * q + axis, wc);
              dep_chg = (v & (b_is_hi ? kStampHiChg : kStampLoChg)) != 0u;
            }
            const uint32_t chg_mask = __ballot_sync(0xffffffffu, dep_chg);
            __syncwarp();
            const unsigned long long tp0 = trace ? gtime() : 0ull;
            bool skip = false;
            if (r1) {  // no giver on either face: the pair is the identity (k_lower3)
              constexpr uint32_t lo_lanes = 0x0ccu, hi_lanes = 0x330u;
              const bool g_lo = site_lo || (chg_mask & lo_lanes) != 0u;
              const bool g_hi = site_hi || (chg_mask & hi_lanes) != 0u;
              skip = !g_lo && !g_hi;
            }
            if (skip) {
              if (lane == 0) st_release(a.stamp_pair[axis] + lo, ep);
            } else {
              const int dx = axis == 0, dy = axis == 1, dz = axis == 2;
              // the faces this pair changes, bit = face position lane + 32 k
              unsigned long long flo = 0, fhi = 0;
              // both face positions of the lane are loaded before any store (the
              // four voxels are distinct): one L2 round trip on the hop, not two
              int la[2], lb[2];
              EV va[2], vb[2];
  #pragma unroll
              for (int k = 0; k < 2; ++k) {
                const int f = lane + 32 * k, i0 = f & 7, j0 = f >> 3;
                int ax, ay, az, bx, by, bz;
                if (axis == 0) { ax = 7; ay = i0; az = j0; bx = 0; by = i0; bz = j0; }
                else if (axis == 1) { ax = i0; ay = 7; az = j0; bx = i0; by = 0; bz = j0; }
                else { ax = i0; ay = j0; az = 7; bx = i0; by = j0; bz = 0; }
                la[k] = ax + 8 * ay + 64 * az;
                lb[k] = bx + 8 * by + 64 * bz;
                va[k] = load_voxel(work, lo, la[k]);
                vb[k] = load_voxel(work, hi, lb[k]);
              }
  #pragma unroll
              for (int k = 0; k < 2; ++k) {
                const bool cb = relax(vb[k], va[k], dx, dy, dz, lim);     // exchange_pair :158
                const bool ca = relax(va[k], vb[k], -dx, -dy, -dz, lim);  // :159
                if (cb) store_voxel(work, hi, lb[k], vb[k]);
                if (ca) store_voxel(work, lo, la[k], va[k]);
                flo |= (unsigned long long)__ballot_sync(0xffffffffu, ca) << (32 * k);
                fhi |= (unsigned long long)__ballot_sync(0xffffffffu, cb) << (32 * k);
              }
              ++n_pairs;
              const bool ac = flo != 0ull, bc = fhi != 0ull;
              const int32_t who[2] = {lo, hi};
              const bool chg[2] = {ac, bc};
              if (lane == 0) {  // the changed faces, published by the release below
                if (ac) a.pair_face[axis][2 * size_t(lo)] = flo;
                if (bc) a.pair_face[axis][2 * size_t(lo) + 1] = fhi;
              }
              __syncwarp();
              if (lane == 0)
                st_release(a.stamp_pair[axis] + lo, ep | (ac ? kStampLoChg : 0u) | (bc ? kStampHiChg : 0u));
              if (trace && lane == 0) {
                tr_add(trace, R, 12 + axis, gtime() - tp0);
                tr_add(trace, R, 15, 1ull);
              }
              if (lane == 0) {
  #pragma unroll
                for (int qq = 0; qq < 2; ++qq) {
                  if (!chg[qq]) continue;
                  if (atomicMax(a.stamp_dirty[np] + who[qq], ep_next) < ep_next) {
                    const uint32_t slot = atomicAdd(RG(ring, kRingCnt + q4n), 1u);
                    *(volatile unsigned long long*)(a.dlist[np] + slot) =
                        (unsigned long long)ep_next << 32 | uint32_t(who[qq]);
                  }
                }
              }
            }
          }  // !dup
        }
        if (trace && lane == 0) tr_max(trace, R, 3 + axis, gtime());
        ++my_done;
      }
      // round accounting, one atomic per warp: the warp whose items complete
      // round R publishes it (every item this warp claimed is done here)
      if (lane == 0 && my_done) {
        // release: this warp's items before the count; acquire: the warp that
        // completes the round sees every item (the counter's release sequence)
        const uint32_t done = atom_add_acq_rel(RG(ring, kRingDone + q4), my_done) + my_done;
        if (done == n_items) {
          if (R == 1) {  // and every round-1 sweep / copy (see r1_ident)
            for (uint32_t it = 0; ld_acquire(a.r1 + 4) < n_blocks; ++it) {
              if (it > (1u << 24)) {
                if (atomicExch(&a.status->watchdog, 1u) == 0u) a.status->pad3[0] = 42u;
                break;
              }
              __nanosleep(64);
            }
          }
          const int q4nn = int((R + 2u) & 3u);
          *RG(ring, kRingCnt + q4nn) = 0u;
          *RG(ring, kRingSwc + q4nn) = *RG(ring, kRingPc + q4nn) = *RG(ring, kRingDone + q4nn) = 0u;
          if (R > 1) a.status->sum_dirty += n_dirty;
          if (trace && R < 54) {  // VXM_TRACE_XR: round completion times
            unsigned long long tm;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tm));
            trace[R] = tm;
            trace[64 + R] = n_dirty;
          }
          st_release(RG(ring, kRingLast), R);  // (orders the zeroing above too)
        }
      }
      // the next round's sweeps re-form the groups (both warps)
      group_sync(bar);
      return true;
  };
  if (lower && n_blocks > 0 && round_body(1u, std::true_type{}))
    for (uint32_t R = 2; round_body(R, std::false_type{}); ++R) {
    }
  grid.sync();
  if (trace && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long tm;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tm));
    trace[62] = tm;
  }
  // ---- changed set of update_esdf (esdf/integrator.cpp:403-411) ------------------
  // Each CTA compares a contiguous chunk of the sorted order (one warp per
  // block); with out_keys the CTA then writes its changed keys at its prefix
  // over the CTAs' counts — the ordered compaction, without another launch.
  __shared__ uint32_t s_cnt, s_pre, s_wsum[kL3Threads / 32];
  const uint32_t chunk = (n_blocks + gridDim.x - 1) / gridDim.x;
  const uint32_t k0 = min(n_blocks, blockIdx.x * chunk), k1 = min(n_blocks, k0 + chunk);
  const int warp_in_cta = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_cnt = 0u;
  __syncthreads();
  // The per-block decisions from stamps are lane-parallel (32 blocks of the
  // chunk per warp at once: on a large map most blocks are decided by their
  // stamps, and one warp per block made that a chain of dependent L2 trips per
  // block); the blocks that need their bytes compared are then compared one
  // after the other by the whole warp.
  // (block k0 + w + 8 (lane + 32 i) to warp w: the CTA's warps share even a
  // short chunk)
  constexpr uint32_t kW = kL3Threads / 32;
  for (uint32_t kb = k0 + uint32_t(warp_in_cta); kb < k1; kb += kW * 32u) {
    const uint32_t k = kb + kW * uint32_t(lane);
    const bool in = k < k1;
    const int32_t s = in ? a.sorted_slots[k] : 0;
    bool ch = false, need = false;
    if (in) {
      ch = a.stamp_new[s] == a.call_epoch || a.stamp_mark[s] == a.call_epoch;
      if (!ch && lower) {
        // a site-free block that round 1 copied unchanged and no later round
        // wrote (every pair or sweep write after round 1 lists the block dirty,
        // stamping it with an epoch of this launch above round 1's) is
        // byte-identical — and quiet for the next update
        const bool late = a.stamp_dirty[0][s] > base_epoch + 1u || a.stamp_dirty[1][s] > base_epoch + 1u;
        if (!late && a.stamp_r1same[s] == a.call_epoch) a.stamp_quiet[s] = a.call_epoch;
        else need = true;
      }
    }
    for (unsigned m = __ballot_sync(0xffffffffu, need); m; m &= m - 1u) {
      const int src = __ffs(m) - 1;
      const int32_t sc = __shfl_sync(0xffffffffu, s, src);
      const uint4* p0 = reinterpret_cast<const uint4*>(pcur + size_t(sc) * 1536);
      const uint4* p1 = reinterpret_cast<const uint4*>(pnxt + size_t(sc) * 1536);
      bool diff = false;
      // all 24 loads of the lane in flight at once (the phase is latency-bound)
      uint4 x[12], y[12];
#pragma unroll
      for (int q = 0; q < 12; ++q) {
        x[q] = __ldcg(p0 + lane + 32 * q);
        y[q] = __ldcg(p1 + lane + 32 * q);
      }
#pragma unroll
      for (int q = 0; q < 12; ++q)
        diff |= (x[q].x != y[q].x) | (x[q].y != y[q].y) | (x[q].z != y[q].z) | (x[q].w != y[q].w);
      diff = __any_sync(0xffffffffu, diff);
      if (lane == src) ch = diff;
      ++n_cmp;
    }
    if (in) a.out_flags[k] = uint8_t(ch);
    const uint32_t nch = __popc(__ballot_sync(0xffffffffu, in && ch));
    if (lane == 0 && nch) atomicAdd(&s_cnt, nch);
  }
  if (lane == 0 && (n_pairs | n_cmp | n_quiet)) {
    atomicAdd(&a.status->sum_pairs, n_pairs);
    atomicAdd(&a.status->cmp_blocks, n_cmp);
    if (n_quiet) atomicAdd(&a.status->quiet_blocks, n_quiet);
  }
  __syncthreads();
  if (a.out_keys && threadIdx.x == 0) a.cta_cnt[blockIdx.x] = s_cnt;
  if (a.out_keys) {
    grid.sync();
    if (threadIdx.x < 32) {  // prefix over the CTAs before this one
      uint32_t sum = 0;
      for (uint32_t c = lane; c < blockIdx.x; c += 32) sum += __ldcg(a.cta_cnt + c);
      sum = __reduce_add_sync(0xffffffffu, sum);
      if (lane == 0) {
        s_pre = sum;
        if (blockIdx.x == gridDim.x - 1) *a.out_n = sum + s_cnt;
      }
    }
    __syncthreads();
    uint32_t base = s_pre;
    for (uint32_t t0 = k0; t0 < k1; t0 += kL3Threads) {  // this CTA's flags, in order
      const uint32_t k = t0 + threadIdx.x;
      const bool f = k < k1 && a.out_flags[k] != 0;
      const uint32_t m = __ballot_sync(0xffffffffu, f);
      if (lane == 0) s_wsum[warp_in_cta] = __popc(m);
      __syncthreads();
      uint32_t off = base, tile = 0;
      for (int w = 0; w < kL3Threads / 32; ++w) {
        const uint32_t c = s_wsum[w];
        if (w < warp_in_cta) off += c;
        tile += c;
      }
      if (f) a.out_keys[off + __popc(m & ((1u << lane) - 1u))] = a.sorted_keys[k];
      base += tile;
      __syncthreads();
    }
  }
  grid.sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (trace) {
      unsigned long long tm;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tm));
      trace[63] = tm;
      trace[58] = a.r1[0];  // round-1 blocks with sites (swept) / without (copied)
      trace[59] = a.r1[1];
    }
    for (int q = 0; q < 8; ++q) a.r1[q] = 0u;  // zero for the next launch
    a.status->rounds = rounds;
    a.status->n_esdf_blocks = n_blocks;
    a.meta->round_epoch = base_epoch + rounds + 2;
    if (lower) a.meta->cur = cur ^ 1u;
  }
}

// Maps above this many blocks use the 3-CTA-per-SM instantiation.
constexpr uint32_t kXrWideBlocks = 24 * 1024;

bool launch_lower_xr(Context* ctx, LowerArgs& la, uint32_t n_blocks_hint) {
  static const bool trace = std::getenv("VXM_TRACE_XR") != nullptr;
  static DevBuf trace_buf;
  if (trace) {
    trace_buf.ensure(512 * sizeof(unsigned long long));
    VXM_CUDA(cudaMemsetAsync(trace_buf.p, 0, 512 * sizeof(unsigned long long), ctx->stream));
    la.trace = trace_buf.as<unsigned long long>();
  }
  static const int wide_mode = [] {  // VXM_XR_WIDE: 0 never, 1 by map size (default), 2 always
    const char* e = std::getenv("VXM_XR_WIDE");
    return e ? std::atoi(e) : 1;
  }();
  const bool wide = wide_mode == 2 || (wide_mode == 1 && n_blocks_hint > kXrWideBlocks);
  static const uint32_t r1_compact_min = [] {
    const char* e = std::getenv("VXM_XR_R1_COMPACT_MIN");
    return e ? uint32_t(std::strtoul(e, nullptr, 10)) : kR1CompactMin;
  }();
  la.r1_compact_min = r1_compact_min;
  // Every block of a layer that only the library has written (mark_sites
  // and the lowering itself) is in the compact sweep format as long as no
  // configuration has had max_sq > kFastOff^2 (parents beyond +-kFastOff,
  // saturation values >= 2^29): then the kernel without the general format
  // runs (C2 k_lower -6 %, C5 -15 %); user-written ESDF data keeps the general
  // kernel for the layer's lifetime.  (VXM_XR_GENERAL=1 forces the general one.)
  static const bool force_general = std::getenv("VXM_XR_GENERAL") != nullptr;
  const bool fast = la.fast_only && !force_general && !trace;
  void (*kern)(LowerArgs) = trace ? (wide ? k_lower_xr<3, true, false> : k_lower_xr<2, true, false>)
                            : fast ? (wide ? k_lower_xr<3, false, true> : k_lower_xr<2, false, true>)
                                   : (wide ? k_lower_xr<3, false, false> : k_lower_xr<2, false, false>);
  const int grid = ctx->resident_per_sm((const void*)kern, kL3Threads, 0, 4) * ctx->sm_count;
  ctx->lower_cta.ensure(sizeof(uint32_t) * grid);  // per-CTA counts of the in-kernel compaction
  la.cta_cnt = ctx->lower_cta.as<uint32_t>();
  void* args[] = {&la};
  ctx->prof_begin("k_lower");
  if (pdl_enabled()) {  // cooperative + programmatic serialization (see launch_pdl)
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kL3Threads);
    cfg.stream = ctx->stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    VXM_CUDA(cudaLaunchKernelEx(&cfg, kern, la));
  } else {
    VXM_CUDA(cudaLaunchCooperativeKernel((const void*)kern, dim3(grid), dim3(kL3Threads), args, 0,
                                         ctx->stream));
  }
  ctx->prof_end();
  ctx->count_launch();
  if (trace) {
    unsigned long long h[512];
    VXM_CUDA(cudaMemcpyAsync(h, trace_buf.p, sizeof h, cudaMemcpyDeviceToHost, ctx->stream));
    VXM_CUDA(cudaStreamSynchronize(ctx->stream));
    std::fprintf(stderr, "[k_lower_xr] round ends (us) / dirty blocks:");
    for (int r = 1; r < 54 && h[r]; ++r) std::fprintf(stderr, " %.1f/%llu", (h[r] - h[0]) * 1e-3, h[64 + r]);
    if (h[60]) std::fprintf(stderr, " | r1 sweeps %.1f (%llu swept, %llu copied)", (h[60] - h[0]) * 1e-3, h[58], h[59]);
    if (h[57])
      std::fprintf(stderr, " | r1 sweep: load+stage %.2f us, sweep %.2f us, %.2f passes", h[54] * 1e-3 / h[57],
                   h[55] * 1e-3 / h[57], double(h[56]) / h[57]);
    if (h[62] && h[63])
      std::fprintf(stderr, " | lowered %.1f, compared %.1f", (h[62] - h[0]) * 1e-3, (h[63] - h[0]) * 1e-3);
    std::fprintf(stderr, "\n");
    // per-round phases (us from the kernel's start): sweeps [first claim, last
    // release] avg duration | pairs first claim | last x / y / z release
    for (int r = 2; r < 24 && h[r]; ++r) {
      const unsigned long long* p = h + 128 + 16 * r;
      auto us = [&](unsigned long long v) { return v ? (double(v) - double(h[0])) * 1e-3 : -1.0; };
      std::fprintf(stderr, "  [xr r%d n=%llu] sw %.1f-%.1f (avg %.2f, %llu) pairs %.1f x %.1f y %.1f z %.1f end %.1f\n", r,
                   h[64 + r], us(p[0] ? ~p[0] : 0), us(p[1]), p[7] ? double(p[6]) * 1e-3 / double(p[7]) : 0.0, p[7],
                   us(p[2] ? ~p[2] : 0), us(p[3]), us(p[4]), us(p[5]), us(h[r]));
      if (p[7] && p[15])
        std::fprintf(stderr, "      sweep avg: wait %.2f load %.2f sweep %.2f store %.2f | pair work avg (all axes) %.2f us over %llu\n",
                     p[8] * 1e-3 / p[7], p[9] * 1e-3 / p[7], p[10] * 1e-3 / p[7], p[11] * 1e-3 / p[7],
                     (p[12] + p[13] + p[14]) * 1e-3 / p[15], p[15]);
    }
    la.trace = nullptr;
  }
  return la.out_keys != nullptr;
}

}  // namespace vxm
