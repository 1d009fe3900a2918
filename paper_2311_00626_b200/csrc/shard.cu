// Block-sharded ESDF update.
//
// Shard p of P owns the blocks with floor(x / slab) mod P == p (the same
// ownership the candidate pass uses, view.cu), each shard in its own context
// (same GPU or another one).  update_esdf over the union map
// (esdf/integrator.cpp:365-413) decomposes as follows:
//   * effective set / mark_sites: voxel-local.  Every shard runs the mark phase
//     with the UNION of the shards' updated lists; filtering by its own TSDF hash
//     keeps exactly its share of the reference's effective set.
//   * "if anything to update, reset + lower from all blocks": a global OR.
//   * lowering rounds (:488-565): sweeps are block-local; y and z pairs never
//     cross an x-slab boundary; an x pair (lo, hi) across a boundary is computed
//     by BOTH owners from the same inputs — the two post-sweep, pre-pair faces,
//     exchanged between the neighbours every round with the blocks' dirty bits
//     (pair existence, :530-538) — and each keeps its own side, so the result
//     is bit-identical to exchange_pair (:144-168); the next dirty list is
//     local; termination is a global sum.
// Rounds are driven from the host: sweep kernel -> face pack -> peer copies
// (cudaMemcpyPeerAsync; NCCL send/recv for one process per GPU) -> border
// kernel (x pairs incl. the cross pairs, grid barrier, y, barrier, z).
#include <cub/cub.cuh>

#include <algorithm>
#include <cstring>
#include <cstdlib>
#include <string>
#include <vector>

#include "shard.cuh"

namespace cg = cooperative_groups;

namespace vxm {

struct ShardRound {
  uint32_t r, ep;         // round (1-based), its epoch (base + r)
  uint32_t cur;           // pool holding the field before this update
  int lowered;            // the update lowered (the new field is in pool cur ^ 1)
  uint32_t n_blocks;       // round r > 1 reads its dirty count on the device (count[r % 3])
  uint32_t* ctr;          // [2] work counters, zeroed by the host per launch
  int rank, world, slab;
  const uint64_t* bnd_keys;  // this shard's boundary blocks, sorted by key
  const int32_t* bnd_slots;
  uint32_t n_bnd;
  uint64_t* snd_keys;
  uint8_t* snd_dirty;
  uint32_t* snd_faces;       // [n_bnd][2 faces (x = 0, x = 7)][64][3 words]
  const uint64_t* rcv_keys[2];  // [0] from the -x neighbour, [1] from the +x neighbour
  const uint8_t* rcv_dirty[2];
  const uint32_t* rcv_faces[2];
  uint32_t n_rcv[2];
};

__device__ inline int shard_owner(int32_t x, int world, int slab) {
  const int32_t q = x >= 0 ? x / slab : -((-x + slab - 1) / slab);
  return ((q % world) + world) % world;
}

// ---- sweeps of round r (round 1: reset_parented + sweep of every block) ------
__device__ void shard_sweep_body(const LowerArgs& a, const ShardRound& sr, GroupSmem* s_grp) {
  const int g = threadIdx.x >> 6, t = threadIdx.x & 63;
  const int bar = 1 + g;
  GroupSmem& G = s_grp[g];
  const bool r1 = sr.r == 1;
  uint32_t* const pcur = a.pool[sr.cur];
  uint32_t* const work = a.pool[sr.cur ^ 1u];
  const int32_t* dirty = a.list[sr.r & 1u];
  const uint32_t n = r1 ? sr.n_blocks : *((volatile const uint32_t*)(a.count + sr.r % 3u));
  const Limits lim = a.lim;
  while (true) {
    if (t == 0) G.bcast = atomicAdd(sr.ctr, 1u);
    group_sync(bar);
    const uint32_t i = G.bcast;
    if (i >= n) break;
    const int32_t s = r1 ? int32_t(i) : __ldcg(dirty + i);
    if (t == 0) {
      unsigned long long m0 = ~0ull, m1 = ~0ull, m2 = ~0ull;
      if (!r1) {  // lines through voxels changed by the last borders
        m0 = atomicExch(a.line_mask + 3 * size_t(s), 0ull);
        m1 = atomicExch(a.line_mask + 3 * size_t(s) + 1, 0ull);
        m2 = atomicExch(a.line_mask + 3 * size_t(s) + 2, 0ull);
      }
      G.mask[0][0] = m0;
      G.mask[1][0] = m1;
      G.mask[2][0] = m2;
      G.mask[0][1] = G.mask[1][1] = G.mask[2][1] = 0ull;
    }
    RawBlock rb;
    bool any_site, fast;
    load_raw3(rb, (r1 ? pcur : work) + size_t(s) * 1536, t, bar, lim, r1, &any_site, &fast);
    if (!any_site) {
      raw_store(rb, work + size_t(s) * 1536, t);
    } else {
      stage_block3(G, rb, t, bar, lim, fast);
      const bool changed = sweep_block3(G, t, bar, lim);
      if (r1 || changed) store_block3(G, work + size_t(s) * 1536, t);
    }
    group_sync(bar);
  }
}
__global__ void __launch_bounds__(kL3Threads, 2) k_shard_sweep(LowerArgs a, ShardRound sr) {
  __shared__ GroupSmem s_grp[kL3Groups];
  shard_sweep_body(a, sr, s_grp);
}

// ---- boundary faces + dirty bits, after the sweeps -----------------------------
// Written to n_dst snapshot buffers: the local send buffer (host-driven
// exchange), or directly into both neighbours' receive buffers over peer
// memory (the fused in-kernel exchange).
__device__ void shard_pack_body(const LowerArgs& a, const ShardRound& sr, const XView* dst_v, int n_dst) {
  const int lane = threadIdx.x & 31;
  const uint32_t nwarps = gridDim.x * (blockDim.x >> 5);
  const uint32_t* work = a.pool[sr.cur ^ 1u];
  const uint32_t cp = sr.r & 1u;
  for (uint32_t k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; k < sr.n_bnd; k += nwarps) {
    const int32_t s = sr.bnd_slots[k];
    const uint8_t dirty = uint8_t(sr.r == 1 || __ldcg(a.stamp_dirty[cp] + s) == sr.ep);
    const uint64_t key = sr.bnd_keys[k];
    uint32_t w[12];
#pragma unroll
    for (int f = 0; f < 2; ++f)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int q = lane + 32 * j, lin = (f ? 7 : 0) + 8 * (q & 7) + 64 * (q >> 3);
        const uint32_t* src = work + size_t(s) * 1536 + lin * 3;
        w[6 * f + 3 * j] = __ldcg(src);
        w[6 * f + 3 * j + 1] = __ldcg(src + 1);
        w[6 * f + 3 * j + 2] = __ldcg(src + 2);
      }
    for (int d = 0; d < n_dst; ++d) {
      const XView& v = dst_v[d];
      if (lane == 0) {
        v.keys[k] = key;
        v.dirty[k] = dirty;
      }
#pragma unroll
      for (int f = 0; f < 2; ++f)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int q = lane + 32 * j;
          uint32_t* dst = v.faces + ((size_t(k) * 2 + f) * 64 + q) * 3;
          dst[0] = w[6 * f + 3 * j];
          dst[1] = w[6 * f + 3 * j + 1];
          dst[2] = w[6 * f + 3 * j + 2];
        }
    }
  }
}
__global__ void k_shard_pack(LowerArgs a, ShardRound sr) {
  const XView v{sr.snd_keys, sr.snd_dirty, sr.snd_faces};
  shard_pack_body(a, sr, &v, 1);
}

__device__ inline int64_t find_key(const uint64_t* keys, uint32_t n, uint64_t k) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (keys[mid] < k) lo = mid + 1;
    else hi = mid;
  }
  return (lo < n && keys[lo] == k) ? int64_t(lo) : -1;
}

// Marks `who` changed by a border pair: line masks for its next sweep, next
// round's dirty list (esdf/integrator.cpp:552-556).
__device__ inline void mark_changed(const LowerArgs& a, uint32_t r, uint32_t ep_next, int np,
                                    int32_t who, unsigned long long m[3], int lane) {
  const unsigned long long r0 = warp_or64(m[0]), r1 = warp_or64(m[1]), r2 = warp_or64(m[2]);
  if (lane == 0) {
    atomicOr(a.line_mask + 3 * size_t(who), r0);
    atomicOr(a.line_mask + 3 * size_t(who) + 1, r1);
    atomicOr(a.line_mask + 3 * size_t(who) + 2, r2);
    if (atomicMax(a.stamp_dirty[np] + who, ep_next) < ep_next) {
      const uint32_t slot = atomicAdd(a.count + (r + 1u) % 3u, 1u);
      a.list[np][slot] = who;
    }
  }
}

// ---- border phase of round r: x (local + cross-shard), y, z ---------------------
__device__ void shard_border_body(const LowerArgs& a, const ShardRound& sr, cg::grid_group& grid) {
  const int lane = threadIdx.x & 31;
  const uint32_t wid = (blockIdx.x * kL3Threads + threadIdx.x) >> 5;
  const uint32_t nwarps = gridDim.x * (kL3Threads >> 5);
  const uint32_t r = sr.r, ep = sr.ep, ep_next = ep + 1;
  const int cp = int(r & 1u), np = cp ^ 1;
  const bool r1 = r == 1;
  uint32_t* const work = a.pool[sr.cur ^ 1u];
  const int32_t* dirty = a.list[cp];
  const uint32_t n_dirty = r1 ? sr.n_blocks : *((volatile const uint32_t*)(a.count + r % 3u));
  const uint32_t sides = r1 ? 1u : 2u;
  const uint32_t per_axis = sides * n_dirty;
  const Limits lim = a.lim;
  uint32_t n_pairs = 0;
  for (int axis = 0; axis < 3; ++axis) {
    if (axis > 0) grid.sync();
    const int dx = axis == 0, dy = axis == 1, dz = axis == 2;
    // pairs with both blocks on this shard (k_lower3's items, phased)
    for (uint32_t w = wid; w < per_axis; w += nwarps) {
      const uint32_t i = r1 ? w : w >> 1;
      const int side = r1 ? 0 : int(w & 1u);
      const int32_t d = r1 ? int32_t(i) : __ldcg(dirty + i);
      int32_t lo, hi;
      if (side == 0) {
        hi = __ldg(a.nbr + size_t(d) * 6 + 2 * axis);
        lo = d;
        if (hi < 0) continue;
      } else {
        lo = __ldg(a.nbr + size_t(d) * 6 + 2 * axis + 1);
        hi = d;
        if (lo < 0) continue;
        if (__ldcg(a.stamp_dirty[cp] + lo) == ep) continue;  // lo's side-0 item has it
      }
      if (r1) {
        // after reset_parented only sites give, and blocks an earlier axis of
        // this round changed (listed for round 2 by mark_changed, visible after
        // the grid barrier): a pair with no giver on either face is the identity
        const bool g_lo = a.site_any[lo] != 0 || (axis > 0 && __ldcg(a.stamp_dirty[np] + lo) == ep_next);
        const bool g_hi = a.site_any[hi] != 0 || (axis > 0 && __ldcg(a.stamp_dirty[np] + hi) == ep_next);
        if (!g_lo && !g_hi) continue;
      }
      bool ac = false, bc = false;
      unsigned long long mlo[3] = {0, 0, 0}, mhi[3] = {0, 0, 0};
      // both face positions of the lane loaded before any store (the four
      // voxels are distinct): one L2 round trip, not two
      int co[2][6];
      EV va[2], vb[2];
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int f = lane + 32 * k, i0 = f & 7, j0 = f >> 3;
        int* c = co[k];  // ax, ay, az, bx, by, bz
        if (axis == 0) { c[0] = 7; c[1] = i0; c[2] = j0; c[3] = 0; c[4] = i0; c[5] = j0; }
        else if (axis == 1) { c[0] = i0; c[1] = 7; c[2] = j0; c[3] = i0; c[4] = 0; c[5] = j0; }
        else { c[0] = i0; c[1] = j0; c[2] = 7; c[3] = i0; c[4] = j0; c[5] = 0; }
        va[k] = load_voxel(work, lo, c[0] + 8 * c[1] + 64 * c[2]);
        vb[k] = load_voxel(work, hi, c[3] + 8 * c[4] + 64 * c[5]);
      }
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const int* c = co[k];
        const bool cb = relax(vb[k], va[k], dx, dy, dz, lim);     // exchange_pair :158
        const bool ca = relax(va[k], vb[k], -dx, -dy, -dz, lim);  // :159
        if (cb) {
          store_voxel(work, hi, c[3] + 8 * c[4] + 64 * c[5], vb[k]);
          line_bits(c[3], c[4], c[5], mhi);
        }
        if (ca) {
          store_voxel(work, lo, c[0] + 8 * c[1] + 64 * c[2], va[k]);
          line_bits(c[0], c[1], c[2], mlo);
        }
        ac |= ca;
        bc |= cb;
      }
      ac = __any_sync(0xffffffffu, ac);
      bc = __any_sync(0xffffffffu, bc);
      ++n_pairs;
      if (ac) mark_changed(a, r, ep_next, np, lo, mlo, lane);
      if (bc) mark_changed(a, r, ep_next, np, hi, mhi, lane);
    }
    if (axis != 0) continue;
    // x pairs across a slab boundary: this shard's side of exchange_pair on the
    // two pre-pair faces (ours from the pool — only this pair touches it — and
    // the neighbour's from the exchanged snapshot)
    for (uint32_t w = wid; w < 2u * sr.n_bnd; w += nwarps) {
      const uint32_t k = w >> 1;
      const int s = (w & 1u) ? -1 : 1;
      const uint64_t bkey = sr.bnd_keys[k];
      if (shard_owner(key_x(bkey) + s, sr.world, sr.slab) == sr.rank) continue;
      const int side = s > 0 ? 1 : 0;
      const int64_t e = find_key(sr.rcv_keys[side], sr.n_rcv[side], key_shift(bkey, 0, s));
      if (e < 0) continue;  // no neighbour block: no pair
      const int32_t b = sr.bnd_slots[k];
      const bool b_dirty = r1 || __ldcg(a.stamp_dirty[cp] + b) == ep;
      if (!b_dirty && !sr.rcv_dirty[side][e]) continue;  // pair not in this round's set
      // the neighbour's face towards us: its x = 0 face when it is hi, x = 7 when lo
      const uint32_t* rf = sr.rcv_faces[side] + (size_t(e) * 2 + (s > 0 ? 0 : 1)) * 64 * 3;
      bool chg = false;
      unsigned long long m[3] = {0, 0, 0};
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int q = lane + 32 * j, y = q & 7, z = q >> 3;
        const EV vr = ev_unpack(__ldcg(rf + 3 * q), __ldcg(rf + 3 * q + 1), __ldcg(rf + 3 * q + 2));
        if (s > 0) {  // (lo = b, hi = neighbour)
          const int la = 7 + 8 * y + 64 * z;
          EV va = load_voxel(work, b, la), vb = vr;
          relax(vb, va, 1, 0, 0, lim);
          if (relax(va, vb, -1, 0, 0, lim)) {
            store_voxel(work, b, la, va);
            line_bits(7, y, z, m);
            chg = true;
          }
        } else {  // (lo = neighbour, hi = b)
          const int lb = 8 * y + 64 * z;
          EV va = vr, vb = load_voxel(work, b, lb);
          if (relax(vb, va, 1, 0, 0, lim)) {
            store_voxel(work, b, lb, vb);
            line_bits(0, y, z, m);
            chg = true;
          }
        }
      }
      chg = __any_sync(0xffffffffu, chg);
      ++n_pairs;
      if (chg) mark_changed(a, r, ep_next, np, b, m, lane);
    }
  }
  if (lane == 0 && n_pairs) atomicAdd(&a.status->sum_pairs, n_pairs);
}
__global__ void __launch_bounds__(kL3Threads, 2) k_shard_border(LowerArgs a, ShardRound sr) {
  cg::grid_group grid = cg::this_grid();
  shard_border_body(a, sr, grid);
}

// ---- the whole lowering in one persistent kernel per shard ------------------------
// Fused exchange over peer memory (NVLink P2P between GPUs, plain device
// memory between shards on one GPU): each round a shard writes its boundary
// snapshot straight into both neighbours' receive buffers, publishes the
// round on their flags with a system-scope release and acquires its own two
// flags before the border phase; the next-dirty counts go to every shard's
// count board (by round parity) and each shard sums the board — so the
// round loop, the exchange and the termination test (esdf/integrator.cpp:506)
// run with no host involvement.  A shard cannot run two rounds ahead: its
// next pack needs the whole board of the current round, which every other
// shard writes only after its own border phase.
constexpr int kFusedMaxShards = 8;
struct ShardPeers {
  XView to_right, to_left;            // the +x neighbour's rcv[0], the -x one's rcv[1]
  uint32_t* flag_right;               // their receive flags ([0] / [1])
  uint32_t* flag_left;
  const uint32_t* my_flag;            // [2] mine (written by the -x / +x neighbours)
  unsigned long long* board[kFusedMaxShards];  // every shard's [2][kFusedMaxShards] count board
  const unsigned long long* my_board;
  uint32_t* go;                       // [2] this shard's "another round" word by parity
  uint32_t* rounds_out;
  uint32_t* ctr;                      // [4] sweep claim counters, 2 per round parity
  int rank, world;
};

__device__ inline void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ inline void st_release_sys64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ inline uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ inline unsigned long long ld_acquire_sys64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// Bounded waits (2 s of globaltimer): a lost peer is an error, never a hang.
__device__ inline unsigned long long now_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void __launch_bounds__(kL3Threads, 2) k_shard_fused(LowerArgs a, ShardRound sr0, ShardPeers pe) {
  cg::grid_group grid = cg::this_grid();
  __shared__ GroupSmem s_grp[kL3Groups];
  const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
  for (uint32_t r = 1;; ++r) {
    ShardRound sr = sr0;
    sr.r = r;
    sr.ep = sr0.ep + r;  // (sr0.ep = the base epoch)
    sr.ctr = pe.ctr + 2 * (r & 1u);
    if (lead) {  // the next round's claim counters and this border's next count
      pe.ctr[2 * ((r + 1u) & 1u)] = pe.ctr[2 * ((r + 1u) & 1u) + 1] = 0u;
      a.count[(r + 1u) % 3u] = 0u;
    }
    shard_sweep_body(a, sr, s_grp);
    grid.sync();
    const XView dst[2] = {pe.to_right, pe.to_left};
    shard_pack_body(a, sr, dst, 2);
    grid.sync();
    if (lead) {
      __threadfence_system();  // every CTA's snapshot stores (ordered by grid.sync) before the flags
      st_release_sys(pe.flag_right, r);
      st_release_sys(pe.flag_left, r);
      const unsigned long long t0 = now_ns();
      while (ld_acquire_sys(pe.my_flag) < r || ld_acquire_sys(pe.my_flag + 1) < r) {
        if (now_ns() - t0 > 2000000000ull) {
          if (atomicExch(&a.status->watchdog, 1u) == 0u) a.status->pad3[0] = 60u;
          break;
        }
        __nanosleep(100);
      }
    }
    grid.sync();
    shard_border_body(a, sr, grid);
    grid.sync();
    if (lead) {
      const uint32_t cnt = *((volatile uint32_t*)(a.count + (r + 1u) % 3u));
      const unsigned long long e = (unsigned long long)r << 32 | cnt;
      const int par = int(r & 1u) * kFusedMaxShards;
      for (int q = 0; q < pe.world; ++q) st_release_sys64(pe.board[q] + par + pe.rank, e);
      unsigned long long sum = 0;
      const unsigned long long t0 = now_ns();
      for (int q = 0; q < pe.world; ++q) {
        unsigned long long v;
        while (((v = ld_acquire_sys64(pe.my_board + par + q)) >> 32) != r) {
          if (now_ns() - t0 > 2000000000ull) {
            if (atomicExch(&a.status->watchdog, 1u) == 0u) a.status->pad3[0] = 61u;
            v = 0;
            break;
          }
          __nanosleep(100);
        }
        sum += v & 0xffffffffull;
      }
      pe.go[r & 1u] = sum != 0 && a.status->watchdog == 0u ? 1u : 0u;
    }
    grid.sync();
    if (*((volatile uint32_t*)(pe.go + (r & 1u))) == 0u) {  // while (!dirty.empty())
      if (lead) *pe.rounds_out = r;
      break;
    }
  }
}

// ---- changed set of the update (esdf/integrator.cpp:403-411) -------------------
__global__ void k_shard_changed(LowerArgs a, ShardRound sr) {
  const int lane = threadIdx.x & 31;
  const uint32_t nwarps = gridDim.x * (blockDim.x >> 5);
  const uint32_t* p0 = a.pool[sr.cur];
  const uint32_t* p1 = a.pool[sr.cur ^ 1u];
  for (uint32_t k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; k < sr.n_blocks; k += nwarps) {
    const int32_t s = a.sorted_slots[k];
    bool ch = a.stamp_new[s] == a.call_epoch || a.stamp_mark[s] == a.call_epoch;
    if (!ch && sr.lowered) {
      const uint4* q0 = reinterpret_cast<const uint4*>(p0 + size_t(s) * 1536);
      const uint4* q1 = reinterpret_cast<const uint4*>(p1 + size_t(s) * 1536);
      bool diff = false;
      for (int q = lane; q < 384; q += 32) {
        const uint4 x = __ldcg(q0 + q), y = __ldcg(q1 + q);
        diff |= (x.x != y.x) | (x.y != y.y) | (x.z != y.z) | (x.w != y.w);
      }
      ch = __any_sync(0xffffffffu, diff);
    }
    if (lane == 0) a.out_flags[k] = uint8_t(ch);
  }
}

__global__ void k_shard_meta(LayerMeta* meta, uint32_t round_epoch, uint32_t cur) {
  meta->round_epoch = round_epoch;
  meta->cur = cur;
}
// (fused path: the round count is on the device)
__global__ void k_shard_meta_dev(LayerMeta* meta, uint32_t base, const uint32_t* rounds, uint32_t cur) {
  meta->round_epoch = base + *rounds + 2u;
  meta->cur = cur;
}

__global__ void k_boundary_flags(const uint64_t* keys, const uint32_t* n_ptr, int slab,
                                 uint8_t* flags) {
  const uint32_t n = *n_ptr;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int32_t x = key_x(keys[i]);
    const int32_t m = ((x % slab) + slab) % slab;
    flags[i] = uint8_t(m == 0 || m == slab - 1);
  }
}

// ---- host driver -------------------------------------------------------------------
// One shard's state through one sharded update.  The exchange between rounds
// is the caller's: in-process peer copies (run_update_esdf_sharded below) or
// a collective library when each shard is its own process (the step C-ABI,
// driven by paper_2311_00626_b200/dist.py over torch.distributed).
//
namespace {

void use(Context* c) { VXM_CUDA(cudaSetDevice(c->device)); }

ShardRound round_args(ShardUpdate& x, uint32_t r) {
  ShardRound sr{};
  sr.r = r;
  sr.ep = x.base + r;
  sr.cur = x.cur;
  sr.lowered = 1;
  sr.n_blocks = x.n_blocks;
  sr.ctr = x.ctr.as<uint32_t>();
  sr.rank = x.rank;
  sr.world = x.world;
  sr.slab = x.slab;
  sr.bnd_keys = x.bnd_keys.as<uint64_t>();
  sr.bnd_slots = x.bnd_slots.as<int32_t>();
  sr.n_bnd = x.n_bnd;
  const XView sv = xview(x.snd.p, x.n_bnd);
  sr.snd_keys = sv.keys;
  sr.snd_dirty = sv.dirty;
  sr.snd_faces = sv.faces;
  for (int i = 0; i < 2; ++i) {
    const XView rv = xview(x.rcv[i].p, x.n_rcv[i]);
    sr.rcv_keys[i] = rv.keys;
    sr.rcv_dirty[i] = rv.dirty;
    sr.rcv_faces[i] = rv.faces;
    sr.n_rcv[i] = x.n_rcv[i];
  }
  return sr;
}

int grid_of(const void* kernel, Context* c) {
  return c->resident_per_sm(kernel, kL3Threads, 0, 4) * c->sm_count;
}

}  // namespace

// Mark phase against the union list, enqueued; shard_begin_finish syncs and
// reads the outcome (x.local_any = this shard has blocks to update / clear).
void shard_begin_launch(ShardUpdate& x, const vxm_esdf_config& cfg) {
  Context* ctx = x.ctx;
  use(ctx);
  ctx->reset_status();
  x.epoch = ++ctx->call_epoch;
  const uint32_t n7 = 7u * std::max<uint32_t>(x.uni.count_hint, 1);
  x.E->note_esdf_source(x.T);
  x.E->ensure_capacity(std::min<uint64_t>(uint64_t(x.E->num_blocks) + n7, x.E->max_blocks));
  x.n_all_cap = x.E->capacity;
  x.s = esdf_scratch(ctx, x.uni.count_hint, x.n_all_cap);
  esdf_mark_phase(x.E, x.T, &x.uni, cfg, x.s, x.epoch);
  x.E->stage_meta();
  x.la = lower_args(x.E, cfg);
  x.la.full = 1;
  x.la.call_epoch = x.epoch;
  x.la.out_flags = x.s.flags;
  if (!x.h_meta) VXM_CUDA(cudaHostAlloc(&x.h_meta, sizeof(LayerMeta), cudaHostAllocDefault));
  VXM_CUDA(cudaMemcpyAsync(x.h_meta, x.E->meta, sizeof(LayerMeta), cudaMemcpyDeviceToHost, ctx->stream));
}

void shard_begin_finish(ShardUpdate& x) {
  Context* ctx = x.ctx;
  use(ctx);
  ctx->sync_status();
  x.E->adopt_meta();
  const DevStatus& st = *ctx->h_status;
  if (st.capacity_error || st.pool_overflow)
    throw Error(VXM_ERR_CAPACITY, "Layer: block capacity exhausted");
  x.local_any = st.any_update != 0;
  const LayerMeta& m = *x.h_meta;
  x.base = m.round_epoch;
  x.cur = m.cur;
  x.n_blocks = m.num_blocks;
  // the sorted order is final once the mark phase (allocation) completed
  x.la.sorted_slots = x.E->sorted_slots[x.E->sorted_parity];
  x.la.stamp_new = x.E->stamp_new;
  x.la.stamp_mark = x.E->stamp_mark;
}

void shard_begin(ShardUpdate& x, const vxm_esdf_config& cfg) {
  shard_begin_launch(x, cfg);
  shard_begin_finish(x);
}

// Boundary blocks (x mod slab in {0, slab - 1}), sorted; the send buffer.
void shard_plan_launch(ShardUpdate& x) {
  use(x.ctx);
  cudaStream_t st = x.ctx->stream;
  const uint32_t n = std::max<uint32_t>(x.n_blocks, 1);
  x.bnd_flags.ensure(n);
  x.bnd_keys.ensure(sizeof(uint64_t) * n);
  x.bnd_slots.ensure(sizeof(int32_t) * n);
  x.bnd_n.ensure(2 * sizeof(uint32_t));
  x.ctr.ensure(4 * sizeof(uint32_t));
  if (!x.h_cnt) VXM_CUDA(cudaHostAlloc(&x.h_cnt, 4 * sizeof(uint32_t), cudaHostAllocDefault));
  const uint64_t* keys = x.E->sorted_keys[x.E->sorted_parity];
  const int32_t* slots = x.E->sorted_slots[x.E->sorted_parity];
  k_boundary_flags<<<grid_for(x.ctx, n), 256, 0, st>>>(keys, &x.E->meta->num_blocks, x.slab,
                                                         x.bnd_flags.as<uint8_t>());
  size_t b1 = 0, b2 = 0;
  cub::DeviceSelect::Flagged(nullptr, b1, keys, x.bnd_flags.as<uint8_t>(), x.bnd_keys.as<uint64_t>(),
                             x.bnd_n.as<uint32_t>(), int(x.n_blocks), st);
  cub::DeviceSelect::Flagged(nullptr, b2, slots, x.bnd_flags.as<uint8_t>(), x.bnd_slots.as<int32_t>(),
                             x.bnd_n.as<uint32_t>() + 1, int(x.n_blocks), st);
  x.cub_tmp.ensure(std::max(b1, b2));
  VXM_CUDA(cub::DeviceSelect::Flagged(x.cub_tmp.p, b1, keys, x.bnd_flags.as<uint8_t>(),
                                      x.bnd_keys.as<uint64_t>(), x.bnd_n.as<uint32_t>(), int(x.n_blocks),
                                      st));
  VXM_CUDA(cub::DeviceSelect::Flagged(x.cub_tmp.p, b2, slots, x.bnd_flags.as<uint8_t>(),
                                      x.bnd_slots.as<int32_t>(), x.bnd_n.as<uint32_t>() + 1,
                                      int(x.n_blocks), st));
  x.ctx->count_launch(3);
  check_launch(x.ctx, "shard_plan");
  VXM_CUDA(cudaMemcpyAsync(x.h_cnt, x.bnd_n.p, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
}

void shard_plan_finish(ShardUpdate& x) {
  use(x.ctx);
  VXM_CUDA(cudaStreamSynchronize(x.ctx->stream));
  x.n_bnd = x.h_cnt[0];
  x.snd.ensure(std::max<size_t>(xbuf_bytes(x.n_bnd), 8));
}

void shard_plan(ShardUpdate& x) {
  shard_plan_launch(x);
  shard_plan_finish(x);
}

void shard_set_neighbours(ShardUpdate& x, uint32_t n_left, uint32_t n_right) {
  use(x.ctx);
  x.n_rcv[0] = n_left;
  x.n_rcv[1] = n_right;
  for (int i = 0; i < 2; ++i) x.rcv[i].ensure(std::max<size_t>(xbuf_bytes(x.n_rcv[i]), 8));
}

// Sweeps of round r and the pack of the send buffer, enqueued on the shard's
// stream (the exchange that reads the send buffer is ordered after it).
void shard_sweep(ShardUpdate& x, uint32_t r) {
  use(x.ctx);
  cudaStream_t st = x.ctx->stream;
  const int g_sweep = grid_of((const void*)k_shard_sweep, x.ctx);
  VXM_CUDA(cudaMemsetAsync(x.ctr.p, 0, 4 * sizeof(uint32_t), st));
  ShardRound sr = round_args(x, r);
  k_shard_sweep<<<g_sweep, kL3Threads, 0, st>>>(x.la, sr);
  k_shard_pack<<<grid_for(x.ctx, uint64_t(std::max<uint32_t>(x.n_bnd, 1)) * 32), 256, 0, st>>>(x.la, sr);
  x.ctx->count_launch(2);
  check_launch(x.ctx, "k_shard_sweep");
}

// Border phase of round r (the receive buffers hold the neighbours' snapshots),
// enqueued; this shard's next dirty count is written to next_count_ptr(x, r)
// on the device and copied to x.h_cnt[1] (valid after a stream sync).
uint32_t* next_count_ptr(ShardUpdate& x, uint32_t r) { return x.la.count + (r + 1u) % 3u; }

void shard_border_launch(ShardUpdate& x, uint32_t r) {
  use(x.ctx);
  cudaStream_t st = x.ctx->stream;
  const int g_border = grid_of((const void*)k_shard_border, x.ctx);
  VXM_CUDA(cudaMemsetAsync(next_count_ptr(x, r), 0, sizeof(uint32_t), st));
  ShardRound sr = round_args(x, r);
  void* args[] = {&x.la, &sr};
  VXM_CUDA(cudaLaunchCooperativeKernel((const void*)k_shard_border, dim3(g_border), dim3(kL3Threads),
                                       args, 0, st));
  x.ctx->count_launch();
  VXM_CUDA(cudaMemcpyAsync(x.h_cnt + 1, next_count_ptr(x, r), sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
  x.rounds = r;
}

// Synchronous form: returns this shard's next dirty count.
uint32_t shard_border(ShardUpdate& x, uint32_t r) {
  shard_border_launch(x, r);
  VXM_CUDA(cudaStreamSynchronize(x.ctx->stream));
  return x.h_cnt[1];
}

// Changed set (esdf/integrator.cpp:403-411) and meta; `lowered`: the global
// decision of this update.
uint32_t* fused_rounds_ptr(ShardUpdate& x);

void shard_finish_launch(ShardUpdate& x, bool lowered, BlockList* out) {
  use(x.ctx);
  cudaStream_t st = x.ctx->stream;
  ShardRound sr = round_args(x, std::max<uint32_t>(x.rounds, 1));
  sr.lowered = lowered ? 1 : 0;
  k_shard_changed<<<grid_for(x.ctx, uint64_t(std::max<uint32_t>(x.n_blocks, 1)) * 32), 256, 0, st>>>(x.la, sr);
  x.ctx->count_launch();
  if (lowered && x.fused) {  // the round count is on the device
    k_shard_meta_dev<<<1, 1, 0, st>>>(x.E->meta, x.base, fused_rounds_ptr(x), x.cur ^ 1u);
    VXM_CUDA(cudaMemcpyAsync(x.h_cnt + 2, fused_rounds_ptr(x), sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    x.ctx->count_launch();
  } else if (lowered) {
    k_shard_meta<<<1, 1, 0, st>>>(x.E->meta, x.base + x.rounds + 2, x.cur ^ 1u);
    x.ctx->count_launch();
  }
  out->bind(x.ctx);
  out->ensure(x.n_all_cap);
  launch_compact_keys(x.ctx, x.E->sorted_keys[x.E->sorted_parity], x.s.flags, &x.E->meta->num_blocks,
                      x.n_all_cap, out->keys.as<uint64_t>(), out->d_count, nullptr, "k_compact_esdf");
  out->host_valid = false;
  out->host_pending = false;
  out->count_hint = x.n_all_cap;
  out->sorted_unique = true;
  x.E->stage_meta();
}

void shard_finish_sync(ShardUpdate& x, bool lowered) {
  use(x.ctx);
  x.ctx->sync_status();
  x.E->adopt_meta();
  if (x.fused) {
    x.rounds = x.h_cnt[2];
    for (void* p : x.ipc_open) cudaIpcCloseMemHandle(p);
    x.ipc_open.clear();
  }
  if (x.ctx->h_status->watchdog)
    throw Error(VXM_ERR_INTERNAL, "sharded ESDF lowering: a peer wait expired (code " +
                                      std::to_string(x.ctx->h_status->pad3[0]) + ")");
  vxm_stats& w = x.ctx->stats;
  w.esdf_calls += 1;
  w.esdf_blocks += x.n_blocks;
  w.lower_rounds += lowered ? x.rounds : 0;
}

void shard_finish(ShardUpdate& x, bool lowered, BlockList* out) {
  shard_finish_launch(x, lowered, out);
  shard_finish_sync(x, lowered);
}

ShardUpdate::~ShardUpdate() {
  for (void* p : ipc_open) cudaIpcCloseMemHandle(p);
  if (h_meta) cudaFreeHost(h_meta);
  if (h_cnt) cudaFreeHost(h_cnt);
  if (ev) cudaEventDestroy(ev);
}

// ---- fused path: one persistent kernel per shard (k_shard_fused) ---------------
namespace {
constexpr size_t kMboxFlags = 0, kMboxBoard = 64, kMboxGo = 64 + 16 * 8, kMboxRounds = kMboxGo + 8,
                 kMboxBytes = 512;
template <typename T>
T* mbox_at(ShardUpdate& x, size_t off) {
  return reinterpret_cast<T*>(static_cast<unsigned char*>(x.mbox.p) + off);
}

// Peer access between every pair of the shards' devices (the count board is
// written by every shard); false when some pair cannot.
bool enable_peers(std::vector<ShardUpdate>& sh) {
  std::vector<int> devs;
  for (auto& x : sh)
    if (std::find(devs.begin(), devs.end(), x.ctx->device) == devs.end()) devs.push_back(x.ctx->device);
  for (int a : devs)
    for (int b : devs) {
      if (a == b) continue;
      int ok = 0;
      VXM_CUDA(cudaDeviceCanAccessPeer(&ok, a, b));
      if (!ok) return false;
      VXM_CUDA(cudaSetDevice(a));
      const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) (void)cudaGetLastError();
      else VXM_CUDA(e);
    }
  return true;
}
}  // namespace

uint32_t* fused_rounds_ptr(ShardUpdate& x) { return mbox_at<uint32_t>(x, kMboxRounds); }

namespace {
ShardPeers make_peers(ShardUpdate& x, ShardUpdate* right, ShardUpdate* left, void* right_rcv0, void* left_rcv1,
                      void* right_mbox, void* left_mbox, void* const* boards, int world) {
  (void)right;
  (void)left;
  ShardPeers pe{};
  pe.to_right = xview(right_rcv0, x.n_bnd);
  pe.to_left = xview(left_rcv1, x.n_bnd);
  pe.flag_right = reinterpret_cast<uint32_t*>(static_cast<unsigned char*>(right_mbox) + kMboxFlags);
  pe.flag_left = reinterpret_cast<uint32_t*>(static_cast<unsigned char*>(left_mbox) + kMboxFlags) + 1;
  pe.my_flag = mbox_at<uint32_t>(x, kMboxFlags);
  for (int q = 0; q < world; ++q)
    pe.board[q] = reinterpret_cast<unsigned long long*>(static_cast<unsigned char*>(boards[q]) + kMboxBoard);
  pe.my_board = mbox_at<unsigned long long>(x, kMboxBoard);
  pe.go = mbox_at<uint32_t>(x, kMboxGo);
  pe.rounds_out = mbox_at<uint32_t>(x, kMboxRounds);
  pe.ctr = x.ctr.as<uint32_t>();
  pe.rank = x.rank;
  pe.world = world;
  return pe;
}

void launch_fused(ShardUpdate& x, ShardPeers& pe, int sharing) {
  use(x.ctx);
  const int per_sm = x.ctx->resident_per_sm((const void*)k_shard_fused, kL3Threads, 0, 4);
  const int grid = std::max(1, per_sm * x.ctx->sm_count / std::max(1, sharing));
  ShardRound sr0 = round_args(x, 0);  // ep = the base epoch
  void* args[] = {&x.la, &sr0, &pe};
  VXM_CUDA(cudaLaunchCooperativeKernel((const void*)k_shard_fused, dim3(grid), dim3(kL3Threads), args, 0,
                                       x.ctx->stream));
  x.ctx->count_launch();
  check_launch(x.ctx, "k_shard_fused");
  x.fused = true;
}
}  // namespace

void shard_ipc_handles(ShardUpdate& x, void* out192) {
  use(x.ctx);
  x.mbox.ensure(kMboxBytes);
  VXM_CUDA(cudaMemsetAsync(x.mbox.p, 0, kMboxBytes, x.ctx->stream));
  VXM_CUDA(cudaMemsetAsync(x.ctr.p, 0, 4 * sizeof(uint32_t), x.ctx->stream));
  VXM_CUDA(cudaStreamSynchronize(x.ctx->stream));
  cudaIpcMemHandle_t h[3];
  VXM_CUDA(cudaIpcGetMemHandle(&h[0], x.rcv[0].p));
  VXM_CUDA(cudaIpcGetMemHandle(&h[1], x.rcv[1].p));
  VXM_CUDA(cudaIpcGetMemHandle(&h[2], x.mbox.p));
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  std::memcpy(out192, h, sizeof h);
}

void shard_lower_fused_ipc(ShardUpdate& x, const void* all, int ranks_on_device) {
  use(x.ctx);
  const int P = x.world, me = x.rank;
  if (P < 2 || P > kFusedMaxShards)
    throw Error(VXM_ERR_INVALID_ARGUMENT, "fused shard exchange: 2..8 shards");
  const cudaIpcMemHandle_t* h = static_cast<const cudaIpcMemHandle_t*>(all);
  auto open = [&](int rank, int which) -> void* {
    if (rank == me) return which == 0 ? x.rcv[0].p : which == 1 ? x.rcv[1].p : x.mbox.p;
    void* p = nullptr;
    VXM_CUDA(cudaIpcOpenMemHandle(&p, h[3 * rank + which], cudaIpcMemLazyEnablePeerAccess));
    x.ipc_open.push_back(p);
    return p;
  };
  const int right = (me + 1) % P, left = (me - 1 + P) % P;
  std::vector<void*> boards(P);
  for (int q = 0; q < P; ++q) boards[q] = open(q, 2);
  void* r0 = open(right, 0);
  void* l1 = open(left, 1);
  ShardPeers pe = make_peers(x, nullptr, nullptr, r0, l1, boards[right], boards[left], boards.data(), P);
  launch_fused(x, pe, ranks_on_device);
}

// The whole round loop on the device: launches k_shard_fused on every shard
// (all resident at once: shards on one GPU split its SMs) and the changed-set
// kernels; the caller synchronises once.
void shard_lower_fused(std::vector<ShardUpdate>& sh) {
  const int P = int(sh.size());
  for (auto& x : sh) {  // fresh mailboxes (the host syncs before any kernel runs)
    use(x.ctx);
    x.mbox.ensure(kMboxBytes);
    VXM_CUDA(cudaMemsetAsync(x.mbox.p, 0, kMboxBytes, x.ctx->stream));
    VXM_CUDA(cudaMemsetAsync(x.ctr.p, 0, 4 * sizeof(uint32_t), x.ctx->stream));
  }
  for (auto& x : sh) {
    use(x.ctx);
    VXM_CUDA(cudaStreamSynchronize(x.ctx->stream));
  }
  std::vector<void*> boards(P);
  for (int q = 0; q < P; ++q) boards[q] = sh[q].mbox.p;
  for (int p = 0; p < P; ++p) {
    ShardUpdate& x = sh[p];
    ShardUpdate& right = sh[(p + 1) % P];
    ShardUpdate& left = sh[(p - 1 + P) % P];
    ShardPeers pe = make_peers(x, &right, &left, right.rcv[0].p, left.rcv[1].p, right.mbox.p, left.mbox.p,
                               boards.data(), P);
    int same = 0;  // shards sharing this GPU share its SMs
    for (auto& y : sh) same += y.ctx->device == x.ctx->device;
    launch_fused(x, pe, same);
  }
}

// All shards in this process (one context each, same or peer GPUs): every
// step is enqueued on all shards before any is waited for, the exchange is
// peer copies ordered by events (no host round trip), and each round costs ONE
// host synchronisation — the global sum of the next dirty counts that ends the
// loop (esdf/integrator.cpp:506).
void run_update_esdf_sharded(int P, Layer** E, Layer** T, BlockList** updated,
                             const vxm_esdf_config& cfg, int slab, BlockList** out) {
  std::vector<ShardUpdate> sh(P);
  for (int p = 0; p < P; ++p) {
    sh[p].E = E[p];
    sh[p].T = T[p];
    sh[p].ctx = E[p]->ctx;
    sh[p].rank = p;
    sh[p].world = P;
    sh[p].slab = slab;
  }
  auto copy_to = [&](ShardUpdate& dst, void* d, Context* src_ctx, const void* s, size_t bytes) {
    if (!bytes) return;
    use(dst.ctx);
    if (dst.ctx->device == src_ctx->device)
      VXM_CUDA(cudaMemcpyAsync(d, s, bytes, cudaMemcpyDeviceToDevice, dst.ctx->stream));
    else
      VXM_CUDA(cudaMemcpyPeerAsync(d, dst.ctx->device, s, src_ctx->device, bytes, dst.ctx->stream));
  };
  auto record = [&](ShardUpdate& x) {
    use(x.ctx);
    if (!x.ev) VXM_CUDA(cudaEventCreateWithFlags(&x.ev, cudaEventDisableTiming));
    VXM_CUDA(cudaEventRecord(x.ev, x.ctx->stream));
  };
  auto wait_for = [&](ShardUpdate& x, ShardUpdate& on) {
    if (&x == &on) return;
    use(x.ctx);
    VXM_CUDA(cudaStreamWaitEvent(x.ctx->stream, on.ev, 0));
  };
  auto sync_all = [&] {
    for (auto& x : sh) {
      use(x.ctx);
      VXM_CUDA(cudaStreamSynchronize(x.ctx->stream));
    }
  };
  // union of the updated lists: every shard marks against all of them
  std::vector<uint32_t> n_upd(P);
  uint64_t total = 0;
  for (int p = 0; p < P; ++p) {
    use(updated[p]->ctx);
    VXM_CUDA(cudaStreamSynchronize(updated[p]->ctx->stream));
    VXM_CUDA(cudaMemcpy(&n_upd[p], updated[p]->d_count, sizeof(uint32_t), cudaMemcpyDeviceToHost));
    total += n_upd[p];
  }
  if (total == 0) {  // esdf/integrator.cpp:371-378
    for (int p = 0; p < P; ++p) out[p]->assign_host(nullptr, 0);
    return;
  }
  for (auto& x : sh) {
    use(x.ctx);
    x.uni.bind(x.ctx);
    x.uni.ensure(uint32_t(total));
    uint64_t off = 0;
    for (int p = 0; p < P; ++p) {
      copy_to(x, x.uni.keys.as<uint64_t>() + off, updated[p]->ctx, updated[p]->keys.p,
              sizeof(uint64_t) * n_upd[p]);
      off += n_upd[p];
    }
    const uint32_t t32 = uint32_t(total);
    VXM_CUDA(cudaMemcpyAsync(x.uni.d_count, &t32, sizeof t32, cudaMemcpyHostToDevice, x.ctx->stream));
    x.uni.count_hint = t32;
    x.uni.host_valid = false;
    x.uni.host_pending = false;
    sort_unique_keys(x.ctx, &x.uni);
    x.uni.sorted_unique = true;
    shard_begin_launch(x, cfg);
  }
  bool any = false;
  for (auto& x : sh) {
    shard_begin_finish(x);
    any |= x.local_any;
  }
  static const bool fused_env = [] {  // VXM_SHARD_FUSED=0: host-driven rounds
    const char* e = std::getenv("VXM_SHARD_FUSED");
    return !(e && e[0] == '0');
  }();
  const bool fused = any && fused_env && P >= 2 && P <= kFusedMaxShards && enable_peers(sh);
  if (any) {
    for (auto& x : sh) shard_plan_launch(x);
    for (auto& x : sh) shard_plan_finish(x);
    for (int p = 0; p < P; ++p)  // [0]: from the -x neighbour, [1]: from the +x one
      shard_set_neighbours(sh[p], sh[(p - 1 + P) % P].n_bnd, sh[(p + 1) % P].n_bnd);
  }
  if (fused) {
    shard_lower_fused(sh);
    for (int p = 0; p < P; ++p) shard_finish_launch(sh[p], true, out[p]);
    for (auto& x : sh) shard_finish_sync(x, true);
    return;
  }
  if (any) {
    for (uint32_t r = 1;; ++r) {
      for (auto& x : sh) {
        shard_sweep(x, r);
        record(x);  // send buffer packed
      }
      for (int p = 0; p < P; ++p) {  // snapshot p -> the +x neighbour's [0], the -x one's [1]
        ShardUpdate& src = sh[p];
        ShardUpdate& right = sh[(p + 1) % P];
        ShardUpdate& left = sh[(p - 1 + P) % P];
        wait_for(right, src);
        copy_to(right, right.rcv[0].p, src.ctx, src.snd.p, xbuf_bytes(src.n_bnd));
        wait_for(left, src);
        copy_to(left, left.rcv[1].p, src.ctx, src.snd.p, xbuf_bytes(src.n_bnd));
      }
      for (auto& x : sh) shard_border_launch(x, r);
      sync_all();  // the round's one host round trip
      uint64_t next = 0;
      for (auto& x : sh) next += x.h_cnt[1];
      if (next == 0) break;  // while (!dirty.empty()) — esdf/integrator.cpp:506
    }
  }
  for (int p = 0; p < P; ++p) shard_finish_launch(sh[p], any, out[p]);
  for (auto& x : sh) shard_finish_sync(x, any);
}

}  // namespace vxm
