// Device building blocks of the ESDF lowering (shared by the fused single-map
// kernel in esdf.cu and the sharded round kernels in shard.cu):
// relax (esdf/integrator.cpp:58-88), the staged block formats and sweeps
// (:96-139), block load/store, stamps.  See esdf.cu for the design notes.
#pragma once

#include <cooperative_groups.h>

#include "runtime.cuh"

namespace vxm {

// ---- voxel register form ---------------------------------------------------------
struct EV {
  int sq, px, py, pz;
  uint32_t f;    // flags
  uint32_t res;  // reserved byte (preserved)
};
__device__ inline EV ev_unpack(uint32_t w0, uint32_t w1, uint32_t w2) {
  EV v;
  v.sq = int(w0);
  v.px = int(int16_t(w1 & 0xffffu));
  v.py = int(int16_t(w1 >> 16));
  v.pz = int(int16_t(w2 & 0xffffu));
  v.f = (w2 >> 16) & 0xffu;
  v.res = w2 >> 24;
  return v;
}
__device__ inline uint32_t ev_w1(const EV& v) { return (uint32_t(v.px) & 0xffffu) | (uint32_t(v.py) << 16); }
__device__ inline uint32_t ev_w2(const EV& v) {
  return (uint32_t(v.pz) & 0xffffu) | (v.f << 16) | (v.res << 24);
}
__device__ inline bool ev_has_parent(const EV& v) { return (v.px | v.py | v.pz) != 0; }

struct Limits {
  int max_sq, cap_sq;
};

// relax — esdf/integrator.cpp:58-88
__device__ inline bool relax(EV& v, const EV& u, int dx, int dy, int dz, const Limits& lim) {
  if (!(u.f & VXM_ESDF_OBSERVED) || (!(u.f & VXM_ESDF_SITE) && !ev_has_parent(u))) return false;
  if (!(v.f & VXM_ESDF_OBSERVED) || (v.f & VXM_ESDF_SITE)) return false;
  const int cx = u.px - dx, cy = u.py - dy, cz = u.pz - dz;
  const int cand = int(uint32_t(cx * cx) + uint32_t(cy * cy) + uint32_t(cz * cz));
  if (cand == 0) return false;
  const int limit = (v.f & VXM_ESDF_INSIDE) ? lim.cap_sq : lim.max_sq;
  if (cand > limit || cand > v.sq) return false;
  if (cand == v.sq && ev_has_parent(v)) {
    const bool less = cx < v.px || (cx == v.px && (cy < v.py || (cy == v.py && cz < v.pz)));
    if (!less) return false;
  }
  v.sq = cand;
  v.px = int(int16_t(cx));
  v.py = int(int16_t(cy));
  v.pz = int(int16_t(cz));
  return true;
}

__device__ inline void reset_to_saturated(EV& v, const Limits& lim) {
  v.sq = (v.f & VXM_ESDF_INSIDE) ? lim.cap_sq : lim.max_sq;
  v.px = v.py = v.pz = 0;
}

// Bank-conflict-free swizzle of the 512 voxels of a block:
// bank = (x0^z0, x1^z1, x2^y2, y0^z0, y1^z1), high bits (x0, x1, y2, z2).  For
// the X-, Y- and Z-line phases every warp's 32 accesses hit 32 distinct banks.
__device__ inline int swz(int x, int y, int z) {
  const int b0 = (x ^ z) & 1, b1 = ((x >> 1) ^ (z >> 1)) & 1, b2 = ((x >> 2) ^ (y >> 2)) & 1;
  const int b3 = (y ^ z) & 1, b4 = ((y >> 1) ^ (z >> 1)) & 1;
  return b0 | (b1 << 1) | (b2 << 2) | (b3 << 3) | (b4 << 4) | ((x & 1) << 5) | (((x >> 1) & 1) << 6) |
         (((y >> 2) & 1) << 7) | (((z >> 2) & 1) << 8);
}
__device__ inline int swz_lin(int lin) { return swz(lin & 7, (lin >> 3) & 7, lin >> 6); }

// Named barrier over one 64-thread group, with an OR reduction of `pred`.
__device__ inline bool group_sync_or(int id, bool pred) {
  int r;
  asm volatile(
      "{\n\t.reg .pred p, q;\n\t"
      "setp.ne.s32 p, %1, 0;\n\t"
      "bar.red.or.pred q, %2, 64, p;\n\t"
      "selp.s32 %0, 1, 0, q;\n\t}"
      : "=r"(r)
      : "r"(int(pred)), "r"(id)
      : "memory");
  return r != 0;
}
__device__ inline void group_sync(int id) {
  asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory");
}

// ===== sweep v3: one 64-thread group per block, one line per thread ============
// Working format in shared memory (converted from the reference's 12-byte voxel
// on load and back on store):
//   w0  = squared distance
//   klo = (py + 2^15) << 16 | (pz + 2^15)
//   khi = (px + 2^15) | flags << 16 | reserved << 24
// so the parent offset is a 48-bit key (khi & 0xffff) << 32 | klo whose
// unsigned order is the lexicographic (x, y, z) order used by relax's tie
// break, and a single-axis step is one 64-bit add.
constexpr unsigned long long kKeyZero = 0x800080008000ull;  // offset (0, 0, 0)

struct GroupSmem {
  // general format: a[0] = w0, a[1] = klo, a[2] = khi (above);
  // compact format: a[0..4] = TH, TL, KEY, GQ, FL (below)
  uint32_t a[5][512];
  unsigned long long mask[3][2];  // dirty lines per phase (X, Y, Z) by pass parity
  uint32_t bcast;
  uint32_t fast;  // 1: the staged block is in the compact format
};

// Compact format, used for a block when max_sq <= kFastOff^2 and every voxel
// has parent components within +-kFastOff, 0 <= sq < 2^29, and (if it can
// give: observed and a site or parented) sq == |parent|^2 — always the case
// for fields produced by update_esdf; other blocks keep the general format.
//   KEY = 10-bit biased parent fields x << 20 | y << 10 | z
//   GQ  = sq - 1 for a giver (so (other two components)^2 - 1 = GQ - pa^2 for
//         a line along any axis), 2^30 + sq for a non-giver (its candidate
//         then exceeds every limit)
//   TH, TL = the taker threshold: a candidate (cand - 1, key) is accepted iff
//         it compares below (TH, TL) as a 64-bit pair.  That single compare is
//         relax's cand != 0, cand <= limit, cand < sq, and the tie rule (an
//         unparented taker carries bit 30 in TL, so any parented candidate
//         wins the tie); non-takers have (0, 0)
//   FL  = flags << 16 | reserved << 24
// so a relax on the line's dependency chain is IMAD -> 64-bit compare -> SEL.
constexpr int kFastOff = 510;
constexpr uint32_t kFastBias = 512u;
constexpr uint32_t kUnpar = 1u << 30;
constexpr uint32_t kNoGive = 1u << 30;

template <int AXIS>
__device__ inline int line_idx3(int q, int k) {  // q in [0, 64): the orthogonal coords
  const int c0 = q & 7, c1 = q >> 3;
  const int x = AXIS == 0 ? k : c0;
  const int y = AXIS == 1 ? k : (AXIS == 0 ? c0 : c1);
  const int z = AXIS == 2 ? k : c1;
  return swz(x, y, z);
}

__device__ inline unsigned long long spread8(uint32_t ch) {  // bit k -> bit 8k
  unsigned long long m = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) m |= (unsigned long long)((ch >> k) & 1u) << (8 * k);
  return m;
}

// One line along AXIS (q = index of the two orthogonal coordinates), X+ then X-
// Gauss-Seidel relaxes in registers — esdf/integrator.cpp:58-88, 96-139.
template <int AXIS>
__device__ inline uint32_t sweep_line3(GroupSmem& g, int q, const Limits& lim) {
  constexpr int sh = AXIS == 0 ? 32 : (AXIS == 1 ? 16 : 0);
  int sq[8], pa[8], qq[8], idx[8];
  unsigned long long key[8];
  uint32_t take = 0, give = 0, in = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    idx[k] = line_idx3<AXIS>(q, k);
    const uint32_t lo = g.a[1][idx[k]], hi = g.a[2][idx[k]];
    sq[k] = int(g.a[0][idx[k]]);
    key[k] = ((unsigned long long)(hi & 0xffffu) << 32) | lo;
    const int px = int(hi & 0xffffu) - 0x8000, py = int(lo >> 16) - 0x8000,
              pz = int(lo & 0xffffu) - 0x8000;
    pa[k] = AXIS == 0 ? px : (AXIS == 1 ? py : pz);
    const int o1 = AXIS == 0 ? py : px, o2 = AXIS == 2 ? py : pz;
    qq[k] = int(uint32_t(o1 * o1) + uint32_t(o2 * o2));
    const uint32_t f = (hi >> 16) & 0xffu;
    const bool obs = f & VXM_ESDF_OBSERVED, site = f & VXM_ESDF_SITE;
    take |= uint32_t(obs && !site) << k;
    give |= uint32_t(obs && (site || key[k] != kKeyZero)) << k;
    in |= uint32_t((f & VXM_ESDF_INSIDE) != 0) << k;
  }
  uint32_t ch = 0;
  auto relax3 = [&](int k, int j, int s) {
    const int pc = pa[j] - s;
    const int cand = int(uint32_t(pc * pc) + uint32_t(qq[j]));
    const unsigned long long ckey = s > 0 ? key[j] - (1ull << sh) : key[j] + (1ull << sh);
    const int limk = ((in >> k) & 1u) ? lim.cap_sq : lim.max_sq;
    const bool better = cand < sq[k] || (cand == sq[k] && (key[k] == kKeyZero || ckey < key[k]));
    const bool ok = ((give >> j) & (take >> k) & 1u) && cand != 0 && cand <= limk && better;
    if (ok) {
      sq[k] = cand;
      key[k] = ckey;
      pa[k] = pc;
      qq[k] = qq[j];
      give |= 1u << k;
      ch |= 1u << k;
    }
  };
#pragma unroll
  for (int k = 1; k < 8; ++k) relax3(k, k - 1, 1);  // X+ (resp. Y+, Z+)
#pragma unroll
  for (int k = 6; k >= 0; --k) relax3(k, k + 1, -1);  // X- (resp. Y-, Z-)
#pragma unroll
  for (int k = 0; k < 8; ++k)
    if (ch & (1u << k)) {
      g.a[0][idx[k]] = uint32_t(sq[k]);
      g.a[1][idx[k]] = uint32_t(key[k]);
      g.a[2][idx[k]] = (g.a[2][idx[k]] & 0xffff0000u) | uint32_t(key[k] >> 32);
    }
  return ch;
}

// Runs one phase of a pass for the group: only lines marked dirty are swept
// (an unchanged line is idempotent under its X+/X- sweep), changes mark the
// lines through the changed voxels for the phases that follow.

// sweep_line3 on the compact format — same relax semantics
// (esdf/integrator.cpp:58-88).  Per voxel in registers: the threshold (th, tl),
// qm = GQ - pa^2, and the giver's outgoing offset along the line and key,
// pre-shifted by the step (po, ko), so the chain per relax is one IMAD, one
// 64-bit compare and the selects.
template <int AXIS>
__device__ inline uint32_t sweep_line_fast(GroupSmem& g, int q) {
  constexpr int sh = AXIS == 0 ? 20 : (AXIS == 1 ? 10 : 0);
  constexpr uint32_t sb = 1u << sh;
  uint32_t th[8], tl[8], qm[8], ko[8];
  int po[8], idx[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    idx[k] = line_idx3<AXIS>(q, k);
    th[k] = g.a[0][idx[k]];
    tl[k] = g.a[1][idx[k]];
    const uint32_t key = g.a[2][idx[k]];
    const int pa = int((key >> sh) & 1023u) - int(kFastBias);
    qm[k] = g.a[3][idx[k]] - uint32_t(pa * pa);
    po[k] = pa - 1;  // outgoing along +axis
    ko[k] = key - sb;
  }
  uint32_t ch = 0;
#pragma unroll
  for (int k = 1; k < 8; ++k) {  // X+ (resp. Y+, Z+)
    const int j = k - 1;
    const uint32_t cm = uint32_t(po[j] * po[j]) + qm[j];  // cand - 1 (mod 2^32)
    const unsigned long long cv = (unsigned long long)cm << 32 | ko[j];
    const unsigned long long tv = (unsigned long long)th[k] << 32 | tl[k];
    if (cv < tv) {
      th[k] = cm;
      tl[k] = ko[j];
      qm[k] = qm[j];
      po[k] = po[j] - 1;
      ko[k] = ko[j] - sb;
      ch |= 1u << k;
    }
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) {  // outgoing along -axis
    po[k] += 2;
    ko[k] += 2u * sb;
  }
#pragma unroll
  for (int k = 6; k >= 0; --k) {  // X- (resp. Y-, Z-)
    const int j = k + 1;
    const uint32_t cm = uint32_t(po[j] * po[j]) + qm[j];
    const unsigned long long cv = (unsigned long long)cm << 32 | ko[j];
    const unsigned long long tv = (unsigned long long)th[k] << 32 | tl[k];
    if (cv < tv) {
      th[k] = cm;
      tl[k] = ko[j];
      qm[k] = qm[j];
      po[k] = po[j] + 1;
      ko[k] = ko[j] + sb;
      ch |= 1u << k;
    }
  }
#pragma unroll
  for (int k = 0; k < 8; ++k)
    if (ch & (1u << k)) {  // now a giver: sq = cand, parent = key
      g.a[0][idx[k]] = th[k];
      g.a[1][idx[k]] = tl[k];
      g.a[2][idx[k]] = tl[k];
      g.a[3][idx[k]] = th[k];
    }
  return ch;
}

// FASTONLY: every staged block is in the compact format (the caller
// guarantees it; see k_lower_xr), so the general format's code is not
// compiled in.
template <int AXIS, bool FASTONLY = false>
__device__ inline uint32_t sweep_phase3(GroupSmem& g, int t, int bar, int p, const Limits& lim) {
  uint32_t ch = 0;
  if ((g.mask[AXIS][p] >> t) & 1ull)
    ch = (FASTONLY || g.fast) ? sweep_line_fast<AXIS>(g, t) : sweep_line3<AXIS>(g, t, lim);
  // Line bits for the phases that follow, OR-reduced over the warp first and
  // then merged with 32-bit shared atomics (a 64-bit shared atomicOr is a CAS
  // loop, which serialises under this contention).
  if (__any_sync(0xffffffffu, ch != 0)) {
    const int c0 = t & 7, c1 = t >> 3;
    unsigned long long ma, mb;
    unsigned long long *da, *db;
    if (AXIS == 0) {  // line (y=c0, z=c1): Y-line k + 8z, Z-line k + 8y (this pass)
      ma = (unsigned long long)ch << (8 * c1), da = &g.mask[1][p];
      mb = (unsigned long long)ch << (8 * c0), db = &g.mask[2][p];
    } else if (AXIS == 1) {  // line (x=c0, z=c1): X-line k + 8z (next), Z-line x + 8k (this)
      ma = (unsigned long long)ch << (8 * c1), da = &g.mask[0][p ^ 1];
      mb = spread8(ch) << c0, db = &g.mask[2][p];
    } else {  // line (x=c0, y=c1): X-line y + 8k, Y-line x + 8k (next pass)
      ma = spread8(ch) << c1, da = &g.mask[0][p ^ 1];
      mb = spread8(ch) << c0, db = &g.mask[1][p ^ 1];
    }
    const uint32_t a0 = __reduce_or_sync(0xffffffffu, uint32_t(ma));
    const uint32_t a1 = __reduce_or_sync(0xffffffffu, uint32_t(ma >> 32));
    const uint32_t b0 = __reduce_or_sync(0xffffffffu, uint32_t(mb));
    const uint32_t b1 = __reduce_or_sync(0xffffffffu, uint32_t(mb >> 32));
    if ((t & 31) == 0) {
      uint32_t* pa = reinterpret_cast<uint32_t*>(da);
      uint32_t* pb = reinterpret_cast<uint32_t*>(db);
      if (a0) atomicOr(pa, a0);
      if (a1) atomicOr(pa + 1, a1);
      if (b0) atomicOr(pb, b0);
      if (b1) atomicOr(pb + 1, b1);
    }
  }
  return ch;
}

// sweep_block (esdf/integrator.cpp:96-139) for one group; masks[.][0] hold the
// initially dirty lines.  Returns whether any voxel changed.
template <bool FASTONLY = false>
__device__ inline bool sweep_block3(GroupSmem& g, int t, int bar, const Limits& lim,
                                    int* n_passes = nullptr) {
  bool block_changed = false;
  for (int pass = 0;; ++pass) {
    if (n_passes) *n_passes = pass + 1;
    const int p = pass & 1;
    uint32_t c = sweep_phase3<0, FASTONLY>(g, t, bar, p, lim);
    group_sync(bar);
    if (t == 0) g.mask[0][p] = 0ull;
    c |= sweep_phase3<1, FASTONLY>(g, t, bar, p, lim);
    group_sync(bar);
    if (t == 0) g.mask[1][p] = 0ull;
    c |= sweep_phase3<2, FASTONLY>(g, t, bar, p, lim);
    const bool pass_changed = group_sync_or(bar, c != 0);
    if (t == 0) g.mask[2][p] = 0ull;
    block_changed |= pass_changed;
    if (!pass_changed) break;
  }
  return block_changed;
}

// A block in registers, reference layout: thread t of the group holds voxels
// lin = 4 * (t + 64 * h) + e (h = 0, 1; e = 0..3) as 3 x 16-byte words each —
// 48 contiguous bytes per thread and h, so the loads and stores coalesce.
struct RawBlock {
  uint32_t w[24];  // voxel (h, e), word f at w[12 * h + 3 * e + f]
};
__device__ inline void raw_load(RawBlock& r, const uint32_t* __restrict__ src, int t) {
  const uint4* s4 = reinterpret_cast<const uint4*>(src);
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const uint4 v = __ldcg(s4 + 3 * (t + 64 * h) + j);
      r.w[12 * h + 4 * j] = v.x;
      r.w[12 * h + 4 * j + 1] = v.y;
      r.w[12 * h + 4 * j + 2] = v.z;
      r.w[12 * h + 4 * j + 3] = v.w;
    }
}
__device__ inline void raw_store(const RawBlock& r, uint32_t* __restrict__ dst, int t) {
  uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      __stcg(d4 + 3 * (t + 64 * h) + j, make_uint4(r.w[12 * h + 4 * j], r.w[12 * h + 4 * j + 1],
                                                   r.w[12 * h + 4 * j + 2], r.w[12 * h + 4 * j + 3]));
}
__device__ inline int raw_lin(int t, int v) { return 4 * (t + 64 * (v >> 2)) + (v & 3); }

// Loads a block (reference layout) into registers; with `reset`, applies
// reset_parented (esdf/integrator.cpp:352-363) on the way in.  Returns, for
// the whole group, whether the block holds a site (after the reset, sites are
// the only givers) and whether it qualifies for the compact format.
__device__ inline void raw_check3(RawBlock& r, int t, int bar, const Limits& lim, bool reset,
                                  bool* any_site_out, bool* fast_out) {
  bool out = lim.max_sq > kFastOff * kFastOff, any_site = false;
#pragma unroll
  for (int v = 0; v < 8; ++v) {
    uint32_t& w0 = r.w[3 * v];
    uint32_t& w1 = r.w[3 * v + 1];
    uint32_t& w2 = r.w[3 * v + 2];
    const uint32_t f = (w2 >> 16) & 0xffu;
    const bool obs = f & VXM_ESDF_OBSERVED, site = f & VXM_ESDF_SITE;
    if (reset && obs && !site && ((w1 | (w2 & 0xffffu)) != 0u)) {
      w0 = uint32_t((f & VXM_ESDF_INSIDE) ? lim.cap_sq : lim.max_sq);
      w1 = 0u;
      w2 &= 0xffff0000u;
    }
    any_site |= obs && site;
    const int px = int(int16_t(w1 & 0xffffu)), py = int(int16_t(w1 >> 16)), pz = int(int16_t(w2 & 0xffffu));
    const bool give = obs && (site || (px | py | pz) != 0);
    out |= w0 >= (1u << 29) || px < -kFastOff || px > kFastOff || py < -kFastOff || py > kFastOff ||
           pz < -kFastOff || pz > kFastOff || (give && w0 != uint32_t(px * px + py * py + pz * pz));
  }
  *fast_out = !group_sync_or(bar, out);
  *any_site_out = reset ? group_sync_or(bar, any_site) : true;
}
__device__ inline void load_raw3(RawBlock& r, const uint32_t* __restrict__ src, int t, int bar,
                                 const Limits& lim, bool reset, bool* any_site_out, bool* fast_out) {
  raw_load(r, src, t);
  raw_check3(r, t, bar, lim, reset, any_site_out, fast_out);
}

// Registers -> working format in shared memory (compact or general).
template <bool FASTONLY = false>
__device__ inline void stage_block3(GroupSmem& g, const RawBlock& r, int t, int bar, const Limits& lim,
                                    bool fast) {
  if (FASTONLY) fast = true;
#pragma unroll
  for (int v = 0; v < 8; ++v) {
    const int si = swz_lin(raw_lin(t, v));
    const uint32_t w0 = r.w[3 * v], w1 = r.w[3 * v + 1], w2 = r.w[3 * v + 2];
    if (fast) {
      const int px = int(int16_t(w1 & 0xffffu)), py = int(int16_t(w1 >> 16)), pz = int(int16_t(w2 & 0xffffu));
      const uint32_t f = (w2 >> 16) & 0xffu;
      const bool obs = f & VXM_ESDF_OBSERVED, site = f & VXM_ESDF_SITE;
      const bool par = (px | py | pz) != 0;
      const uint32_t key = (uint32_t(px + int(kFastBias)) << 20) | (uint32_t(py + int(kFastBias)) << 10) |
                           uint32_t(pz + int(kFastBias));
      const uint32_t lim1 = uint32_t(((f & VXM_ESDF_INSIDE) ? lim.cap_sq : lim.max_sq) + 1);
      const uint32_t tq = w0 < lim1 ? w0 : lim1;
      const bool open = obs && !site && tq > 0u;  // a taker with room to improve
      g.a[0][si] = open ? tq - 1u : 0u;
      g.a[1][si] = open ? (w0 < lim1 ? (key | (par ? 0u : kUnpar)) : 0u) : 0u;
      g.a[2][si] = key;
      g.a[3][si] = (obs && (site || par)) ? w0 - 1u : kNoGive + w0;
      g.a[4][si] = w2 & 0xffff0000u;
    } else {
      g.a[0][si] = w0;
      g.a[1][si] = (((w1 >> 16) ^ 0x8000u) << 16) | ((w2 & 0xffffu) ^ 0x8000u);
      g.a[2][si] = ((w1 & 0xffffu) ^ 0x8000u) | (w2 & 0xffff0000u);
    }
  }
  if (t == 0) g.fast = fast;
  group_sync(bar);
}

// Working format in shared memory -> global block (reference layout).
template <bool FASTONLY = false>
__device__ inline void store_block3(const GroupSmem& g, uint32_t* __restrict__ dst, int t) {
  RawBlock r;
  const bool fast = FASTONLY || g.fast;
#pragma unroll
  for (int v = 0; v < 8; ++v) {
    const int si = swz_lin(raw_lin(t, v));
    uint32_t w0, w1, w2;
    if (fast) {
      const uint32_t key = g.a[2][si], gq = g.a[3][si];
      w0 = (gq - kNoGive) < (1u << 29) ? gq - kNoGive : gq + 1u;
      const uint32_t px = ((key >> 20) & 1023u) - kFastBias, py = ((key >> 10) & 1023u) - kFastBias,
                     pz = (key & 1023u) - kFastBias;
      w1 = (px & 0xffffu) | (py << 16);
      w2 = (pz & 0xffffu) | g.a[4][si];
    } else {
      const uint32_t lo = g.a[1][si], hi = g.a[2][si];
      w0 = g.a[0][si];
      w1 = ((hi & 0xffffu) ^ 0x8000u) | (((lo >> 16) ^ 0x8000u) << 16);
      w2 = ((lo & 0xffffu) ^ 0x8000u) | (hi & 0xffff0000u);
    }
    r.w[3 * v] = w0;
    r.w[3 * v + 1] = w1;
    r.w[3 * v + 2] = w2;
  }
  raw_store(r, dst, t);
}

// ---- cooperative lowering kernel ------------------------------------------------
struct LowerArgs {
  uint32_t* pool[2];
  LayerMeta* meta;
  const int32_t* nbr;
  int fast_only;         // k_lower_xr: every block is compact-format eligible (see launch_lower_xr)
  uint32_t* stamp_dirty[2];
  uint32_t* stamp_lchg;
  int32_t* list[2];
  uint32_t* count;  // [2]
  Limits lim;
  int full;                    // 1: update_esdf (reset + all blocks, ping-pong)
  const int32_t* seeds;        // seeded mode
  const uint32_t* n_seeds;
  DevStatus* status;
  // changed-set output (full mode)
  const int32_t* sorted_slots;
  const uint32_t* stamp_new;
  const uint32_t* stamp_mark;
  uint32_t call_epoch;
  uint32_t lchg_tag;
  uint8_t* out_flags;
  // k_lower_xr: the changed list itself (sorted keys -> ordered compaction), or null
  const uint64_t* sorted_keys;
  uint64_t* out_keys;
  uint32_t* out_n;
  uint32_t* cta_cnt;  // [grid] per-CTA changed counts (scratch)
  unsigned long long* trace;  // optional phase timestamps (VXM_TRACE_LOWER)
  uint32_t* work_ctr;         // [4] dynamic scheduling counters (sweeps, pairs) by parity
  unsigned long long* line_mask;  // [cap][3] lines touched by the last border phase
  uint32_t* stamp_swept;      // [cap] round epoch when the block's sweep was stored
  uint32_t* stamp_pair[3];    // [cap] round epoch when pair (b, b + axis) was done
  uint32_t* stamp_r1same;     // [cap] call epoch: the round-1 reset + copy left the block unchanged
  uint32_t* stamp_quiet;      // [cap] call epoch: untouched by that update, reset its identity (k_lower_xr)
  uint32_t quiet_epoch;       // the previous k_lower_xr update of an unbroken quiet chain, else 0
  uint32_t quiet_dense;       // most blocks were quiet last time: round-1 copies claimed 32 at a time
  int dataflow;               // 1: pair items wait on dependencies; 0: phased barriers
  const uint8_t* site_any;    // [cap] 0: the block holds no site
  uint8_t* site_near;         // [cap] k_lower_xr: bit 0 a site within +-x, bit 1 within the 3x3 (x, y)
  int32_t* r1_list;           // [3][cap] k_lower_xr: round 1's pairs that may change something
  uint32_t r1_compact_min;    // k_lower_xr: maps above this many blocks use r1_list
  uint32_t* r1;               // [8] round-1 split: #site, #no-site, group / warp work counters,
                              //     completed sweeps + copies, x / y / z compact pair counts
  uint32_t* ring;             // cross-round lowering: [0..3] dirty counts, [4..7] sweep claims,
                              // [8..11] pair claims, [12..15] pairs done (by round % 4), [16] last
                              // completed round
  unsigned long long* dlist[2];  // (epoch << 32 | slot) dirty lists by round parity
  uint32_t capacity;             // slots of the layer (bounds every per-round list)
  unsigned long long* pair_face[3];  // [cap][2] (by lower block): face voxels the pair changed
};

__device__ inline uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ inline uint32_t ld_relaxed(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ inline void st_release(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ inline uint32_t atom_add_release(uint32_t* p, uint32_t v) {
  uint32_t r;
  asm volatile("atom.release.gpu.global.add.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "r"(v) : "memory");
  return r;
}
__device__ inline uint32_t atom_add_acq_rel(uint32_t* p, uint32_t v) {
  uint32_t r;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "r"(v) : "memory");
  return r;
}
// Pair stamps carry, besides the round epoch, whether the pair changed its
// lower / upper block (read by the dependent pairs of round 1).
constexpr uint32_t kStampLoChg = 1u << 31, kStampHiChg = 1u << 30, kStampEp = kStampHiChg - 1u;

// Bounded spin (~0.5 s): a missing producer is a bug, never a hang — the
// watchdog flag turns it into VXM_ERR_INTERNAL on the host.  Returns the
// stamp word (epoch + change bits).
__device__ inline uint32_t wait_stamp(const uint32_t* p, uint32_t ep, uint32_t* watchdog,
                                      uint32_t code, int32_t blk) {
  // spin on acquire loads: the block data is read through L2 (ld.cg), so the
  // L1 invalidation of each acquire costs little, and the hand-off saves the
  // separate acquire's round trip (measured: k_lower -2 % on C2 / -1 % on C5)
  uint32_t v;
  for (uint32_t it = 0; ((v = ld_acquire(p)) & kStampEp) != ep; ++it) {
    if (it > (1u << 22)) {
      if (atomicExch(watchdog, 1u) == 0u) {  // record the first expired wait
        watchdog[1] = code;
        watchdog[2] = uint32_t(blk);
        watchdog[3] = ep * 1000u + ((ld_acquire(p) & kStampEp) % 1000u);  // expected, seen
      }
      return 0u;
    }
    __nanosleep(20);
  }
  return v;
}

__device__ inline const EV load_voxel(const uint32_t* pool, int32_t slot, int lin) {
  const uint32_t* p = pool + size_t(slot) * 1536 + lin * 3;
  return ev_unpack(__ldcg(p), __ldcg(p + 1), __ldcg(p + 2));
}
__device__ inline void store_voxel(uint32_t* pool, int32_t slot, int lin, const EV& v) {
  uint32_t* p = pool + size_t(slot) * 1536 + lin * 3;
  __stcg(p, uint32_t(v.sq));
  __stcg(p + 1, ev_w1(v));
  __stcg(p + 2, ev_w2(v));
}

// Round 1, block without sites: reset_parented (esdf/integrator.cpp:352-363)
// leaves it without givers, so its sweep is the identity — one warp copies the
// reset block to the work buffer (lane: voxels 4 * (lane + 32 h) .. + 3).
// Returns (warp-uniform) whether the reset changed any voxel.
__device__ inline bool warp_reset_copy(const uint32_t* __restrict__ src, uint32_t* __restrict__ dst,
                                       int lane, const Limits& lim) {
  const uint4* s4 = reinterpret_cast<const uint4*>(src);
  uint4* d4 = reinterpret_cast<uint4*>(dst);
  uint32_t w[48];
#pragma unroll
  for (int h = 0; h < 4; ++h)
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const uint4 v = __ldcg(s4 + 3 * (lane + 32 * h) + j);
      w[12 * h + 4 * j] = v.x;
      w[12 * h + 4 * j + 1] = v.y;
      w[12 * h + 4 * j + 2] = v.z;
      w[12 * h + 4 * j + 3] = v.w;
    }
  bool changed = false;
#pragma unroll
  for (int v = 0; v < 16; ++v) {
    const uint32_t f = (w[3 * v + 2] >> 16) & 0xffu;
    if ((f & VXM_ESDF_OBSERVED) && !(f & VXM_ESDF_SITE) && ((w[3 * v + 1] | (w[3 * v + 2] & 0xffffu)) != 0u)) {
      const uint32_t sq = uint32_t((f & VXM_ESDF_INSIDE) ? lim.cap_sq : lim.max_sq);
      changed = true;  // a parented voxel: its offset is cleared
      w[3 * v] = sq;
      w[3 * v + 1] = 0u;
      w[3 * v + 2] &= 0xffff0000u;
    }
  }
#pragma unroll
  for (int h = 0; h < 4; ++h)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      __stcg(d4 + 3 * (lane + 32 * h) + j, make_uint4(w[12 * h + 4 * j], w[12 * h + 4 * j + 1],
                                                     w[12 * h + 4 * j + 2], w[12 * h + 4 * j + 3]));
  return __any_sync(0xffffffffu, changed);
}

// ---- lowering v3: group-per-block sweeps with line masks --------------------------
constexpr int kL3Threads = 256;

constexpr int kL3Groups = kL3Threads / 64;

__device__ inline void line_bits(int x, int y, int z, unsigned long long m[3]) {
  m[0] |= 1ull << (y + 8 * z);  // X-line through the voxel
  m[1] |= 1ull << (x + 8 * z);  // Y-line
  m[2] |= 1ull << (x + 8 * y);  // Z-line
}
__device__ inline unsigned long long warp_or64(unsigned long long v) {
  const uint32_t lo = __reduce_or_sync(0xffffffffu, uint32_t(v));
  const uint32_t hi = __reduce_or_sync(0xffffffffu, uint32_t(v >> 32));
  return (unsigned long long)hi << 32 | lo;
}


}  // namespace vxm
