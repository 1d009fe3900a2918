// View candidates + block allocation.
//
// Reference: blocks_in_view (proj/src/sensor/view.cpp:61-111), cast_ray
// (:45-57), traverse_grid (proj/include/voxmap/sensor/traversal.hpp:29-73),
// dilate_and_sort (view.cpp:25-41), allocation loop (integrator.cpp:84-87).
//
// B200 design (no hash sets, no sort):
//   K_rays    one thread per camera tile (or LiDAR pixel) runs the exact FP64
//             Amanatides-Woo DDA and sets bits in a dense bitmap over the
//             cube of cells reachable from the sensor's cell (L2-resident).
//   K_dilate  one thread per 32-cell bitmap word computes the 27-neighbour
//             dilation with shifts/ORs, looks every candidate up in the
//             layer's block hash, and emits (key, slot) in lexicographic
//             (x, y, z) order through a single-pass decoupled look-back scan;
//             new blocks get slots num_blocks + rank(new) in sorted order and
//             are inserted into the hash in the same pass.  The bitmap layout
//             (x slowest, z fastest) makes word order == GridIndex order, so
//             the candidate list is sorted for free.
#include <math_constants.h>

#include <cmath>
#include <cstring>
#include <vector>

#include "runtime.cuh"
#include "scan.cuh"

namespace vxm {

struct Cube {
  int32_t ox, oy, oz;  // cell of index 0 along each axis (origin cell - r)
  int32_t S;           // side in cells
  int32_t SZw;         // 32-bit words per z-row
  uint32_t* bits;
  __device__ inline bool locate(int32_t x, int32_t y, int32_t z, uint32_t& word,
                                uint32_t& mask) const {
    const int32_t dx = x - ox, dy = y - oy, dz = z - oz;
    if (dx < 0 || dy < 0 || dz < 0 || dx >= S || dy >= S || dz >= S) return false;
    word = (uint32_t(dx) * uint32_t(S) + uint32_t(dy)) * uint32_t(SZw) + uint32_t(dz >> 5);
    mask = 1u << (dz & 31);
    return true;
  }
};

// Pinned-order FP64 helpers (no FMA contraction: TU compiled with --fmad=false,
// and the explicit __d*_rn intrinsics make the intent independent of flags).
__device__ inline double sum3(double a0, double a1, double a2) {
  return __dadd_rn(a0, __dadd_rn(a1, a2));
}
__device__ inline void pose_apply(const vxm_pose& T, double x, double y, double z, double out[3]) {
#pragma unroll
  for (int i = 0; i < 3; ++i)
    out[i] = __dadd_rn(sum3(__dmul_rn(T.R[3 * i], x), __dmul_rn(T.R[3 * i + 1], y),
                            __dmul_rn(T.R[3 * i + 2], z)),
                       T.t[i]);
}

// Sets the cell's bit with a fire-and-forget RED (no load on the DDA's critical
// path).  With DEDUP (LiDAR: 131k rays, thousands per warp-step near the
// sensor) lanes at the same step that hit the same word combine their bits and
// one of them issues the RED, so the hot words near the sensor do not
// serialise in L2; the camera's 4800 rays gain nothing from it.
template <bool DEDUP>
__device__ inline void mark_cell(const Cube& c, int32_t x, int32_t y, int32_t z,
                                 DevStatus* status) {
  uint32_t w = 0xffffffffu, m = 0u;
  const bool ok = c.locate(x, y, z, w, m);
  uint32_t mm = m;
  if (DEDUP) {
    const unsigned act = __activemask();
    const unsigned peers = __match_any_sync(act, w);
    mm = __reduce_or_sync(peers, m);
    if ((threadIdx.x & 31) != __ffs(peers) - 1) return;
  }
  if (!ok) {
    atomicOr(&status->bitmap_overflow, 1u);
    return;
  }
  atomicOr(c.bits + w, mm);
}

// traverse_grid — traversal.hpp:29-73, visiting into the bitmap.
template <bool DEDUP>
__device__ void traverse(const double s[3], const double e[3], double cs, const Cube& cube,
                         DevStatus* status) {
  double d[3], t_max[3], t_delta[3];
  int cell[3], end_cell[3], step[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    d[i] = __dsub_rn(e[i], s[i]);
    cell[i] = int(floor(__ddiv_rn(s[i], cs)));
    end_cell[i] = int(floor(__ddiv_rn(e[i], cs)));
    step[i] = 0;
    t_max[i] = CUDART_INF;
    t_delta[i] = CUDART_INF;
  }
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    if (d[i] > 0.0) {
      step[i] = 1;
      t_delta[i] = __ddiv_rn(cs, d[i]);
      t_max[i] = __ddiv_rn(__dsub_rn(__dmul_rn(double(cell[i] + 1), cs), s[i]), d[i]);
    } else if (d[i] < 0.0) {
      step[i] = -1;
      t_delta[i] = __ddiv_rn(-cs, d[i]);
      t_max[i] = __ddiv_rn(__dsub_rn(__dmul_rn(double(cell[i]), cs), s[i]), d[i]);
    }
  }
  mark_cell<DEDUP>(cube, cell[0], cell[1], cell[2], status);
  int guard = abs(end_cell[0] - cell[0]) + abs(end_cell[1] - cell[1]) +
              abs(end_cell[2] - cell[2]) + 3;
  // the stepping state in named registers (dynamic indexing of the arrays
  // would put them in local memory, one load per step on the critical path)
  int cx = cell[0], cy = cell[1], cz = cell[2];
  double tx = t_max[0], ty = t_max[1], tz = t_max[2];
  // DEDUP only over a ray's first kDedupSteps cells: near the sensor the rays
  // of a warp share cells (one RED per word instead of one per ray), farther
  // out they have spread and the match costs more than the REDs it saves
  // (measured on C3, 0.8 m cells: k_rays_lidar 88 us always, 77 / 58 / 47 /
  // 46 / 61 us for 8 / 16 / 32 / 48 / 96 cells)
  constexpr int kDedupSteps = 48;
  int steps = 0;
  while (guard-- > 0) {
    // axis = 0; if (t_max[1] < t_max[0]) axis = 1; if (t_max[2] < t_max[axis]) axis = 2;
    const bool y_first = ty < tx;
    const double t_xy = y_first ? ty : tx;
    const bool z_first = tz < t_xy;
    const double t_min = z_first ? tz : t_xy;
    if (t_min > 1.0) break;
    if (z_first) {
      cz += step[2];
      tz = __dadd_rn(tz, t_delta[2]);
    } else if (y_first) {
      cy += step[1];
      ty = __dadd_rn(ty, t_delta[1]);
    } else {
      cx += step[0];
      tx = __dadd_rn(tx, t_delta[0]);
    }
    if (DEDUP && ++steps <= kDedupSteps) mark_cell<true>(cube, cx, cy, cz, status);
    else mark_cell<false>(cube, cx, cy, cz, status);
  }
}

__device__ inline bool valid_depth(float d) { return d > 0.0f && isfinite(d); }

// reach = std::min(depth, max_int) + truncation — view.cpp:49-51
__device__ inline double ray_reach(double depth, double max_int, double trunc) {
  const double capped = max_int < depth ? max_int : depth;
  return __dadd_rn(capped, trunc);
}

// Camera: ONE WARP PER PIXEL TILE — view.cpp:66-91 — with a lane-parallel,
// exact traverse_grid (traversal.hpp:29-73).
//
// The serial DDA takes, at each step, the smallest of the three next-crossing
// parameters t_x, t_y, t_z (ties to the lowest axis), steps that axis and
// adds its t_delta — so the visited cells are the prefix (value <= 1, fewer
// than `guard` steps) of the STABLE MERGE of the three per-axis sequences
// t_a(i+1) = t_a(i) + t_delta_a (each rounded exactly as the serial loop
// rounds it).  Lanes 0-2 generate those sequences (one FP64 add per element,
// into shared memory); then every lane takes elements, finds the element's
// merge position by binary search in the two other sequences (ties: a
// lower axis precedes) and, if that position is below `guard`, marks the cell
// start + (counts of the three axes up to it).  The set of marked cells is the
// serial loop's, bit for bit; the per-ray latency drops from ~35 dependent
// steps to one sequence scan plus a search.  Rays with more than
// kRayMaxSteps crossings on one axis (none at the BASELINE configs) run the
// serial loop.  Every ray starts in the sensor's cell, so the cells near it
// are hit by thousands of rays: they are ORed into a per-CTA shared bitmap of
// the 16^3 cells around the sensor and flushed once per CTA.
constexpr int kRayWarps = 8;       // rays (camera tiles) per 256-thread CTA
constexpr int kRayMaxSteps = 64;   // stored crossings per axis
constexpr int kLocR = 8;           // near-sensor cube: cells [c - 8, c + 8) per axis

struct RaySmem {
  double t[kRayWarps][3][kRayMaxSteps];
  uint32_t loc[16 * 16 * 16 / 32];
};

// Count of entries of the increasing sequence q[0..n) that are < v (or <= v).
__device__ inline int seq_rank(const double* q, int n, double v, bool inclusive) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    const double x = q[mid];
    if (inclusive ? !(v < x) : x < v) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// sc: the sensor's cell floor(t / cs) (every ray's start, computed on the host
// with the same IEEE division); dirs: per tile the unprojection factors
// ((u - cu) / fu, (v - cv) / fv) of camera.hpp:52-55 (frame-independent, host
// LUT, identical IEEE operations).
__global__ void __launch_bounds__(256) k_rays_camera(const float* __restrict__ depth, int W, int H,
                                                     int tile, const double2* __restrict__ dirs,
                                                     vxm_pose T, int3 sc3, double cs, double max_int,
                                                     double trunc, Cube cube, DevStatus* status) {
  pdl_wait();  // see launch_pdl
  pdl_trigger();
  __shared__ RaySmem sm;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 128; i += blockDim.x) sm.loc[i] = 0u;
  const int sc[3] = {sc3.x, sc3.y, sc3.z};
  const int lx = sc[0] - kLocR - cube.ox, ly = sc[1] - kLocR - cube.oy, lz = sc[2] - kLocR - cube.oz;
  const bool use_loc = lx >= 0 && ly >= 0 && lz >= 0 && lx + 2 * kLocR <= cube.S &&
                       ly + 2 * kLocR <= cube.S && lz + 2 * kLocR <= cube.S;
  __syncthreads();
  auto mark = [&](int x, int y, int z) {
    const int dx = x - (sc[0] - kLocR), dy = y - (sc[1] - kLocR), dz = z - (sc[2] - kLocR);
    if (use_loc && unsigned(dx) < 16u && unsigned(dy) < 16u && unsigned(dz) < 16u) {
      const int b = dz + 16 * (dy + 16 * dx);
      atomicOr(&sm.loc[b >> 5], 1u << (b & 31));
    } else {
      uint32_t w, m;
      if (cube.locate(x, y, z, w, m)) atomicOr(cube.bits + w, m);
      else atomicOr(&status->bitmap_overflow, 1u);
    }
  };

  const int tiles_x = (W + tile - 1) / tile;
  const int tiles_y = (H + tile - 1) / tile;
  // grid-stride over the tiles: one resident wave, no tail wave
  for (int t = blockIdx.x * kRayWarps + warp; t < tiles_x * tiles_y; t += gridDim.x * kRayWarps) {
    const int col0 = (t % tiles_x) * tile, row0 = (t / tiles_x) * tile;
    const int row1 = min(row0 + tile, H), col1 = min(col0 + tile, W);
    const int tw = col1 - col0, npx = tw * (row1 - row0);
    // tile_max over the valid depths (d > 0 and finite): positive floats
    // order like their bit patterns
    uint32_t mb = 0u;
    for (int q = lane; q < npx; q += 32) {
      const float d = __ldg(depth + size_t(row0 + q / tw) * W + (col0 + q % tw));
      if (valid_depth(d)) mb = max(mb, __float_as_uint(d));
    }
    mb = __reduce_max_sync(0xffffffffu, mb);
    const float tile_max = __uint_as_float(mb);
    if (!(tile_max > 0.0f)) continue;
    const double reach = ray_reach(double(tile_max), max_int, trunc);
    // CameraIntrinsics::unproject — camera.hpp:52-55: (u - cu) / fu * depth
    const double2 dr = __ldg(dirs + t);
    const double end_S[3] = {__dmul_rn(dr.x, reach), __dmul_rn(dr.y, reach), reach};
    double e[3];
    pose_apply(T, end_S[0], end_S[1], end_S[2], e);
    // traverse_grid set-up (traversal.hpp:41-58), as the serial traverse():
    // lane a < 3 computes axis a
    const int ax = lane < 3 ? lane : 0;
    const double ea = ax == 0 ? e[0] : (ax == 1 ? e[1] : e[2]);
    const double sa = T.t[ax];
    const int sca = ax == 0 ? sc[0] : (ax == 1 ? sc[1] : sc[2]);
    const double dd = __dsub_rn(ea, sa);
    const int endc = int(floor(__ddiv_rn(ea, cs)));
    int stp = 0;
    double tmax = CUDART_INF, tdel = CUDART_INF;
    if (dd > 0.0) {
      stp = 1;
      tdel = __ddiv_rn(cs, dd);
      tmax = __ddiv_rn(__dsub_rn(__dmul_rn(double(sca + 1), cs), sa), dd);
    } else if (dd < 0.0) {
      stp = -1;
      tdel = __ddiv_rn(-cs, dd);
      tmax = __ddiv_rn(__dsub_rn(__dmul_rn(double(sca), cs), sa), dd);
    }
    int ad = lane < 3 ? abs(endc - sca) : 0;
    const int guard = __reduce_add_sync(0xffffffffu, ad) + 3;
    const int step[3] = {__shfl_sync(0xffffffffu, stp, 0), __shfl_sync(0xffffffffu, stp, 1),
                         __shfl_sync(0xffffffffu, stp, 2)};
    // lanes 0-2: the crossings of axis `lane` with t <= 1 (at most guard)
    int n = 0;
    bool more = false;
    if (lane < 3) {
      double tv = tmax;
      double* q = sm.t[warp][lane];
      while (n < guard && tv <= 1.0) {
        if (n == kRayMaxSteps) {
          more = true;
          break;
        }
        q[n++] = tv;
        tv = __dadd_rn(tv, tdel);
      }
    }
    const int nx = __shfl_sync(0xffffffffu, n, 0), ny = __shfl_sync(0xffffffffu, n, 1),
              nz = __shfl_sync(0xffffffffu, n, 2);
    __syncwarp();
    if (__any_sync(0xffffffffu, more)) {
      if (lane == 0) traverse<false>(T.t, e, cs, cube, status);  // long ray: serial loop
    } else {
      if (lane == 0) mark(sc[0], sc[1], sc[2]);
      const double* qx = sm.t[warp][0];
      const double* qy = sm.t[warp][1];
      const double* qz = sm.t[warp][2];
      for (int k = lane; k < nx + ny + nz; k += 32) {
        int a, i;
        if (k < nx) a = 0, i = k;
        else if (k < nx + ny) a = 1, i = k - nx;
        else a = 2, i = k - nx - ny;
        const double val = sm.t[warp][a][i];
        // merge position: lower axes with equal t go first
        const int cx = a == 0 ? i + 1 : seq_rank(qx, nx, val, true);
        const int cy = a == 1 ? i + 1 : seq_rank(qy, ny, val, a > 1);
        const int cz = a == 2 ? i + 1 : seq_rank(qz, nz, val, false);
        if (cx + cy + cz - 1 < guard) mark(sc[0] + step[0] * cx, sc[1] + step[1] * cy, sc[2] + step[2] * cz);
      }
    }
    __syncwarp();  // the warp's sequences are read before the next tile rewrites them
  }
  __syncthreads();
  if (use_loc) {  // flush the near-sensor cube: 2 rows of 16 z-cells per word
    for (int w = threadIdx.x; w < 128; w += blockDim.x) {
      const uint32_t bits = sm.loc[w];
      if (!bits) continue;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint32_t zb = (bits >> (16 * h)) & 0xffffu;
        if (!zb) continue;
        const int row = 2 * w + h, dx = row >> 4, dy = row & 15;
        const uint32_t base = (uint32_t(lx + dx) * uint32_t(cube.S) + uint32_t(ly + dy)) * uint32_t(cube.SZw);
        const int sh = lz & 31;
        atomicOr(cube.bits + base + uint32_t(lz >> 5), zb << sh);
        if (sh > 16) atomicOr(cube.bits + base + uint32_t(lz >> 5) + 1u, zb >> (32 - sh));
      }
    }
  }
}

// LiDAR: one thread per valid pixel — view.cpp:94-111.  The per-pixel unit
// directions (lidar.hpp:68-74, glibc sin/cos) come from a host-built LUT.
__global__ void k_rays_lidar(const float* __restrict__ depth, int W, int H,
                             const double* __restrict__ dirs, vxm_pose T, double cs,
                             double max_int, double trunc, Cube cube, DevStatus* status) {
  pdl_wait();  // see launch_pdl
  pdl_trigger();
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= W * H) return;
  const float d = __ldg(depth + p);
  if (!valid_depth(d)) return;
  const double reach = ray_reach(double(d), max_int, trunc);
  const double end_S[3] = {__dmul_rn(__ldg(dirs + 3 * p), reach),
                           __dmul_rn(__ldg(dirs + 3 * p + 1), reach),
                           __dmul_rn(__ldg(dirs + 3 * p + 2), reach)};
  double end_L[3];
  pose_apply(T, end_S[0], end_S[1], end_S[2], end_L);
  traverse<true>(T.t, end_L, cs, cube, status);
}

__device__ inline uint32_t zdilate(uint32_t prev, uint32_t w, uint32_t next) {
  return w | (w << 1) | (w >> 1) | (prev >> 31) | (next << 31);
}

__device__ inline bool owned(int32_t x, int rank, int world, int slab) {
  if (world <= 1) return true;
  const int32_t q = x >= 0 ? x / slab : -((-x + slab - 1) / slab);
  return ((q % world) + world) % world == rank;
}

struct AllocArgs {
  HashView hash;           // mask == 0 and keys == nullptr: no allocation
  uint64_t* slot_keys;
  LayerMeta* meta;
  uint32_t capacity;       // physical pool slots
  uint64_t max_blocks;     // Layer::max_blocks
};

// Dilation + ordered emission + fused allocation.  One thread per 32-cell word
// computes the dilation; the tile's candidates are then processed one per
// thread (so the hash look-ups of a tile are issued in parallel, not as a
// serial chain per word): look-up, new-block ranking, one look-back for the
// (candidates, new blocks) prefix, ordered output with slot assignment and
// hash insertion of the new blocks.
constexpr int kDilThreads = 256;
constexpr int kDilMaxCand = kDilThreads * 32;

struct DilTile {
  uint32_t dil[kDilThreads];  // dilated word of each thread
  uint32_t off[kDilThreads];  // exclusive prefix of the words' candidate counts
};

// Candidate `idx` of the tile: the word that holds it (largest o with
// off[o] <= idx) and the cell's packed key.
__device__ inline uint64_t tile_candidate(const DilTile& d, uint32_t idx, uint32_t tile,
                                          const Cube& cube) {
  int o = 0;
#pragma unroll
  for (int step = kDilThreads / 2; step >= 1; step >>= 1)
    if (d.off[o + step] <= idx) o += step;
  const int bit = int(__fns(d.dil[o], 0u, int(idx - d.off[o]) + 1));
  const uint32_t wi = tile * kDilThreads + uint32_t(o);
  const int32_t wz = int32_t(wi % uint32_t(cube.SZw));
  const uint32_t t = wi / uint32_t(cube.SZw);
  const int32_t dy = int32_t(t % uint32_t(cube.S)), dx = int32_t(t / uint32_t(cube.S));
  return pack_key(cube.ox + dx, cube.oy + dy, cube.oz + wz * 32 + bit);
}

__global__ void __launch_bounds__(kDilThreads) k_dilate_alloc(Cube cube, uint32_t n_words, AllocArgs al,
                                                              int rank, int world, int slab,
                                                              uint64_t* __restrict__ cand_keys,
                                                              int32_t* __restrict__ cand_slots,
                                                              DevStatus* status, ScanTiles st,
                                                              uint32_t* __restrict__ clear_bits,
                                                              uint32_t clear_words) {
  pdl_wait();  // see launch_pdl
  pdl_trigger();
  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_scan[64];
  __shared__ uint32_t s_pre[2];
  __shared__ uint32_t s_base, s_nnew;
  __shared__ DilTile s_d;
  __shared__ int32_t s_slot[kDilMaxCand];  // found slot, or -2 - (tile-local new rank)
  scan_prepare_next(st);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < clear_words; i += gridDim.x * blockDim.x)
    clear_bits[i] = 0u;  // the next call's bitmap
  const uint32_t tile = scan_take_tile(st, &s_tile);
  const uint32_t wi = tile * blockDim.x + threadIdx.x;
  const bool do_alloc = al.hash.keys != nullptr;
  uint32_t dil = 0;
  if (wi < n_words) {
    const int32_t S = cube.S, SZw = cube.SZw;
    const int32_t wz = int32_t(wi % uint32_t(SZw));
    const uint32_t t = wi / uint32_t(SZw);
    const int32_t dy = int32_t(t % uint32_t(S)), dx = int32_t(t / uint32_t(S));
    for (int ddx = -1; ddx <= 1; ++ddx) {
      const int32_t xx = dx + ddx;
      if (xx < 0 || xx >= S) continue;
      for (int ddy = -1; ddy <= 1; ++ddy) {
        const int32_t yy = dy + ddy;
        if (yy < 0 || yy >= S) continue;
        const uint32_t* row = cube.bits + (uint32_t(xx) * uint32_t(S) + uint32_t(yy)) * uint32_t(SZw);
        const uint32_t w = row[wz];
        const uint32_t prev = wz > 0 ? row[wz - 1] : 0u;
        const uint32_t next = wz + 1 < SZw ? row[wz + 1] : 0u;
        dil |= zdilate(prev, w, next);
      }
    }
    const int32_t zbits = S - wz * 32;  // valid bits in this word
    if (zbits < 32) dil &= (zbits <= 0 ? 0u : ((1u << zbits) - 1u));
    if (!owned(cube.ox + dx, rank, world, slab)) dil = 0;
  }
  uint32_t ea, eb, n_cand, tb;
  block_scan2(__popc(dil), 0u, ea, eb, n_cand, tb, s_scan);
  s_d.dil[threadIdx.x] = dil;
  s_d.off[threadIdx.x] = ea;
  if (threadIdx.x == 0) {
    s_base = do_alloc ? al.meta->num_blocks : 0u;
    s_nnew = 0u;
  }
  __syncthreads();
  // look-ups, one candidate per thread; new blocks ranked in key order
  if (do_alloc) {
    for (uint32_t c0 = 0; c0 < n_cand; c0 += kDilThreads) {
      const uint32_t idx = c0 + threadIdx.x;
      int32_t found = 0;
      if (idx < n_cand) found = hash_find_rw(al.hash, tile_candidate(s_d, idx, tile, cube));
      const bool is_new = idx < n_cand && found < 0;
      uint32_t rn, rb, tn, tb2;
      block_scan2(is_new ? 1u : 0u, 0u, rn, rb, tn, tb2, s_scan);
      if (idx < n_cand) s_slot[idx] = is_new ? -2 - int32_t(s_nnew + rn) : found;
      __syncthreads();
      if (threadIdx.x == 0) s_nnew += tn;
      __syncthreads();
    }
  }
  const uint32_t n_new = s_nnew;
  if (threadIdx.x < 32) {  // warp 0: look-back
    uint32_t pa, pb;
    scan_lookback(st, tile, n_cand, n_new, pa, pb);
    if (threadIdx.x == 0) {
      s_pre[0] = pa;
      s_pre[1] = pb;
    }
  }
  __syncthreads();
  const uint32_t base = s_base;
  const uint64_t limit = al.capacity < al.max_blocks ? uint64_t(al.capacity) : al.max_blocks;
  for (uint32_t idx = threadIdx.x; idx < n_cand; idx += kDilThreads) {
    const uint64_t k = tile_candidate(s_d, idx, tile, cube);
    int32_t slot = 0;
    if (do_alloc) {
      slot = s_slot[idx];
      if (slot <= -2) {
        const uint64_t s = uint64_t(base) + s_pre[1] + uint32_t(-2 - slot);
        if (s < limit) {
          hash_insert(al.hash, k, int32_t(s));
          al.slot_keys[s] = k;
          slot = int32_t(s) | int32_t(0x80000000u);
        } else {
          slot = -1;
        }
      }
    }
    cand_keys[s_pre[0] + idx] = k;
    cand_slots[s_pre[0] + idx] = slot;
  }
  // The last tile publishes totals (all earlier tiles have read s_base: they
  // published before this tile's look-back could complete).
  if (threadIdx.x == 0 && tile == gridDim.x - 1) {
    const uint32_t total_c = s_pre[0] + n_cand, total_n = s_pre[1] + n_new;
    status->n_candidates = total_c;
    status->n_new = total_n;
    if (do_alloc) {
      const uint64_t want = uint64_t(base) + total_n;
      // Physical pool too small (and the logical limit not yet reached):
      // the host grows the pool and re-runs; otherwise MapCapacityError.
      if (want > al.capacity && al.capacity < al.max_blocks) status->pool_overflow = 1u;
      if (want > al.max_blocks) status->capacity_error = 1u;
      al.meta->num_blocks = uint32_t(want < limit ? want : limit);
    }
  }
}

// ---- host driver ------------------------------------------------------------------
// Per camera tile: ((u - cu) / fu, (v - cv) / fv) at the tile centre
// (view.cpp:75-80 with camera.hpp:52-55), the frame-independent part of
// every camera ray.
static void ensure_camera_lut(Context* ctx, const vxm_camera& cam, int W, int H, int tile) {
  if (ctx->cam_lut_valid && std::memcmp(&ctx->cam_key, &cam, sizeof cam) == 0 && ctx->cam_key_w == W &&
      ctx->cam_key_h == H && ctx->cam_key_tile == tile)
    return;
  const int tx = (W + tile - 1) / tile, ty = (H + tile - 1) / tile;
  std::vector<double> d(size_t(tx) * ty * 2);
  for (int t = 0; t < tx * ty; ++t) {
    const int col0 = (t % tx) * tile, row0 = (t / tx) * tile;
    const int row1 = std::min(row0 + tile, H), col1 = std::min(col0 + tile, W);
    const double u = 0.5 * double(col0 + col1), v = 0.5 * double(row0 + row1);
    d[2 * size_t(t)] = (u - cam.cu) / cam.fu;
    d[2 * size_t(t) + 1] = (v - cam.cv) / cam.fv;
  }
  ctx->cam_dirs.ensure(d.size() * sizeof(double));
  VXM_CUDA(cudaMemcpyAsync(ctx->cam_dirs.p, d.data(), d.size() * sizeof(double), cudaMemcpyHostToDevice,
                           ctx->stream));
  VXM_CUDA(cudaStreamSynchronize(ctx->stream));
  ctx->cam_key = cam;
  ctx->cam_key_w = W;
  ctx->cam_key_h = H;
  ctx->cam_key_tile = tile;
  ctx->cam_lut_valid = true;
}

static void ensure_lidar_lut(Context* ctx, const vxm_lidar& li) {
  if (ctx->lut_valid && std::memcmp(&ctx->lut_key, &li, sizeof li) == 0) return;
  const int W = li.num_azimuth, H = li.num_elevation;
  std::vector<double> dirs(size_t(W) * H * 3);
  // LidarIntrinsics::ray_direction(col + 0.5, row + 0.5) — lidar.hpp:68-74,
  // evaluated with the host libm exactly as the reference does.
  const double raz = li.azimuth_fov / li.num_azimuth;
  const double rel = li.elevation_fov / li.num_elevation;
  for (int row = 0; row < H; ++row)
    for (int col = 0; col < W; ++col) {
      const double az = li.azimuth_start + (col + 0.5) * raz;
      const double polar = li.elevation_start + (row + 0.5) * rel;
      const double sp = std::sin(polar);
      double* d = &dirs[(size_t(row) * W + col) * 3];
      d[0] = std::cos(az) * sp;
      d[1] = std::sin(az) * sp;
      d[2] = std::cos(polar);
    }
  ctx->lidar_dirs.ensure(dirs.size() * sizeof(double));
  VXM_CUDA(cudaMemcpyAsync(ctx->lidar_dirs.p, dirs.data(), dirs.size() * sizeof(double),
                           cudaMemcpyHostToDevice, ctx->stream));
  VXM_CUDA(cudaStreamSynchronize(ctx->stream));
  ctx->lut_key = li;
  ctx->lut_valid = true;
}

void run_view(Context* ctx, const ViewArgs& a, Layer* L, uint32_t* cand_cap_out) {
  const double cs = a.block_size;
  // Cube of cells any ray (plus one dilation ring) can reach.
  double norm_max;
  const double reach_max = a.cfg.max_integration_distance + a.cfg.truncation;
  if (!a.lidar) {
    const double ax = std::max(std::fabs(a.cam.cu), std::fabs(a.width - a.cam.cu)) / std::fabs(a.cam.fu);
    const double ay = std::max(std::fabs(a.cam.cv), std::fabs(a.height - a.cam.cv)) / std::fabs(a.cam.fv);
    norm_max = std::fabs(reach_max) * std::sqrt(1.0 + ax * ax + ay * ay);
  } else {
    norm_max = std::fabs(reach_max);
  }
  norm_max = norm_max * 1.0001 + 1e-9;
  const double rc = std::ceil(norm_max / cs) + 3.0;
  if (!(rc < 1e6)) throw Error(VXM_ERR_INVALID_ARGUMENT, "view volume too large");
  const int32_t r = int32_t(rc);
  const int32_t S = 2 * r + 1;
  const int32_t SZw = (S + 31) / 32;
  const uint64_t n_words = uint64_t(S) * uint64_t(S) * uint64_t(SZw);
  if (n_words * 4 > (uint64_t(1) << 31))
    throw Error(VXM_ERR_INVALID_ARGUMENT,
                "view volume too large for the candidate bitmap (max_integration_distance / block "
                "size ratio)");
  Cube cube;
  const int64_t ocx = int64_t(std::floor(a.T_LS.t[0] / cs));
  const int64_t ocy = int64_t(std::floor(a.T_LS.t[1] / cs));
  const int64_t ocz = int64_t(std::floor(a.T_LS.t[2] / cs));
  if (!coord_ok(ocx - r) || !coord_ok(ocx + r) || !coord_ok(ocy - r) || !coord_ok(ocy + r) ||
      !coord_ok(ocz - r) || !coord_ok(ocz + r))
    throw Error(VXM_ERR_INVALID_ARGUMENT, "sensor position outside the supported block range");
  cube.ox = int32_t(ocx - r);
  cube.oy = int32_t(ocy - r);
  cube.oz = int32_t(ocz - r);
  cube.S = S;
  cube.SZw = SZw;
  // This call's bitmap was zeroed by the previous call's k_dilate_alloc (or is
  // zeroed here); k_dilate_alloc zeroes the other one for the next call.
  const int bp = ctx->bitmap_parity;
  ctx->bitmap_parity ^= 1;
  DevBuf& bm = ctx->bitmap[bp];
  if (bm.bytes < n_words * 4) ctx->bitmap_clean[bp] = 0;
  bm.ensure(n_words * 4);
  cube.bits = bm.as<uint32_t>();
  if (ctx->bitmap_clean[bp] < n_words) {
    VXM_CUDA(cudaMemsetAsync(cube.bits, 0, n_words * 4, ctx->stream));
    ctx->count_launch();
  }
  ctx->bitmap_clean[bp] = 0;
  DevBuf& other = ctx->bitmap[bp ^ 1];
  const uint64_t other_words = other.bytes / 4;

  host_trace_dev(ctx, "memset");
  if (!a.lidar) {
    const int tile = std::max(1, a.cfg.pixel_subsample);
    const int nt = ((a.width + tile - 1) / tile) * ((a.height + tile - 1) / tile);
    if (nt > 0) {
      ensure_camera_lut(ctx, a.cam, a.width, a.height, tile);
      const int3 sc3 = make_int3(int(std::floor(a.T_LS.t[0] / cs)), int(std::floor(a.T_LS.t[1] / cs)),
                                 int(std::floor(a.T_LS.t[2] / cs)));
      ctx->prof_begin("k_rays");
      // one resident wave of 8-warp CTAs; warps loop over the tiles
      const int per_sm = ctx->resident_per_sm((const void*)k_rays_camera, 32 * kRayWarps);
      launch_pdl(ctx->stream, k_rays_camera,
                 dim3(std::max<uint32_t>(1u, std::min<uint32_t>(ceil_div(nt, kRayWarps), uint32_t(per_sm * ctx->sm_count)))),
                 dim3(32 * kRayWarps), 0, 
          a.depth_dev, a.width, a.height, tile, ctx->cam_dirs.as<const double2>(), a.T_LS, sc3, cs,
          a.cfg.max_integration_distance, a.cfg.truncation, cube, ctx->status_w());
      ctx->prof_end();
      ctx->count_launch();
    }
  } else {
    ensure_lidar_lut(ctx, a.li);
    const int np = a.width * a.height;
    if (np > 0) {
      ctx->prof_begin("k_rays");
      launch_pdl(ctx->stream, k_rays_lidar, dim3(ceil_div(np, 64)), dim3(64), 0, 
          a.depth_dev, a.width, a.height, ctx->lidar_dirs.as<double>(), a.T_LS, cs,
          a.cfg.max_integration_distance, a.cfg.truncation, cube, ctx->status_w());
      ctx->prof_end();
      ctx->count_launch();
    }
  }
  check_launch(ctx, "k_rays");

  // Candidate arrays: bounded by the cube's cell count.
  const uint64_t max_cand = uint64_t(S) * S * S;
  const uint32_t cand_cap = uint32_t(std::min<uint64_t>(max_cand, (uint64_t(1) << 31) - 1));
  ctx->cand_keys.ensure(sizeof(uint64_t) * cand_cap);
  ctx->cand_slots.ensure(sizeof(int32_t) * cand_cap);
  AllocArgs al{};
  if (L) {
    al.hash = L->hash;
    al.slot_keys = L->slot_keys;
    al.meta = L->meta;
    al.capacity = L->capacity;
    al.max_blocks = L->max_blocks;
  }
  const uint32_t tiles = ceil_div(n_words, 256);
  const ScanTiles st = ctx->next_scan(tiles);
  host_trace_dev(ctx, "rays");
  ctx->prof_begin("k_dilate_alloc");
  launch_pdl(ctx->stream, k_dilate_alloc, dim3(tiles), dim3(256), 0, cube, uint32_t(n_words), al, ctx->rank, ctx->world,
                                                 ctx->slab, ctx->cand_keys.as<uint64_t>(),
                                                 ctx->cand_slots.as<int32_t>(), ctx->status_w(), st,
                                                 other.as<uint32_t>(), uint32_t(other_words));
  ctx->bitmap_clean[bp ^ 1] = other_words;
  ctx->prof_end();
  ctx->count_launch();
  check_launch(ctx, "k_dilate_alloc");
  if (cand_cap_out) *cand_cap_out = cand_cap;
}

}  // namespace vxm
