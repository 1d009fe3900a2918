// Marching-cubes meshing of the TSDF.
//
// Reference: mesh_block (proj/src/mesh/marching_cubes.cpp:95-209) with
// fill_corners (:37-78) and edge_lattice_key (:80-91); update_mesh (:211-242);
// the Lorensen-Cline tables (marching_cubes_tables.cpp:20-305, packed in
// mc_table.cuh); MeshLayer (include/voxmap/mesh/mesh_layer.hpp:27-66).
//
// B200 design: one 512-thread CTA per target block, one thread per cube.  The
// 9^3 corner lattice (block + its +x/+y/+z face layers) is staged in shared
// memory.  The reference's serial, welded vertex numbering is reproduced
// without hashing: a lattice edge's vertex is created by the first active cube
// (scan order z, y, x) that references it, so each cube counts the edges it
// references first (in the reference's call order i0, i2, i1 per triangle)
// that no earlier active cube shares; a block-wide exclusive scan of those
// counts (and of the triangle counts) gives every vertex and triangle its
// serial index.  Vertex normals sum the incident face normals in serial
// triangle order (the <= 4 cubes around the edge, ascending), so every FP32
// sum rounds exactly as the reference's.  A count pass sizes the output; the
// emit pass writes it; the host keeps the per-block meshes (MeshLayer).
#include <algorithm>
#include <cmath>
#include <cstddef>

#include "esdf_host.cuh"
#include "mc_table.cuh"
#include "mesh.cuh"

namespace vxm {

namespace {

constexpr int kG = 9;                // corner lattice per block side
constexpr int kLat = kG * kG * kG;   // 729
constexpr int kMaxV = 3 * 8 * 81;    // lattice edges touched by the 512 cubes
constexpr int kMaxT = 512 * 5;
constexpr int kMeshThreads = 512;

// Lorensen-Cline corner c: (x, y, z) = ((c + 1) >> 1 & 1, c >> 1 & 1, c >> 2)
// (marching_cubes_tables.cpp:22-25); edge e joins corners (e, e+1 mod 4) on the
// z = 0 / z = 1 faces and (e - 8, e - 4) for the verticals (:27-30).
__device__ inline int corner_x(int c) { return ((c + 1) >> 1) & 1; }
__device__ inline int corner_y(int c) { return (c >> 1) & 1; }
__device__ inline int corner_z(int c) { return c >> 2; }
__device__ inline int edge_a(int e) { return e < 8 ? e : e - 8; }
__device__ inline int edge_b(int e) { return e < 4 ? ((e + 1) & 3) : e < 8 ? 4 + ((e + 1) & 3) : e - 4; }
__device__ inline int lat(int x, int y, int z) { return x + kG * (y + kG * z); }

struct EdgeRef {
  int lx, ly, lz, axis;
};
// edge_lattice_key (marching_cubes.cpp:80-91): lower corner + axis.
__device__ inline EdgeRef edge_ref(int cx, int cy, int cz, int e) {
  const int a = edge_a(e), b = edge_b(e);
  EdgeRef r;
  r.lx = cx + min(corner_x(a), corner_x(b));
  r.ly = cy + min(corner_y(a), corner_y(b));
  r.lz = cz + min(corner_z(a), corner_z(b));
  r.axis = corner_x(a) != corner_x(b) ? 0 : corner_y(a) != corner_y(b) ? 1 : 2;
  return r;
}
__device__ inline int edge_slot(const EdgeRef& r) { return r.axis * kLat + lat(r.lx, r.ly, r.lz); }

// The (up to 4) cubes sharing a lattice edge, in ascending scan order:
// k = 2 * hi + lo over the two other axes (hi = the more significant).
__device__ inline int sharing_cube(const EdgeRef& r, int k) {
  int c[3] = {r.lx, r.ly, r.lz};
  const int lo_axis = r.axis == 0 ? 1 : 0, hi_axis = r.axis == 2 ? 1 : 2;
  c[hi_axis] -= 1 - (k >> 1);
  c[lo_axis] -= 1 - (k & 1);
  if (c[0] < 0 || c[1] < 0 || c[2] < 0 || c[0] > 7 || c[1] > 7 || c[2] > 7) return -1;
  return c[0] + 8 * c[1] + 64 * c[2];
}

struct MeshSmem {
  float dist[kLat];
  uint8_t known[kLat + 3];
  uint32_t active[16];
  int32_t nb[4];
  uint32_t warp_sum[16];
  // emit pass only
  uint16_t vmap[3 * kLat];
  uint16_t tbase[512];
  uint8_t ntri[512];
  float vpos[3 * kMaxV];
  float vfb[3 * kMaxV];
  float tn[3 * kMaxT];
  uint16_t tv[3 * kMaxT];
};
constexpr size_t kCountSmem = offsetof(MeshSmem, vmap);

struct MeshArgs {
  const uint64_t* keys;
  uint32_t n;
  HashView tsdf_hash;
  const float2* tsdf_pool;
  float min_weight;
  double vs;
  uint32_t* counts;  // count pass: [n][2] (vertices, triangles)
  const uint32_t* voff;
  const uint32_t* toff;
  float* verts;
  float* normals;
  uint8_t* colors;  // null: no color layer
  uint32_t* tris;
  HashView color_hash;
  const uint2* color_pool;
  double color_vs;
};

__device__ inline int64_t floor_div8_i64(int64_t a) { return a >= 0 ? a / 8 : -((-a + 7) / 8); }

template <bool EMIT>
__global__ void __launch_bounds__(kMeshThreads) k_mesh(MeshArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  MeshSmem& S = *reinterpret_cast<MeshSmem*>(smem_raw);
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int cx = t & 7, cy = (t >> 3) & 7, cz = t >> 6;
  for (uint32_t b = blockIdx.x; b < a.n; b += gridDim.x) {
    const uint64_t key = a.keys[b];
    if (t < 4) S.nb[t] = hash_find(a.tsdf_hash, t == 0 ? key : key_shift(key, t - 1, 1));
    __syncthreads();
    // fill_corners (marching_cubes.cpp:37-78): the block plus its +face layers;
    // lattice points needing an edge/corner neighbour stay unknown
    for (int i = t; i < kLat; i += kMeshThreads) {
      const int x = i % kG, y = (i / kG) % kG, z = i / (kG * kG);
      const int n8 = (x == 8) + (y == 8) + (z == 8);
      int32_t s = -1;
      int lx = x, ly = y, lz = z;
      if (n8 == 0) {
        s = S.nb[0];
      } else if (n8 == 1) {
        const int axis = x == 8 ? 0 : y == 8 ? 1 : 2;
        s = S.nb[1 + axis];
        if (axis == 0) lx = 0; else if (axis == 1) ly = 0; else lz = 0;
      }
      bool kn = false;
      float d = 0.0f;
      if (s >= 0) {
        const float2 v = __ldg(a.tsdf_pool + size_t(s) * kVPB + lx + 8 * (ly + 8 * lz));
        if (v.y >= a.min_weight) {
          kn = true;
          d = v.x;
        }
      }
      S.known[i] = kn;
      S.dist[i] = d;
    }
    __syncthreads();
    // this thread's cube: active iff all 8 corners are known (:127-140)
    int config = 0;
    bool act = true;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const int li = lat(cx + corner_x(c), cy + corner_y(c), cz + corner_z(c));
      if (!S.known[li]) act = false;
      else if (S.dist[li] < 0.0f) config |= 1 << c;
    }
    const uint32_t am = __ballot_sync(0xffffffffu, act);
    if (lane == 0) S.active[warp] = am;
    const bool mc = act && config != 0 && config != 255;
    const uint64_t row = mc ? kMcTri[config] : 0ull;
    const int nt = mc ? int(row >> 60) : 0;
    __syncthreads();
    // edges this cube references first (call order i0, i2, i1 per triangle,
    // :177-183) that no earlier active cube shares: the vertices it creates
    uint32_t seen = 0;
    uint64_t newlist = 0;
    int n_new = 0;
    for (int k = 0; k < nt; ++k) {
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        const int pos = 3 * k + (q == 0 ? 0 : q == 1 ? 2 : 1);
        const int e = int(row >> (4 * pos)) & 15;
        if (seen & (1u << e)) continue;
        seen |= 1u << e;
        const EdgeRef r = edge_ref(cx, cy, cz, e);
        bool owned = true;
        for (int s = 0; s < 4; ++s) {
          const int c = sharing_cube(r, s);
          if (c >= 0 && c < t && ((S.active[c >> 5] >> (c & 31)) & 1u)) owned = false;
        }
        if (owned) {
          newlist |= uint64_t(e) << (4 * n_new);
          ++n_new;
        }
      }
    }
    // block-wide exclusive scan of (n_new << 16 | nt)
    const uint32_t packed = (uint32_t(n_new) << 16) | uint32_t(nt);
    uint32_t incl = packed;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if (lane == 31) S.warp_sum[warp] = incl;
    __syncthreads();
    uint32_t wpre = 0, total = 0;
    for (int w = 0; w < 16; ++w) {
      const uint32_t s = S.warp_sum[w];
      if (w < warp) wpre += s;
      total += s;
    }
    const uint32_t pre = wpre + incl - packed;
    if (!EMIT) {
      if (t == 0) {
        a.counts[2 * b] = total >> 16;
        a.counts[2 * b + 1] = total & 0xffffu;
      }
      __syncthreads();
      continue;
    }
    const uint32_t vbase = pre >> 16, tb = pre & 0xffffu;
    S.tbase[t] = uint16_t(tb);
    S.ntri[t] = uint8_t(nt);
    // vertex_on_edge for the created vertices (:143-168)
    const double edge = 8.0 * a.vs;
    const double ox = __dmul_rn(double(key_x(key)), edge), oy = __dmul_rn(double(key_y(key)), edge),
                 oz = __dmul_rn(double(key_z(key)), edge);  // block_origin (indexing.hpp:129-132)
    for (int j = 0; j < n_new; ++j) {
      const int e = int(newlist >> (4 * j)) & 15;
      const int idx = int(vbase) + j;
      S.vmap[edge_slot(edge_ref(cx, cy, cz, e))] = uint16_t(idx);
      const int ca = edge_a(e), cb = edge_b(e);
      const int ax = cx + corner_x(ca), ay = cy + corner_y(ca), az = cz + corner_z(ca);
      const int bx = cx + corner_x(cb), by = cy + corner_y(cb), bz = cz + corner_z(cb);
      const double da = double(S.dist[lat(ax, ay, az)]), db = double(S.dist[lat(bx, by, bz)]);
      const double tt = __ddiv_rn(da, __dsub_rn(da, db));
      // corner_center: origin + (x + 0.5) * vs per axis (:114-118)
      const double pa[3] = {__dadd_rn(ox, __dmul_rn(double(ax) + 0.5, a.vs)),
                            __dadd_rn(oy, __dmul_rn(double(ay) + 0.5, a.vs)),
                            __dadd_rn(oz, __dmul_rn(double(az) + 0.5, a.vs))};
      const double pb[3] = {__dadd_rn(ox, __dmul_rn(double(bx) + 0.5, a.vs)),
                            __dadd_rn(oy, __dmul_rn(double(by) + 0.5, a.vs)),
                            __dadd_rn(oz, __dmul_rn(double(bz) + 0.5, a.vs))};
      float dir[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const double dk = __dsub_rn(pb[k], pa[k]);
        S.vpos[3 * idx + k] = __double2float_rn(__dadd_rn(pa[k], __dmul_rn(tt, dk)));
        dir[k] = __double2float_rn(dk);
      }
      // (pb - pa).cast<float>().normalized(); negated when da >= 0 (:164-165)
      const float z = __fadd_rn(__fmul_rn(dir[0], dir[0]),
                                __fadd_rn(__fmul_rn(dir[1], dir[1]), __fmul_rn(dir[2], dir[2])));
      const float sz = __fsqrt_rn(z);
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const float u = z > 0.0f ? __fdiv_rn(dir[k], sz) : dir[k];
        S.vfb[3 * idx + k] = da < 0.0 ? u : -u;
      }
    }
    __syncthreads();
    // triangles (i0, i2, i1 winding, :172-186) and their face normals
    for (int k = 0; k < nt; ++k) {
      uint16_t iv[3];
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        const int pos = 3 * k + (q == 0 ? 0 : q == 1 ? 2 : 1);
        iv[q] = S.vmap[edge_slot(edge_ref(cx, cy, cz, int(row >> (4 * pos)) & 15))];
      }
      const int ti = int(tb) + k;
      S.tv[3 * ti] = iv[0];
      S.tv[3 * ti + 1] = iv[1];
      S.tv[3 * ti + 2] = iv[2];
      const float* v0 = &S.vpos[3 * iv[0]];
      const float* v1 = &S.vpos[3 * iv[1]];
      const float* v2 = &S.vpos[3 * iv[2]];
      const float e1[3] = {__fsub_rn(v1[0], v0[0]), __fsub_rn(v1[1], v0[1]), __fsub_rn(v1[2], v0[2])};
      const float e2[3] = {__fsub_rn(v2[0], v0[0]), __fsub_rn(v2[1], v0[1]), __fsub_rn(v2[2], v0[2])};
      S.tn[3 * ti] = __fsub_rn(__fmul_rn(e1[1], e2[2]), __fmul_rn(e1[2], e2[1]));
      S.tn[3 * ti + 1] = __fsub_rn(__fmul_rn(e1[2], e2[0]), __fmul_rn(e1[0], e2[2]));
      S.tn[3 * ti + 2] = __fsub_rn(__fmul_rn(e1[0], e2[1]), __fmul_rn(e1[1], e2[0]));
      uint32_t* out = a.tris + 3 * (size_t(a.toff[b]) + ti);
      out[0] = iv[0];
      out[1] = iv[1];
      out[2] = iv[2];
    }
    __syncthreads();
    // vertex normals: incident face normals summed in serial triangle order,
    // normalized, or the edge fallback (:189-194); colors (:196-207)
    for (int j = 0; j < n_new; ++j) {
      const int e = int(newlist >> (4 * j)) & 15;
      const int idx = int(vbase) + j;
      const EdgeRef r = edge_ref(cx, cy, cz, e);
      float acc[3] = {0.0f, 0.0f, 0.0f};
      for (int s = 0; s < 4; ++s) {
        const int c = sharing_cube(r, s);
        if (c < 0) continue;
        const int base = S.tbase[c], cnt = S.ntri[c];
        for (int k = 0; k < cnt; ++k) {
          const int ti = base + k;
          if (S.tv[3 * ti] == idx || S.tv[3 * ti + 1] == idx || S.tv[3 * ti + 2] == idx) {
            acc[0] = __fadd_rn(acc[0], S.tn[3 * ti]);
            acc[1] = __fadd_rn(acc[1], S.tn[3 * ti + 1]);
            acc[2] = __fadd_rn(acc[2], S.tn[3 * ti + 2]);
          }
        }
      }
      const float nrm = __fsqrt_rn(__fadd_rn(__fmul_rn(acc[0], acc[0]),
                                             __fadd_rn(__fmul_rn(acc[1], acc[1]), __fmul_rn(acc[2], acc[2]))));
      const size_t gv = size_t(a.voff[b]) + idx;
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        a.verts[3 * gv + k] = S.vpos[3 * idx + k];
        a.normals[3 * gv + k] = nrm > 1e-12f ? __fdiv_rn(acc[k], nrm) : S.vfb[3 * idx + k];
      }
      if (a.colors) {
        // position_to_global_voxel (indexing.hpp:96-102) in the color layer
        int64_t g[3];
        bool ok = true;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
          g[k] = int64_t(floor(__ddiv_rn(double(S.vpos[3 * idx + k]), a.color_vs)));
        }
        const int64_t bx = floor_div8_i64(g[0]), by = floor_div8_i64(g[1]), bz = floor_div8_i64(g[2]);
        ok = coord_ok(bx) && coord_ok(by) && coord_ok(bz);
        uint8_t rgb[3] = {128, 128, 128};
        if (ok) {
          const int32_t cs = hash_find(a.color_hash, pack_key(int32_t(bx), int32_t(by), int32_t(bz)));
          if (cs >= 0) {
            const int lin = int(g[0] - 8 * bx) + 8 * int(g[1] - 8 * by) + 64 * int(g[2] - 8 * bz);
            const uint2 cv = a.color_pool[size_t(cs) * kVPB + lin];
            if (__uint_as_float(cv.y) > 0.0f) {
              rgb[0] = uint8_t(cv.x);
              rgb[1] = uint8_t(cv.x >> 8);
              rgb[2] = uint8_t(cv.x >> 16);
            }
          }
        }
        a.colors[3 * gv] = rgb[0];
        a.colors[3 * gv + 1] = rgb[1];
        a.colors[3 * gv + 2] = rgb[2];
      }
    }
    __syncthreads();
  }
}

__global__ void k_mesh_lookup(const uint64_t* keys, uint32_t n, HashView h, int32_t* out) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = hash_find(h, keys[i]);
}

std::vector<int32_t> lookup(Context* ctx, const Layer* L, const std::vector<uint64_t>& keys) {
  const uint32_t n = uint32_t(keys.size());
  std::vector<int32_t> out(n);
  if (!n) return out;
  DevBuf dk, ds;
  dk.ensure(sizeof(uint64_t) * n);
  ds.ensure(sizeof(int32_t) * n);
  VXM_CUDA(cudaMemcpyAsync(dk.p, keys.data(), sizeof(uint64_t) * n, cudaMemcpyHostToDevice, ctx->stream));
  k_mesh_lookup<<<grid_for(ctx, n), 256, 0, ctx->stream>>>(dk.as<uint64_t>(), n, L->hash, ds.as<int32_t>());
  ctx->count_launch();
  check_launch(ctx, "k_mesh_lookup");
  VXM_CUDA(cudaMemcpyAsync(out.data(), ds.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, ctx->stream));
  VXM_CUDA(cudaStreamSynchronize(ctx->stream));
  return out;
}

void mesh_sorted_keys(MeshLayerH* M, Layer* T, const std::vector<uint64_t>& targets, float min_weight,
                      Layer* color) {
  Context* ctx = T->ctx;
  const uint32_t n = uint32_t(targets.size());
  if (!n) return;
  ctx->once_attr((const void*)k_mesh<true>, [] {  // per device (function attributes are per context)
    VXM_CUDA(cudaFuncSetAttribute(k_mesh<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(sizeof(MeshSmem))));
    VXM_CUDA(cudaFuncSetAttribute(k_mesh<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(kCountSmem)));
  });
  DevBuf dkeys, dcounts, doff;
  dkeys.ensure(sizeof(uint64_t) * n);
  dcounts.ensure(sizeof(uint32_t) * 2 * n);
  doff.ensure(sizeof(uint32_t) * 2 * n);
  VXM_CUDA(cudaMemcpyAsync(dkeys.p, targets.data(), sizeof(uint64_t) * n, cudaMemcpyHostToDevice,
                           ctx->stream));
  MeshArgs a{};
  a.keys = dkeys.as<uint64_t>();
  a.n = n;
  a.tsdf_hash = T->hash;
  a.tsdf_pool = static_cast<const float2*>(T->pool[0]);
  a.min_weight = min_weight;
  a.vs = T->vs;
  a.counts = dcounts.as<uint32_t>();
  const uint32_t grid = std::min<uint32_t>(n, uint32_t(ctx->sm_count) * 4);
  ctx->prof_begin("k_mesh_count");
  k_mesh<false><<<grid, kMeshThreads, kCountSmem, ctx->stream>>>(a);
  ctx->prof_end();
  ctx->count_launch();
  check_launch(ctx, "k_mesh_count");
  std::vector<uint32_t> counts(2 * n), off(2 * n);
  VXM_CUDA(cudaMemcpyAsync(counts.data(), dcounts.p, sizeof(uint32_t) * 2 * n, cudaMemcpyDeviceToHost,
                           ctx->stream));
  VXM_CUDA(cudaStreamSynchronize(ctx->stream));
  uint64_t nv = 0, ntr = 0;
  for (uint32_t i = 0; i < n; ++i) {
    off[i] = uint32_t(nv);
    off[n + i] = uint32_t(ntr);
    nv += counts[2 * i];
    ntr += counts[2 * i + 1];
  }
  DevBuf dv, dn, dc, dt;
  dv.ensure(sizeof(float) * 3 * std::max<uint64_t>(nv, 1));
  dn.ensure(sizeof(float) * 3 * std::max<uint64_t>(nv, 1));
  dt.ensure(sizeof(uint32_t) * 3 * std::max<uint64_t>(ntr, 1));
  if (color) dc.ensure(3 * std::max<uint64_t>(nv, 1));
  VXM_CUDA(cudaMemcpyAsync(doff.p, off.data(), sizeof(uint32_t) * 2 * n, cudaMemcpyHostToDevice, ctx->stream));
  a.voff = doff.as<uint32_t>();
  a.toff = doff.as<uint32_t>() + n;
  a.verts = dv.as<float>();
  a.normals = dn.as<float>();
  a.tris = dt.as<uint32_t>();
  a.colors = color ? dc.as<uint8_t>() : nullptr;
  if (color) {
    a.color_hash = color->hash;
    a.color_pool = static_cast<const uint2*>(color->pool[0]);
    a.color_vs = color->vs;
  }
  ctx->prof_begin("k_mesh");
  k_mesh<true><<<grid, kMeshThreads, sizeof(MeshSmem), ctx->stream>>>(a);
  ctx->prof_end();
  ctx->count_launch();
  check_launch(ctx, "k_mesh");
  std::vector<float> hv(3 * nv), hn(3 * nv);
  std::vector<uint32_t> ht(3 * ntr);
  std::vector<uint8_t> hc(color ? 3 * nv : 0);
  if (nv) {
    VXM_CUDA(cudaMemcpyAsync(hv.data(), dv.p, sizeof(float) * 3 * nv, cudaMemcpyDeviceToHost, ctx->stream));
    VXM_CUDA(cudaMemcpyAsync(hn.data(), dn.p, sizeof(float) * 3 * nv, cudaMemcpyDeviceToHost, ctx->stream));
    if (color) VXM_CUDA(cudaMemcpyAsync(hc.data(), dc.p, 3 * nv, cudaMemcpyDeviceToHost, ctx->stream));
  }
  if (ntr)
    VXM_CUDA(cudaMemcpyAsync(ht.data(), dt.p, sizeof(uint32_t) * 3 * ntr, cudaMemcpyDeviceToHost, ctx->stream));
  VXM_CUDA(cudaStreamSynchronize(ctx->stream));
  // update_mesh stores every target's MeshBlock (:236-240)
  for (uint32_t i = 0; i < n; ++i) {
    MeshBlockH& mb = M->blocks[targets[i]];
    const size_t v0 = off[i], c = counts[2 * i], t0 = off[n + i], tc = counts[2 * i + 1];
    mb.vertices.assign(hv.begin() + 3 * v0, hv.begin() + 3 * (v0 + c));
    mb.normals.assign(hn.begin() + 3 * v0, hn.begin() + 3 * (v0 + c));
    if (color) mb.colors.assign(hc.begin() + 3 * v0, hc.begin() + 3 * (v0 + c));
    else mb.colors.clear();
    mb.triangles.assign(ht.begin() + 3 * t0, ht.begin() + 3 * (t0 + tc));
  }
}

}  // namespace

void run_mesh_blocks(MeshLayerH* M, Layer* T, BlockList* targets, float min_weight, Layer* color) {
  const auto& h = targets->fetch();
  std::vector<uint64_t> keys(h.size());
  for (size_t i = 0; i < h.size(); ++i) {
    if (!(coord_ok(h[i].x) && coord_ok(h[i].y) && coord_ok(h[i].z)))
      throw Error(VXM_ERR_INVALID_ARGUMENT, "mesh_block: block is not allocated");
    keys[i] = pack_key(h[i].x, h[i].y, h[i].z);
  }
  const auto slots = lookup(T->ctx, T, keys);
  for (int32_t s : slots)  // marching_cubes.cpp:97-99
    if (s < 0) throw Error(VXM_ERR_INVALID_ARGUMENT, "mesh_block: block is not allocated");
  mesh_sorted_keys(M, T, keys, min_weight, color);
}

std::vector<vxm_grid_index> run_update_mesh(MeshLayerH* M, Layer* T, BlockList* updated,
                                            float min_weight, Layer* color) {
  const auto& h = updated->fetch();
  // targets: g and its -x, -y, -z neighbours that are allocated (:215-230)
  std::vector<uint64_t> cand;
  cand.reserve(4 * h.size());
  for (const auto& g : h) {
    const int32_t c[4][3] = {{g.x, g.y, g.z}, {g.x - 1, g.y, g.z}, {g.x, g.y - 1, g.z}, {g.x, g.y, g.z - 1}};
    for (const auto& k : c)
      if (coord_ok(k[0]) && coord_ok(k[1]) && coord_ok(k[2])) cand.push_back(pack_key(k[0], k[1], k[2]));
  }
  std::sort(cand.begin(), cand.end());
  cand.erase(std::unique(cand.begin(), cand.end()), cand.end());
  const auto slots = lookup(T->ctx, T, cand);
  std::vector<uint64_t> targets;
  for (size_t i = 0; i < cand.size(); ++i)
    if (slots[i] >= 0) targets.push_back(cand[i]);
  mesh_sorted_keys(M, T, targets, min_weight, color);
  std::vector<vxm_grid_index> out(targets.size());
  for (size_t i = 0; i < targets.size(); ++i)
    out[i] = {key_x(targets[i]), key_y(targets[i]), key_z(targets[i])};
  return out;
}

}  // namespace vxm
