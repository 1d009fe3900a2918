// Batch distance / gradient queries.
//
// Reference: query_point / query_batch (proj/src/query/query.cpp:64-161),
// esdf_distance (proj/include/voxmap/esdf/integrator.hpp:59-63).  One thread
// per point, the production evaluation order of query.cpp (bit-identical
// results), block look-ups through the ESDF layer's device hash.
#include <cmath>

#include "runtime.cuh"

namespace vxm {

struct QueryArgs {
  const double* xyz;
  uint64_t n;
  HashView hash;
  const uint32_t* pool;
  double vs;
  int want_gradient, interpolate;
  vxm_query_result* out;
};

__device__ inline int64_t fdiv8(int64_t a) { return a >= 0 ? a / 8 : -((-a + 7) / 8); }

// Returns pointer to the voxel's 3 words or nullptr.
__device__ inline const uint32_t* voxel_at(const QueryArgs& a, int64_t gx, int64_t gy, int64_t gz) {
  const int64_t bx = fdiv8(gx), by = fdiv8(gy), bz = fdiv8(gz);
  if (!coord_ok(bx) || !coord_ok(by) || !coord_ok(bz)) return nullptr;
  const int32_t s = hash_find(a.hash, pack_key(int32_t(bx), int32_t(by), int32_t(bz)));
  if (s < 0) return nullptr;
  const int lin = int(gx - bx * 8) + 8 * int(gy - by * 8) + 64 * int(gz - bz * 8);
  return a.pool + size_t(s) * 1536 + lin * 3;
}
__device__ inline uint32_t vflags(const uint32_t* v) { return (__ldg(v + 2) >> 16) & 0xffu; }
__device__ inline double esdf_distance(const uint32_t* v, double vs) {
  const double d = __dmul_rn(__dsqrt_rn(double(int32_t(__ldg(v)))), vs);
  return (vflags(v) & VXM_ESDF_INSIDE) ? -d : d;
}
__device__ inline void parent_gradient(const uint32_t* v, double g[3]) {  // query.cpp:58-64
  const uint32_t w1 = __ldg(v + 1), w2 = __ldg(v + 2);
  const double off[3] = {double(int16_t(w1 & 0xffffu)), double(int16_t(w1 >> 16)),
                         double(int16_t(w2 & 0xffffu))};
  g[0] = g[1] = g[2] = 0.0;
  if (off[0] == 0.0 && off[1] == 0.0 && off[2] == 0.0) return;
  const double z = __dadd_rn(__dmul_rn(off[0], off[0]),
                             __dadd_rn(__dmul_rn(off[1], off[1]), __dmul_rn(off[2], off[2])));
  const double s = __dsqrt_rn(z);
  const bool inside = vflags(v) & VXM_ESDF_INSIDE;
  for (int k = 0; k < 3; ++k) {
    const double nrm = __ddiv_rn(off[k], s);
    g[k] = inside ? nrm : -nrm;
  }
}

__global__ void k_query(QueryArgs a) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < a.n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    vxm_query_result r;
    r.known = 0;
    r.pad_ = 0;
    r.distance = 0.0;
    r.gradient[0] = r.gradient[1] = r.gradient[2] = 0.0;
    const double p[3] = {a.xyz[3 * i], a.xyz[3 * i + 1], a.xyz[3 * i + 2]};
    if (isfinite(p[0]) && isfinite(p[1]) && isfinite(p[2])) {
      const double vs = a.vs;
      const uint32_t* at = voxel_at(a, int64_t(floor(__ddiv_rn(p[0], vs))),
                                    int64_t(floor(__ddiv_rn(p[1], vs))),
                                    int64_t(floor(__ddiv_rn(p[2], vs))));
      if (at && (vflags(at) & VXM_ESDF_OBSERVED)) {
        r.known = 1;
        double w[3];
        int64_t base[3];
        for (int k = 0; k < 3; ++k) {
          const double q = __dsub_rn(__ddiv_rn(p[k], vs), 0.5);
          const double fl = floor(q);
          base[k] = int64_t(fl);
          w[k] = __dsub_rn(q, fl);
          if (w[k] < 1e-6) w[k] = 0.0;
          else if (w[k] > 1.0 - 1e-6) w[k] = 1.0;
        }
        bool corners = a.interpolate != 0;
        double d[2][2][2];
        if (corners) {
          for (int dz = 0; dz < 2 && corners; ++dz)
            for (int dy = 0; dy < 2 && corners; ++dy)
              for (int dx = 0; dx < 2; ++dx) {
                const uint32_t* v = voxel_at(a, base[0] + dx, base[1] + dy, base[2] + dz);
                if (!v || !(vflags(v) & VXM_ESDF_OBSERVED)) {
                  corners = false;
                  break;
                }
                d[dx][dy][dz] = esdf_distance(v, vs);
              }
        }
        if (!corners) {
          r.distance = esdf_distance(at, vs);
          if (a.want_gradient) parent_gradient(at, r.gradient);
        } else {
          const double ix = __dsub_rn(1.0, w[0]), iy = __dsub_rn(1.0, w[1]), iz = __dsub_rn(1.0, w[2]);
#define M_ __dmul_rn
#define A_ __dadd_rn
#define S_ __dsub_rn
          r.distance = A_(M_(iz, A_(M_(iy, A_(M_(ix, d[0][0][0]), M_(w[0], d[1][0][0]))),
                                    M_(w[1], A_(M_(ix, d[0][1][0]), M_(w[0], d[1][1][0]))))),
                          M_(w[2], A_(M_(iy, A_(M_(ix, d[0][0][1]), M_(w[0], d[1][0][1]))),
                                      M_(w[1], A_(M_(ix, d[0][1][1]), M_(w[0], d[1][1][1]))))));
          if (a.want_gradient) {
            double g[3];
            g[0] = A_(M_(iz, A_(M_(iy, S_(d[1][0][0], d[0][0][0])), M_(w[1], S_(d[1][1][0], d[0][1][0])))),
                      M_(w[2], A_(M_(iy, S_(d[1][0][1], d[0][0][1])), M_(w[1], S_(d[1][1][1], d[0][1][1])))));
            g[1] = A_(M_(iz, A_(M_(ix, S_(d[0][1][0], d[0][0][0])), M_(w[0], S_(d[1][1][0], d[1][0][0])))),
                      M_(w[2], A_(M_(ix, S_(d[0][1][1], d[0][0][1])), M_(w[0], S_(d[1][1][1], d[1][0][1])))));
            g[2] = A_(M_(iy, A_(M_(ix, S_(d[0][0][1], d[0][0][0])), M_(w[0], S_(d[1][0][1], d[1][0][0])))),
                      M_(w[1], A_(M_(ix, S_(d[0][1][1], d[0][1][0])), M_(w[0], S_(d[1][1][1], d[1][1][0])))));
            const double nrm = __dsqrt_rn(A_(M_(g[0], g[0]), A_(M_(g[1], g[1]), M_(g[2], g[2]))));
            if (nrm > 1e-9) {
              for (int k = 0; k < 3; ++k) r.gradient[k] = __ddiv_rn(g[k], nrm);
            } else {
              parent_gradient(at, r.gradient);
            }
          }
#undef M_
#undef A_
#undef S_
        }
      }
    }
    a.out[i] = r;
  }
}

void run_query(Layer* E, const double* xyz_host, uint64_t n, int want_gradient, int interpolate,
               vxm_query_result* out_host) {
  Context* ctx = E->ctx;
  if (n == 0) return;
  E->refresh();
  DevBuf dx, dout;
  dx.ensure(sizeof(double) * 3 * n);
  dout.ensure(sizeof(vxm_query_result) * n);
  VXM_CUDA(cudaMemcpyAsync(dx.p, xyz_host, sizeof(double) * 3 * n, cudaMemcpyHostToDevice,
                           ctx->stream));
  QueryArgs a{};
  a.xyz = dx.as<double>();
  a.n = n;
  a.hash = E->hash;
  a.pool = static_cast<const uint32_t*>(E->pool[E->cur_host]);
  a.vs = E->vs;
  a.want_gradient = want_gradient;
  a.interpolate = interpolate;
  a.out = dout.as<vxm_query_result>();
  if (E->num_blocks == 0 || !a.hash.keys) {
    VXM_CUDA(cudaMemsetAsync(dout.p, 0, sizeof(vxm_query_result) * n, ctx->stream));
  } else {
    const uint32_t grid = uint32_t(std::min<uint64_t>(ceil_div(n, 256), uint64_t(ctx->sm_count) * 16));
    k_query<<<grid, 256, 0, ctx->stream>>>(a);
    ctx->count_launch();
    check_launch(ctx, "k_query");
  }
  VXM_CUDA(cudaMemcpyAsync(out_host, dout.p, sizeof(vxm_query_result) * n, cudaMemcpyDeviceToHost,
                           ctx->stream));
  VXM_CUDA(cudaStreamSynchronize(ctx->stream));
}

}  // namespace vxm
