// Color fusion into the TSDF surface band.
//
// Reference: integrate_color (proj/src/integrate/integrator.cpp:191-273),
// color_update (include/voxmap/integrate/updates.hpp:74-92),
// sample_color_nearest (include/voxmap/sensor/image.hpp:108-119),
// CameraIntrinsics::project/contains (sensor/camera.hpp:35-46).
//
// B200 design: the candidates come from the same DDA/bitmap view kernels as
// depth integration (run_view, no allocation); one warp per candidate tests the
// TSDF block for a surface-band voxel (weight > 0 and |d| <= trunc) and an
// order-preserving compaction gives the work list (sorted, as the reference's
// candidate order); the color blocks are allocated for the work list in one
// pass; one warp per work block then fuses its 512 voxels (16 per lane), and
// the changed list is a compaction of the work list.
#include <cmath>

#include "esdf_host.cuh"
#include "runtime.cuh"

namespace vxm {

struct ColorArgs {
  const uint64_t* work_keys;
  const uint32_t* n_work;
  const int32_t* color_slots;
  HashView tsdf_hash;
  const float2* tsdf_pool;
  uint2* color_pool;     // ColorVoxel {r, g, b, reserved | float weight}
  const uint8_t* rgb;    // row-major W x H x 3
  int W, H;
  vxm_pose T_SL;
  double fu, fv, cu, cv;
  double vs;
  float eps, max_weight;
  uint8_t* changed;
};

// Per candidate: is there a TSDF block with a surface-band voxel
// (integrator.cpp:212-227)?  One warp per candidate.
__global__ void __launch_bounds__(256) k_color_band(const uint64_t* cand, const DevStatus* st,
                                                    HashView tsdf_hash, const float2* tsdf_pool,
                                                    float eps, uint8_t* flags) {
  const uint32_t n = st->n_candidates;
  const int lane = threadIdx.x & 31;
  const uint32_t nwarps = gridDim.x * (blockDim.x >> 5);
  for (uint32_t ci = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; ci < n; ci += nwarps) {
    const int32_t ts = hash_find(tsdf_hash, cand[ci]);
    bool band = false;
    if (ts >= 0) {
      const float2* blk = tsdf_pool + size_t(ts) * kVPB;
#pragma unroll 4
      for (int j = 0; j < 16; ++j) {
        const float2 v = __ldg(blk + lane + 32 * j);
        band |= v.y > 0.0f && fabsf(v.x) <= eps;
      }
    }
    band = __any_sync(0xffffffffu, band);
    if (lane == 0) flags[ci] = band ? 1 : 0;
  }
}

__device__ inline uint8_t blend_channel(float w, uint8_t cur, uint8_t obs, float w_sum) {
  // (double(w) * cur + double(1.0f) * obs) / w_sum, round half away from zero,
  // clamp to [0, 255] — updates.hpp:81-84
  const double v = __ddiv_rn(__dadd_rn(__dmul_rn(double(w), double(cur)), __dmul_rn(1.0, double(obs))),
                             double(w_sum));
  double r = round(v);
  r = r < 0.0 ? 0.0 : (255.0 < r ? 255.0 : r);
  return uint8_t(r);
}

// One warp per work block, voxel lin = lane + 32 j (integrator.cpp:233-262).
__global__ void __launch_bounds__(256) k_color(ColorArgs a) {
  const uint32_t n = *a.n_work;
  const int lane = threadIdx.x & 31;
  const uint32_t nwarps = gridDim.x * (blockDim.x >> 5);
  const double* R = a.T_SL.R;
  for (uint32_t wi = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; wi < n; wi += nwarps) {
    const uint64_t key = a.work_keys[wi];
    const int32_t cs = a.color_slots[wi];
    const int32_t ts = hash_find(a.tsdf_hash, key);
    bool any = false;
    if (cs >= 0 && ts >= 0) {
      const float2* tb = a.tsdf_pool + size_t(ts) * kVPB;
      uint2* cb = a.color_pool + size_t(cs) * kVPB;
      const int32_t gx = key_x(key), gy = key_y(key), gz = key_z(key);
#pragma unroll 1
      for (int j = 0; j < 16; ++j) {
        const int lin = lane + 32 * j;
        const float2 tv = __ldg(tb + lin);
        if (!(tv.y > 0.0f) || fabsf(tv.x) > a.eps) continue;
        // voxel_center (indexing.hpp:113-119) and T_SL * c (pose.hpp:58-60, a0 + (a1 + a2))
        const double c[3] = {
            __dmul_rn(__dadd_rn(__dadd_rn(__dmul_rn(double(gx), 8.0), double(lin & 7)), 0.5), a.vs),
            __dmul_rn(__dadd_rn(__dadd_rn(__dmul_rn(double(gy), 8.0), double((lin >> 3) & 7)), 0.5), a.vs),
            __dmul_rn(__dadd_rn(__dadd_rn(__dmul_rn(double(gz), 8.0), double(lin >> 6)), 0.5), a.vs)};
        double p[3];
#pragma unroll
        for (int i = 0; i < 3; ++i)
          p[i] = __dadd_rn(__dadd_rn(__dmul_rn(R[3 * i], c[0]),
                                     __dadd_rn(__dmul_rn(R[3 * i + 1], c[1]), __dmul_rn(R[3 * i + 2], c[2]))),
                           a.T_SL.t[i]);
        if (!(p[2] > 0.0)) continue;  // project — camera.hpp:35-42
        const double u = __dadd_rn(__ddiv_rn(__dmul_rn(a.fu, p[0]), p[2]), a.cu);
        const double v = __dadd_rn(__ddiv_rn(__dmul_rn(a.fv, p[1]), p[2]), a.cv);
        if (!(u >= 0.0 && u < double(a.W) && v >= 0.0 && v < double(a.H))) continue;  // contains
        const int col = int(floor(u)), row = int(floor(v));  // sample_color_nearest
        if (col >= a.W || row >= a.H) continue;
        const uint8_t* px = a.rgb + (size_t(row) * a.W + col) * 3;
        const uint2 old = cb[lin];
        const float w = __uint_as_float(old.y);
        const float w_sum = __fadd_rn(w, 1.0f);
        const uint8_t r = blend_channel(w, uint8_t(old.x), px[0], w_sum);
        const uint8_t g = blend_channel(w, uint8_t(old.x >> 8), px[1], w_sum);
        const uint8_t b = blend_channel(w, uint8_t(old.x >> 16), px[2], w_sum);
        uint2 nv;
        nv.x = uint32_t(r) | (uint32_t(g) << 8) | (uint32_t(b) << 16) | (old.x & 0xff000000u);
        nv.y = __float_as_uint(a.max_weight < w_sum ? a.max_weight : w_sum);
        if (nv.x != old.x || nv.y != old.y) {
          cb[lin] = nv;
          any = true;
        }
      }
    }
    any = __any_sync(0xffffffffu, any);
    if (lane == 0) a.changed[wi] = any ? 1 : 0;
  }
}

void run_integrate_color(Layer* C, Layer* T, const uint8_t* rgb_host, const ViewArgs& va,
                         const vxm_integrator_config& cfg, BlockList* changed_out) {
  Context* ctx = C->ctx;
  ctx->reset_status();
  uint32_t cand_cap = 0;
  run_view(ctx, va, nullptr, &cand_cap);  // blocks_in_view (integrator.cpp:205-208)
  const float eps = float(cfg.truncation);
  DevBuf flags, rgb;
  flags.ensure(std::max<uint32_t>(cand_cap, 1));
  const size_t rgb_bytes = size_t(va.width) * size_t(va.height) * 3;
  rgb.ensure(std::max<size_t>(rgb_bytes, 4));
  if (rgb_bytes) VXM_CUDA(cudaMemcpyAsync(rgb.p, rgb_host, rgb_bytes, cudaMemcpyHostToDevice, ctx->stream));
  if (cand_cap) {
    ctx->prof_begin("k_color_band");
    k_color_band<<<grid_for(ctx, uint64_t(cand_cap) * 32), 256, 0, ctx->stream>>>(
        ctx->cand_keys.as<uint64_t>(), ctx->status_w(), T->hash, static_cast<const float2*>(T->pool[0]),
        eps, flags.as<uint8_t>());
    ctx->prof_end();
    ctx->count_launch();
    check_launch(ctx, "k_color_band");
  }
  BlockList work;
  work.ctx = ctx;
  work.ensure(std::max<uint32_t>(cand_cap, 1));
  launch_compact_keys(ctx, ctx->cand_keys.as<uint64_t>(), flags.as<uint8_t>(),
                      &ctx->d_status->n_candidates, cand_cap, work.keys.as<uint64_t>(), work.d_count,
                      ctx->status_w(), "k_compact");
  work.count_hint = cand_cap;
  work.host_valid = false;
  work.host_pending = false;
  work.sorted_unique = true;
  // get_or_allocate of the work blocks (integrator.cpp:226)
  DevBuf slots;
  slots.ensure(sizeof(int32_t) * std::max<uint32_t>(cand_cap, 1));
  alloc_key_list(C, &work, slots.as<int32_t>());
  ColorArgs a{};
  a.work_keys = work.keys.as<uint64_t>();
  a.n_work = work.d_count;
  a.color_slots = slots.as<int32_t>();
  a.tsdf_hash = T->hash;
  a.tsdf_pool = static_cast<const float2*>(T->pool[0]);
  a.color_pool = static_cast<uint2*>(C->pool[0]);
  a.rgb = rgb.as<uint8_t>();
  a.W = va.width;
  a.H = va.height;
  vxm_pose_inverse(&va.T_LS, &a.T_SL);  // integrator.cpp:229
  a.fu = va.cam.fu; a.fv = va.cam.fv; a.cu = va.cam.cu; a.cv = va.cam.cv;
  a.vs = C->vs;
  a.eps = eps;
  a.max_weight = cfg.max_weight;
  DevBuf changed;
  changed.ensure(std::max<uint32_t>(cand_cap, 1));
  a.changed = changed.as<uint8_t>();
  if (cand_cap) {
    ctx->prof_begin("k_color");
    k_color<<<grid_for(ctx, uint64_t(cand_cap) * 32, 8), 256, 0, ctx->stream>>>(a);
    ctx->prof_end();
    ctx->count_launch();
    check_launch(ctx, "k_color");
  }
  changed_out->ctx = ctx;
  changed_out->ensure(std::max<uint32_t>(cand_cap, 1));
  launch_compact_keys(ctx, work.keys.as<uint64_t>(), changed.as<uint8_t>(), work.d_count, cand_cap,
                      changed_out->keys.as<uint64_t>(), changed_out->d_count, ctx->status_w(),
                      "k_compact");
  changed_out->count_hint = cand_cap;
  changed_out->host_valid = false;
  changed_out->host_pending = false;
  changed_out->sorted_unique = true;
  C->stage_meta();
  ctx->sync_status();
  C->adopt_meta();
  const DevStatus& s = *ctx->h_status;
  if (s.bitmap_overflow) throw Error(VXM_ERR_INTERNAL, "candidate bitmap overflow");
  if (s.capacity_error || s.pool_overflow) throw Error(VXM_ERR_CAPACITY, "Layer: block capacity exhausted");
  changed_out->fetch();
}

}  // namespace vxm
