// TSDF / occupancy projective integration (
// occupancy: §8(f) rank 3).
//
// Reference: integrate_impl (proj/src/integrate/integrator.cpp:71-134) with
// integrate_tsdf / integrate_occupancy (:136-158), tsdf_update /
// weight_for_depth (proj/include/voxmap/integrate/updates.hpp:27-54),
// occupancy_update (updates.hpp:59-72), quantize_log_odds (config.hpp:29-31),
// CameraIntrinsics::project/contains (sensor/camera.hpp:35-46), LiDAR project
// (sensor/lidar.hpp:43-55), sample_depth_nearest/linear (sensor/image.hpp:65-106).
//
// B200 design: persistent one-wave grid of 256-thread CTAs, ONE WARP PER
// CANDIDATE BLOCK, 16 voxels per lane (lin = lane + 32 j; no shared memory and
// no block-wide barrier).  The voxel centres are separable, so each lane forms
// the per-axis products R_SL(i, a) * centre_a(v) for its x and two y rows once
// and the z products per voxel pair: every voxel transform is then 9 FP64 adds
// in the reference's association order (bit-exact).  The camera projection's
// two FP64 divides are replaced by an FP32 pre-filter with a rigorous error
// bound: nearest-pixel sampling only needs floor(u), floor(v), so whenever
// [u-E, u+E] contains no integer the FP32 floor is exact; otherwise (rare) the
// exact FP64 path runs.  Voxels are read only when they project onto a valid
// pixel (new blocks are known-zero and are not read at all) and written only
// when their bytes change; each block's changed flag is a warp vote
// (__any_sync) and the changed list is an order-preserving compaction of the
// (sorted) candidate list.
#include <cmath>

#include "runtime.cuh"
#include "scan.cuh"

namespace vxm {

struct IntegrateArgs {
  const uint64_t* cand_keys;
  const int32_t* cand_slots;
  const DevStatus* status_ro;
  void* pool;  // float2 (TSDF) or float (occupancy log-odds) per voxel
  uint8_t* changed;
  uint32_t* stamp_mod;  // Layer::stamp_mod of the changed blocks := mod_epoch
  uint32_t mod_epoch;
  const float* depth;
  const double4* atab;  // LiDAR: atan2 table (vxm_atan2)
  int W, H;
  vxm_pose T_SL;
  int lidar;
  double fu, fv, cu, cv;          // camera
  float fu_f, fv_f, cu_f, cv_f;   // camera, FP32 pre-filter
  double az0, el0, u_scale, v_scale;  // lidar: N/fov, M/fov_el
  int na, ne;
  double vs;
  double max_voxel_depth;
  float eps, max_weight, max_gap;
  int inv_sq, linear;
  float hit, miss, lo_min, lo_max;  // occupancy: quantize_log_odds of the config values
};

// The per-voxel update of each layer kind (the reference's UpdateFn,
// integrator.cpp:136-158).  apply() runs after the common occlusion test
// d_p < -eps (both updates return the voxel unchanged there) and returns
// whether the voxel's bytes change.
template <bool OCC>
struct VoxOps;
template <>
struct VoxOps<false> {  // tsdf_update — updates.hpp:39-54
  using V = float2;
  __device__ static V zero() { return make_float2(0.0f, 0.0f); }
  __device__ static V load_cs(const V* p) { return __ldcs(p); }
  __device__ static bool apply(const IntegrateArgs& a, V o, float d_p, float s, V& nv) {
    float w_new = 1.0f;
    if (a.inv_sq) {  // weight_for_depth — updates.hpp:27-32
      const double dd = __dmul_rn(double(s), double(s));
      w_new = __double2float_rn(__ddiv_rn(1.0, dd < 1e-6 ? 1e-6 : dd));
    }
    const float d_t = d_p < -a.eps ? -a.eps : (a.eps < d_p ? a.eps : d_p);
    const float w_sum = __fadd_rn(o.y, w_new);
    const float avg = __fdiv_rn(__fadd_rn(__fmul_rn(o.y, o.x), __fmul_rn(w_new, d_t)), w_sum);
    nv.x = avg < -a.eps ? -a.eps : (a.eps < avg ? a.eps : avg);
    nv.y = a.max_weight < w_sum ? a.max_weight : w_sum;
    return __float_as_uint(nv.x) != __float_as_uint(o.x) || __float_as_uint(nv.y) != __float_as_uint(o.y);
  }
};
template <>
struct VoxOps<true> {  // occupancy_update — updates.hpp:59-72
  using V = float;
  __device__ static V zero() { return 0.0f; }
  __device__ static V load_cs(const V* p) { return __ldcs(p); }
  __device__ static bool apply(const IntegrateArgs& a, V o, float d_p, float, V& nv) {
    const float v = __fadd_rn(o, d_p <= 0.0f ? a.hit : a.miss);
    nv = v < a.lo_min ? a.lo_min : (a.lo_max < v ? a.lo_max : v);  // std::clamp
    return __float_as_uint(nv) != __float_as_uint(o);
  }
};

// d > 0 && isfinite(d): the positive finite floats are the bit patterns 1 .. 0x7f7fffff
__device__ inline bool valid_depth_i(float d) { return __float_as_uint(d) - 1u < 0x7f7fffffu; }

// ---- FP64 atan2 for the LiDAR projection ----------------------------------------
// lidar.hpp:43-55 evaluates atan2 (azimuth) and acos (polar angle) per voxel;
// the CUDA libm versions were half of k_integrate's LiDAR instructions (one in
// six of them materialising polynomial constants).  vxm_atan2 instead rotates
// (x, y) by a table vector near its angle and sums a short series:
//   octant o = (|y| > |x|, x < 0, y < 0), t = min/max of |x|, |y| in FP32,
//   k     = round(128 t): the table direction of octant o at base angle
//           atan(k/128) (mirrored into the octant: pi/2 - a, pi - a, -a)
//   (c,s) = that direction's (cos, sin) rounded to double; psi = the exact
//           angle atan2(s, c) of the rounded vector as a double-double
//           (host long double, kAtanTabN = 8 x 129 entries)
//   x' = x c + y s,  y' = y c - x s      (y' by Kahan's difference of products)
//   atan2(y, x) = psi + atan(y'/x'),  |y'/x'| < 0.005:  q - q^3/3 + q^5/5 - q^7/7
// (the octant and t replace an FP32 polynomial estimate of the angle: the
// table index needs no arctangent).  Accuracy ~1 ulp (libm class: glibc and
// CUDA libm also differ in the last ulp); the tolerance
// tests (tests/helpers.py:36) and tests/test_gpu_lidar_angles.py cover it.
// y == 0 (signed zero / -pi vs pi) goes to the libm routine.
constexpr int kAtanK = 128;
constexpr int kAtanTabN = 8 * (kAtanK + 1);

// sqrt to ~1 ulp (an atan2 argument; not the depth, which stays correctly
// rounded): MUFU.RSQ64H seed + two Newton steps, 0 for 0.
__device__ inline double sqrt_approx(double h2) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(h2));
  y = y * fma(-0.5 * h2, y * y, 1.5);
  y = y * fma(-0.5 * h2, y * y, 1.5);
  return h2 > 0.0 ? h2 * y : 0.0;
}
__constant__ double kAtanQ[3] = {-1.0 / 3.0, 1.0 / 5.0, -1.0 / 7.0};

__device__ inline double vxm_atan2(double y, double x, const double4* __restrict__ tab) {
  if (y == 0.0) return atan2(y, x);
  const float ax = fabsf(float(x)), ay = fabsf(float(y));
  const bool sw = ay > ax;
  float rm;  // 1 / max (MUFU.RCP): t only picks the table entry
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rm) : "f"(sw ? ay : ax));
  const int k = __float2int_rn((sw ? ax : ay) * rm * float(kAtanK));
  // octant from the sign bits (y != 0 here; x = -0 and +0 give the same
  // direction, pi / 2, at t = 0)
  const int o = (sw ? 1 : 0) | ((__double2hiint(x) >> 30) & 2) | ((__double2hiint(y) >> 29) & 4);
  const double2* tp = reinterpret_cast<const double2*>(tab + (o * (kAtanK + 1) + k));
  const double2 CS = __ldg(tp), PSI = __ldg(tp + 1);  // (c, s), (psi_hi, psi_lo)
  const double xr = fma(x, CS.x, y * CS.y);
  const double w = x * CS.y;
  const double yr = fma(y, CS.x, -w) - fma(x, CS.y, -w);
  // q = yr / xr (xr > 0): approximate reciprocal (MUFU.RCP64H) + two Newton steps
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(xr));
  r = fma(r, fma(-xr, r, 1.0), r);
  r = fma(r, fma(-xr, r, 1.0), r);
  const double q = yr * r, q2 = q * q;
  const double d = fma(q * q2, fma(q2, fma(q2, kAtanQ[2], kAtanQ[1]), kAtanQ[0]), q);
  return PSI.x + (PSI.y + d);
}

// polar angle acos(z / |p|) = atan2(|(x, y)|, z) (lidar.hpp:53)
__device__ inline double lidar_polar(double px, double py, double pz, const double4* tab) {
  const double hxy = sqrt_approx(__dadd_rn(__dmul_rn(px, px), __dmul_rn(py, py)));
  return hxy == 0.0 ? (pz > 0.0 ? 0.0 : 3.141592653589793) : vxm_atan2(hxy, pz, tab);
}

__device__ inline bool sample_nearest_d(const float* img, int W, int H, double u, double v,
                                        float* out) {
  const int col = int(floor(u)), row = int(floor(v));
  if (u < 0.0 || v < 0.0 || col >= W || row >= H) return false;
  const float d = __ldg(img + size_t(row) * W + col);
  if (!valid_depth_i(d)) return false;
  *out = d;
  return true;
}

// sample_depth_linear — image.hpp:79-106
__device__ inline bool sample_linear_d(const float* img, int W, int H, double u, double v,
                                       float gap, float* out) {
  const double gu = __dsub_rn(u, 0.5), gv = __dsub_rn(v, 0.5);
  const double fx0 = floor(gu), fy0 = floor(gv);
  const int x0 = int(fx0), y0 = int(fy0);
  // x0 < 0 || x0 + 1 >= W (and the same for y) as one unsigned compare each
  if (unsigned(x0) >= unsigned(W - 1) || unsigned(y0) >= unsigned(H - 1)) return false;
  const float d00 = __ldg(img + size_t(y0) * W + x0), d10 = __ldg(img + size_t(y0) * W + x0 + 1);
  const float d01 = __ldg(img + size_t(y0 + 1) * W + x0);
  const float d11 = __ldg(img + size_t(y0 + 1) * W + x0 + 1);
  if (!valid_depth_i(d00) || !valid_depth_i(d10) || !valid_depth_i(d01) || !valid_depth_i(d11))
    return false;
  float lo = d00, hi = d00;
  lo = d10 < lo ? d10 : lo; hi = hi < d10 ? d10 : hi;
  lo = d01 < lo ? d01 : lo; hi = hi < d01 ? d01 : hi;
  lo = d11 < lo ? d11 : lo; hi = hi < d11 ? d11 : hi;
  if (__fsub_rn(hi, lo) > gap) return false;
  const double wx = __dsub_rn(gu, fx0), wy = __dsub_rn(gv, fy0);  // (fx0 == double(x0))
  const double omx = __dsub_rn(1.0, wx), omy = __dsub_rn(1.0, wy);
  const double top = __dadd_rn(__dmul_rn(omx, double(d00)), __dmul_rn(wx, double(d10)));
  const double bot = __dadd_rn(__dmul_rn(omx, double(d01)), __dmul_rn(wx, double(d11)));
  const double d = __dadd_rn(__dmul_rn(omy, top), __dmul_rn(wy, bot));
  *out = __double2float_rn(d);
  return true;
}

// Exact-floor FP32 pre-filter for one projected coordinate.  Returns true and
// sets *idx when floor(u_exact) is certain; u_exact = (f*x)/z + c in FP64.
__device__ inline bool fast_floor(float f, float c, float xf, float zf, int* idx) {
  // approximate division (<= 2 ulp): the bound E below covers >= 16 units
  const float t = __fdividef(__fmul_rn(f, xf), zf);
  const float u = __fadd_rn(t, c);
  const float E = __fmul_rn(__fadd_rn(__fadd_rn(fabsf(t), fabsf(c)), fabsf(u)), 9.5367431640625e-07f) +
                  1e-30f;  // (|t| + |c| + |u|) * 2^-20 >= 16 units of the error
  const float lo = floorf(__fsub_rn(u, E)), hi = floorf(__fadd_rn(u, E));
  if (!(lo == hi) || !(fabsf(lo) < 1.0e9f)) return false;
  *idx = int(lo);
  return true;
}

// One voxel: projection, sample, update (integrator.cpp:98-123); returns
// whether its bytes changed.  p = T_SL * centre (FP64, pinned order).
template <bool OCC, bool LIDAR, bool LINEAR>
__device__ inline bool integrate_voxel(const IntegrateArgs& a, typename VoxOps<OCC>::V* blk, int lin, double px,
                                       double py, double pz, bool is_new, uint32_t& n_read,
                                       uint32_t& n_upd) {
  double d_v;
  if (!LIDAR) {
    d_v = pz;  // CameraIntrinsics::depth_of — camera.hpp:49
  } else {     // LidarIntrinsics::depth_of — lidar.hpp:62
    d_v = __dsqrt_rn(__dadd_rn(__dmul_rn(px, px), __dadd_rn(__dmul_rn(py, py), __dmul_rn(pz, pz))));
  }
  if (!(d_v > 0.0) || d_v > a.max_voxel_depth) return false;  // integrator.cpp:104-107
  using Ops = VoxOps<OCC>;
  using V = typename Ops::V;
  float s;
  bool ok;
  V old = Ops::zero();
  bool have_old = false;
  if (!LIDAR) {
    if (!LINEAR) {
      int col, row;
      const float xf = __double2float_rn(px), yf = __double2float_rn(py), zf = __double2float_rn(pz);
      if (!(fast_floor(a.fu_f, a.cu_f, xf, zf, &col) && fast_floor(a.fv_f, a.cv_f, yf, zf, &row))) {
        // exact FP64 projection — camera.hpp:39-40
        const double u = __dadd_rn(__ddiv_rn(__dmul_rn(a.fu, px), pz), a.cu);
        const double v = __dadd_rn(__ddiv_rn(__dmul_rn(a.fv, py), pz), a.cv);
        if (!(u >= 0.0 && u < double(a.W) && v >= 0.0 && v < double(a.H))) return false;
        col = int(floor(u));
        row = int(floor(v));
      }
      if (col < 0 || row < 0 || col >= a.W || row >= a.H) return false;
      // the old voxel is loaded together with the depth sample (one round trip)
      if (!is_new) {
        old = blk[lin];
        have_old = true;
      }
      s = __ldg(a.depth + size_t(row) * a.W + col);
      ok = valid_depth_i(s);
    } else {
      const double u = __dadd_rn(__ddiv_rn(__dmul_rn(a.fu, px), pz), a.cu);
      const double v = __dadd_rn(__ddiv_rn(__dmul_rn(a.fv, py), pz), a.cv);
      if (!(u >= 0.0 && u < double(a.W) && v >= 0.0 && v < double(a.H))) return false;
      ok = sample_linear_d(a.depth, a.W, a.H, u, v, a.max_gap, &s);
    }
  } else {
    // LidarIntrinsics::project — lidar.hpp:43-55: polar = acos(z / |p|)
    // (= atan2(|(x, y)|, z)) and azimuth = atan2(y, x), both by vxm_atan2.
    // The elevation is evaluated first: a voxel outside the beam fan then
    // needs no azimuth (C3 k_integrate -5 %).
    const double polar = lidar_polar(px, py, pz, a.atab);
    const double v = __dmul_rn(__dsub_rn(polar, a.el0), a.v_scale);
    if (!(v >= 0.0 && v < double(a.ne))) return false;
    const double kTwoPi = 6.283185307179586;
    double az = __dsub_rn(vxm_atan2(py, px, a.atab), a.az0);
    // az - 2 pi floor(az / 2 pi): when 0 <= az < 2 pi (1 - 2^-40) the quotient
    // is certainly in [0, 1) and the floor is 0 (no division); otherwise the
    // exact expression
    if (!(az >= 0.0 && az < 6.283185307173872)) az = __dsub_rn(az, __dmul_rn(kTwoPi, floor(__ddiv_rn(az, kTwoPi))));
    const double u = __dmul_rn(az, a.u_scale);
    if (!(u >= 0.0 && u < double(a.na))) return false;
    ok = LINEAR ? sample_linear_d(a.depth, a.W, a.H, u, v, a.max_gap, &s)
                : sample_nearest_d(a.depth, a.W, a.H, u, v, &s);
  }
  if (!ok) return false;
  const float d_p = __fsub_rn(s, __double2float_rn(d_v));  // integrator.cpp:116
  if (d_p < -a.eps) return false;  // occluded: voxel unchanged (updates.hpp:42, :62)
  if (!is_new && !have_old) old = blk[lin];
  n_read += is_new ? 0u : 1u;
  V nv;
  if (Ops::apply(a, old, d_p, s, nv)) {
    blk[lin] = nv;
    ++n_upd;
    return true;
  }
  return false;
}

// One warp per candidate block, 16 voxels per lane (lin = lane + 32 j): many
// independent voxels per lane hide the depth-gather and voxel latencies, and
// there is no block-wide barrier.  The per-axis products R_SL(i, a) *
// centre_a(v) are formed per lane (bit-identical to the reference's
// R * centre rows, pose.hpp:58-60 with the pinned a0 + (a1 + a2) order).
// FASTCAM: camera + nearest sampling (the C2 path: 4 CTAs / SM, 64 registers);
// otherwise the general per-voxel path (LiDAR / linear: 3 CTAs / SM).  The
// occupancy is the measured optimum of each (C2 -13 %, C3 -8 % kernel time vs
// the register-unbounded build).
// MODE: kIntegCamNearest (FASTCAM), kIntegCamLinear, kIntegLidarNearest,
// kIntegLidarLinear — the sensor and sampling are compile-time in each.
constexpr int kIntegCamNearest = 0, kIntegCamLinear = 1, kIntegLidarNearest = 2, kIntegLidarLinear = 3;
template <bool OCC, int MODE>
#ifndef VXM_INTEG_GEN_MINB
#define VXM_INTEG_GEN_MINB 4
#endif
__global__ void __launch_bounds__(256, MODE == kIntegCamNearest ? 4 : VXM_INTEG_GEN_MINB) k_integrate(IntegrateArgs a) {
  constexpr bool FASTCAM = MODE == kIntegCamNearest;
  constexpr bool LIDAR = MODE >= kIntegLidarNearest;
  constexpr bool LINEAR = MODE == kIntegCamLinear || MODE == kIntegLidarLinear;
  pdl_wait();  // see launch_pdl
  pdl_trigger();
  using Ops = VoxOps<OCC>;
  using V = typename Ops::V;
  const DevStatus* st = a.status_ro;
  if (st->pool_overflow || st->capacity_error || st->bitmap_overflow) return;
  const uint32_t n = st->n_candidates;
  const double* R = a.T_SL.R;
  const int lane = threadIdx.x & 31;
  uint32_t n_read = 0, n_upd = 0;  // work counters (algorithmic bytes)
  DevStatus* const claim_st = const_cast<DevStatus*>(st);
  // each warp's first block by its index, then (general path) a dynamic
  // schedule: the next candidate is claimed when a warp is done — LiDAR blocks
  // differ widely in work (new, occluded, far), and a static stride left up to
  // a third of the SM time idle at the tail (C3 k_integrate -11 %); the camera
  // fast path (~2 blocks per warp) keeps the static stride (a claim costs more
  // than it balances there)
  const uint32_t nwarps = gridDim.x * (blockDim.x >> 5);
  uint32_t stride_next = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  auto claim = [&]() -> uint32_t {
    if (FASTCAM) return stride_next += nwarps;
    uint32_t c = 0;
    if (lane == 0) c = atomicAdd(&claim_st->integ_claim, 1u);
    return nwarps + __shfl_sync(0xffffffffu, c, 0);
  };
  for (uint32_t ci = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; ci < n; ci = claim()) {
    const uint64_t key = a.cand_keys[ci];
    const int32_t sraw = a.cand_slots[ci];
    const bool is_new = sraw < 0;
    const int32_t slot = sraw & 0x7fffffff;
    V* blk = static_cast<V*>(a.pool) + size_t(slot) * kVPB;
    // voxel_center — indexing.hpp:113-119: ((g * 8 + v) + 0.5) * vs
    auto centre = [&](int32_t g, int v) {
      return __dmul_rn(__dadd_rn(__dadd_rn(__dmul_rn(double(g), 8.0), double(v)), 0.5), a.vs);
    };
    const int vx = lane & 7, vy0 = lane >> 3;
    const double cx = centre(key_x(key), vx);
    const double cy0 = centre(key_y(key), vy0), cy1 = centre(key_y(key), vy0 + 4);
    double Ax[3], Ay0[3], Ay1[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      Ax[i] = __dmul_rn(R[3 * i], cx);
      Ay0[i] = __dmul_rn(R[3 * i + 1], cy0);
      Ay1[i] = __dmul_rn(R[3 * i + 1], cy1);
    }
    const int32_t gz = key_z(key);
    bool any = false;
    if (FASTCAM) {
      // camera, nearest sampling (the hot configuration): per chunk of 4 voxels
      // all depth samples and old voxels are loaded before any is used
#pragma unroll 1
      for (int j0 = 0; j0 < 16; j0 += 4) {
        float sd[4];
        V ov[4];
        float dv[4];
        uint32_t live = 0;
        // voxels j and j + 1 share z (j even): R(i, z) * c_z once per z
        double Rz[2][3];
#pragma unroll
        for (int zi = 0; zi < 2; ++zi) {
          const double cz = centre(gz, (j0 >> 1) + zi);
          Rz[zi][0] = __dmul_rn(R[2], cz);
          Rz[zi][1] = __dmul_rn(R[5], cz);
          Rz[zi][2] = __dmul_rn(R[8], cz);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          // p = (A_x + (A_y + R_z c_z)) + t — pose.hpp:58-60, the pinned a0 + (a1 + a2) order
          const double* Ay = (q & 1) ? Ay1 : Ay0;
          const double* rz = Rz[q >> 1];
          const double pz = __dadd_rn(__dadd_rn(Ax[2], __dadd_rn(Ay[2], rz[2])), a.T_SL.t[2]);
          const double px = __dadd_rn(__dadd_rn(Ax[0], __dadd_rn(Ay[0], rz[0])), a.T_SL.t[0]);
          const double py = __dadd_rn(__dadd_rn(Ax[1], __dadd_rn(Ay[1], rz[1])), a.T_SL.t[1]);
          const int lin = lane + 32 * (j0 + q);
          sd[q] = 0.0f;
          ov[q] = Ops::zero();
          dv[q] = __double2float_rn(pz);
          if (!(pz > 0.0) || pz > a.max_voxel_depth) continue;  // integrator.cpp:104-107
          int col, row;
          const float xf = __double2float_rn(px), yf = __double2float_rn(py), zf = dv[q];
          if (!(fast_floor(a.fu_f, a.cu_f, xf, zf, &col) && fast_floor(a.fv_f, a.cv_f, yf, zf, &row))) {
            const double u = __dadd_rn(__ddiv_rn(__dmul_rn(a.fu, px), pz), a.cu);  // camera.hpp:39-40
            const double v = __dadd_rn(__ddiv_rn(__dmul_rn(a.fv, py), pz), a.cv);
            if (!(u >= 0.0 && u < double(a.W) && v >= 0.0 && v < double(a.H))) continue;
            col = int(floor(u));
            row = int(floor(v));
          }
          if (col < 0 || row < 0 || col >= a.W || row >= a.H) continue;
          sd[q] = __ldg(a.depth + size_t(row) * a.W + col);
          if (!is_new) ov[q] = Ops::load_cs(blk + lin);
          live |= 1u << q;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (!((live >> q) & 1u) || !valid_depth_i(sd[q])) continue;
          const float d_p = __fsub_rn(sd[q], dv[q]);  // integrator.cpp:116
          if (d_p < -a.eps) continue;                 // occluded (updates.hpp:42, :62)
          n_read += is_new ? 0u : 1u;
          V nv;
          if (Ops::apply(a, ov[q], d_p, sd[q], nv)) {
            blk[lane + 32 * (j0 + q)] = nv;
            ++n_upd;
            any = true;
          }
        }
      }
    } else {
      // voxels j and j + 1 share z: R(i, z) * c_z once per pair;
      // p = (A_x + (A_y + R_z c_z)) + t as in the camera path
      // voxel_center's ((g * 8 + v) + 0.5) * vs with g * 8 once per block
      // (the same operands as centre())
      const double gz8 = __dmul_rn(double(gz), 8.0);
#pragma unroll 1
      for (int j0 = 0; j0 < 16; j0 += 2) {
        const double cz = __dmul_rn(__dadd_rn(__dadd_rn(gz8, double(j0 >> 1)), 0.5), a.vs);
        const double rz0 = __dmul_rn(R[2], cz), rz1 = __dmul_rn(R[5], cz), rz2 = __dmul_rn(R[8], cz);
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const double* Ay = q ? Ay1 : Ay0;
          const double pz = __dadd_rn(__dadd_rn(Ax[2], __dadd_rn(Ay[2], rz2)), a.T_SL.t[2]);
          const double px = __dadd_rn(__dadd_rn(Ax[0], __dadd_rn(Ay[0], rz0)), a.T_SL.t[0]);
          const double py = __dadd_rn(__dadd_rn(Ax[1], __dadd_rn(Ay[1], rz1)), a.T_SL.t[1]);
          any |= integrate_voxel<OCC, LIDAR, LINEAR>(a, blk, lane + 32 * (j0 + q), px, py, pz, is_new, n_read,
                                                    n_upd);
        }
      }
    }
    any = __any_sync(0xffffffffu, any);
    if (lane == 0) {
      a.changed[ci] = uint8_t(any);
      if (any) a.stamp_mod[slot] = a.mod_epoch;
    }
  }
  n_read = __reduce_add_sync(0xffffffffu, n_read);
  n_upd = __reduce_add_sync(0xffffffffu, n_upd);
  if (lane == 0 && (n_read | n_upd)) {
    DevStatus* sw = const_cast<DevStatus*>(st);
    atomicAdd(&sw->vox_read, n_read);
    atomicAdd(&sw->vox_upd, n_upd);
  }
}

// Order-preserving compaction of keys by flag; count read from the device.
constexpr int kCompactItems = 4;
__global__ void __launch_bounds__(256) k_compact_keys(const uint64_t* __restrict__ in,
                                                      const uint8_t* __restrict__ flags,
                                                      const uint32_t* n_ptr, uint64_t* out,
                                                      uint32_t* n_out, ScanTiles st,
                                                      const DevStatus* guard) {
  pdl_wait();  // see launch_pdl
  pdl_trigger();
  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_scan[64];
  __shared__ uint32_t s_pre;
  scan_prepare_next(st);
  const bool skip = guard && (guard->pool_overflow || guard->capacity_error || guard->bitmap_overflow);
  const uint32_t n = skip ? 0u : *n_ptr;
  const uint32_t per_tile = blockDim.x * kCompactItems;
  const uint32_t tiles = (n + per_tile - 1) / per_tile;
  if (tiles == 0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) *n_out = 0;
    return;
  }
  while (true) {
    const uint32_t tile = scan_take_tile(st, &s_tile);
    if (tile >= tiles) break;
    const uint32_t base = tile * per_tile + threadIdx.x * kCompactItems;
    uint32_t keep = 0;
#pragma unroll
    for (int k = 0; k < kCompactItems; ++k)
      if (base + k < n && flags[base + k]) keep |= 1u << k;
    uint32_t ea, eb, ta, tb;
    block_scan2(__popc(keep), 0u, ea, eb, ta, tb, s_scan);
    if (threadIdx.x < 32) {  // warp 0: look-back
      uint32_t pa, pb;
      scan_lookback(st, tile, ta, 0u, pa, pb);
      if (threadIdx.x == 0) {
        s_pre = pa;
        if (tile == tiles - 1) *n_out = pa + ta;
      }
    }
    __syncthreads();
    uint32_t pos = s_pre + ea;
#pragma unroll
    for (int k = 0; k < kCompactItems; ++k)
      if (keep & (1u << k)) out[pos++] = in[base + k];
    __syncthreads();
  }
}

void launch_compact_keys(Context* ctx, const uint64_t* in, const uint8_t* flags,
                         const uint32_t* n_ptr, uint32_t n_cap, uint64_t* out, uint32_t* n_out,
                         const DevStatus* guard, const char* prof_name) {
  const uint32_t tiles_cap = ceil_div(std::max<uint32_t>(n_cap, 1), 256 * kCompactItems);
  const ScanTiles st = ctx->next_scan(tiles_cap);
  const uint32_t grid = std::max<uint32_t>(1, std::min<uint32_t>(tiles_cap, ctx->sm_count * 4));
  ctx->prof_begin(prof_name);
  launch_pdl(ctx->stream, k_compact_keys, dim3(grid), dim3(256), 0, in, flags, n_ptr, out, n_out, st, guard);
  ctx->prof_end();
  ctx->count_launch();
  check_launch(ctx, "k_compact_keys");
}

// quantize_log_odds — integrate/config.hpp:29-31 (host, as the reference)
static float quantize_log_odds(float v) {
  return static_cast<float>(std::nearbyint(double(v) * 4096.0) / 4096.0);
}

// The vxm_atan2 table (host long double): entry o * 129 + k holds (c, s) =
// (cos, sin) of octant o's direction at base angle atan(k / 128), rounded to
// double, and the exact angle of that rounded vector as a double-double.
static const double4* ensure_atan_table(Context* ctx) {
  if (ctx->atan_tab.p) return ctx->atan_tab.as<const double4>();
  std::vector<double4> t(kAtanTabN);
  const long double pi = 3.141592653589793238462643383279502884L;
  for (int o = 0; o < 8; ++o) {
    for (int k = 0; k <= kAtanK; ++k) {
      long double phi = atanl((long double)k / kAtanK);
      if (o & 1) phi = pi / 2 - phi;  // |y| > |x|
      if (o & 2) phi = pi - phi;      // x < 0
      if (o & 4) phi = -phi;          // y < 0
      const double c = double(cosl(phi)), s = double(sinl(phi));
      long double psi = atan2l((long double)s, (long double)c);
      psi += 2.0L * pi * roundl((phi - psi) / (2.0L * pi));  // phi = +-pi: the side of +-pi it is on
      const double hi = double(psi);
      t[o * (kAtanK + 1) + k] = make_double4(c, s, hi, double(psi - (long double)hi));
    }
  }
  ctx->atan_tab.ensure(sizeof(double4) * t.size());
  VXM_CUDA(cudaMemcpyAsync(ctx->atan_tab.p, t.data(), sizeof(double4) * t.size(), cudaMemcpyHostToDevice,
                           ctx->stream));
  VXM_CUDA(cudaStreamSynchronize(ctx->stream));
  return ctx->atan_tab.as<const double4>();
}

// vxm_diag_lidar_angles: the projection's two angles, as integrate_voxel
// evaluates them.
__global__ void k_diag_angles(const double* __restrict__ xyz, uint64_t n, const double4* tab, double* az,
                              double* polar) {
  for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x) {
    const double x = xyz[3 * i], y = xyz[3 * i + 1], z = xyz[3 * i + 2];
    az[i] = vxm_atan2(y, x, tab);
    polar[i] = lidar_polar(x, y, z, tab);
  }
}
void diag_lidar_angles(Context* ctx, const double* xyz, uint64_t n, double* az, double* polar) {
  if (n == 0) return;
  const double4* tab = ensure_atan_table(ctx);
  DevBuf d;
  d.ensure(sizeof(double) * 5 * n);
  double* dx = d.as<double>();
  VXM_CUDA(cudaMemcpyAsync(dx, xyz, sizeof(double) * 3 * n, cudaMemcpyHostToDevice, ctx->stream));
  k_diag_angles<<<std::max<uint64_t>(1, std::min<uint64_t>(4096, (n + 255) / 256)), 256, 0, ctx->stream>>>(
      dx, n, tab, dx + 3 * n, dx + 4 * n);
  ctx->count_launch();
  VXM_CUDA(cudaMemcpyAsync(az, dx + 3 * n, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
  VXM_CUDA(cudaMemcpyAsync(polar, dx + 4 * n, sizeof(double) * n, cudaMemcpyDeviceToHost, ctx->stream));
  VXM_CUDA(cudaStreamSynchronize(ctx->stream));
}

uint32_t integrate_launch(Layer* L, const ViewArgs& va, const vxm_integrator_config& cfg,
                          BlockList* changed_out) {
  Context* ctx = L->ctx;
  // Headroom: a frame cannot allocate more blocks than it has candidates;
  // the bound below is generous, the device check catches the rest.
  L->ensure_capacity(std::min<uint64_t>(uint64_t(L->num_blocks) + 65536, L->max_blocks));
  uint32_t cand_cap = 0;
  run_view(ctx, va, L, &cand_cap);
  ctx->cand_flags.ensure(cand_cap);
  IntegrateArgs a{};
  a.cand_keys = ctx->cand_keys.as<uint64_t>();
  a.cand_slots = ctx->cand_slots.as<int32_t>();
  a.status_ro = ctx->status_w();
  a.pool = L->pool[0];
  a.changed = ctx->cand_flags.as<uint8_t>();
  a.stamp_mod = L->stamp_mod;
  a.mod_epoch = next_mod_tick();
  a.depth = va.depth_dev;
  if (va.lidar) a.atab = ensure_atan_table(ctx);
  a.W = va.width;
  a.H = va.height;
  vxm_pose_inverse(&va.T_LS, &a.T_SL);  // integrator.cpp:89 (host, pinned order)
  a.lidar = va.lidar ? 1 : 0;
  a.fu = va.cam.fu; a.fv = va.cam.fv; a.cu = va.cam.cu; a.cv = va.cam.cv;
  a.fu_f = float(va.cam.fu); a.fv_f = float(va.cam.fv);
  a.cu_f = float(va.cam.cu); a.cv_f = float(va.cam.cv);
  a.az0 = va.li.azimuth_start;
  a.el0 = va.li.elevation_start;
  a.u_scale = va.li.num_azimuth / va.li.azimuth_fov;
  a.v_scale = va.li.num_elevation / va.li.elevation_fov;
  a.na = va.li.num_azimuth;
  a.ne = va.li.num_elevation;
  a.vs = L->vs;
  a.max_voxel_depth = cfg.max_integration_distance + cfg.truncation;
  a.eps = float(cfg.truncation);
  a.max_weight = cfg.max_weight;
  a.max_gap = cfg.max_sample_gap;
  a.inv_sq = cfg.weighting == VXM_WEIGHT_INVERSE_SQUARE;
  a.linear = (va.lidar ? cfg.lidar_sample : cfg.camera_sample) == VXM_SAMPLE_LINEAR;
  a.hit = quantize_log_odds(cfg.hit_log_odds);
  a.miss = quantize_log_odds(cfg.miss_log_odds);
  a.lo_min = quantize_log_odds(cfg.log_odds_min);
  a.lo_max = quantize_log_odds(cfg.log_odds_max);
  const bool occ = L->type == VXM_LAYER_OCCUPANCY;
  const int mode = a.lidar ? (a.linear ? kIntegLidarLinear : kIntegLidarNearest)
                           : (a.linear ? kIntegCamLinear : kIntegCamNearest);
  void (*const kerns[2][4])(IntegrateArgs) = {
      {k_integrate<false, kIntegCamNearest>, k_integrate<false, kIntegCamLinear>,
       k_integrate<false, kIntegLidarNearest>, k_integrate<false, kIntegLidarLinear>},
      {k_integrate<true, kIntegCamNearest>, k_integrate<true, kIntegCamLinear>,
       k_integrate<true, kIntegLidarNearest>, k_integrate<true, kIntegLidarLinear>}};
  void (*kern)(IntegrateArgs) = kerns[occ ? 1 : 0][mode];
  // resident CTAs per SM: the persistent grid is one wave
  const int per_sm = ctx->resident_per_sm((const void*)kern, 256);
  const uint32_t grid = std::max<uint32_t>(1, std::min<uint32_t>(cand_cap, ctx->sm_count * per_sm));
  host_trace_dev(ctx, "dilate");
  ctx->prof_begin("k_integrate");
  launch_pdl(ctx->stream, kern, dim3(grid), dim3(256), 0, a);
  ctx->prof_end();
  ctx->count_launch();
  check_launch(ctx, "k_integrate");
  changed_out->ensure(cand_cap);
  launch_compact_keys(ctx, ctx->cand_keys.as<uint64_t>(), ctx->cand_flags.as<uint8_t>(),
                      &ctx->d_status->n_candidates, cand_cap, changed_out->keys.as<uint64_t>(),
                      changed_out->d_count, ctx->status_w(), "k_compact");
  changed_out->host_valid = false;
  changed_out->host_pending = false;
  // changed blocks are distinct allocated blocks: bounded by the pool too
  changed_out->count_hint = std::min<uint32_t>(cand_cap, L->capacity);
  if (changed_out->want_host) changed_out->enqueue_host();  // host result, same sync
  ctx->queue_copy(changed_out->d_count, &ctx->d_status->n_changed);
  return cand_cap;
}

bool integrate_finish(Layer* L, const ViewArgs& va, BlockList* changed_out, uint32_t nb_before) {
  Context* ctx = L->ctx;
  const DevStatus& s = *ctx->h_status;
  if (s.bitmap_overflow)
    throw Error(VXM_ERR_INTERNAL, "candidate ray left the candidate cube (bitmap bound)");
  if (s.pool_overflow) {
    // No voxel was touched: grow to fit and run the frame again (blocks
    // already inserted are zero and count as existing on the re-run).
    L->ensure_capacity(std::min<uint64_t>(uint64_t(nb_before) + s.n_new + 1024, L->max_blocks));
    return false;
  }
  if (s.capacity_error) throw Error(VXM_ERR_CAPACITY, "Layer: block capacity exhausted");
  changed_out->count_hint = s.n_candidates;
  vxm_stats& w = ctx->stats;
  w.integrate_calls += 1;
  w.candidate_blocks += s.n_candidates;
  w.new_blocks += s.n_new;
  w.changed_blocks += s.n_changed;
  w.voxels_read += s.vox_read;
  w.voxels_updated += s.vox_upd;
  w.depth_pixels += uint64_t(va.width) * uint64_t(va.height);
  return true;
}

void run_integrate(Layer* L, const ViewArgs& va, const vxm_integrator_config& cfg,
                   BlockList* changed_out) {
  Context* ctx = L->ctx;
  for (int attempt = 0; attempt < 4; ++attempt) {
    ctx->reset_status();
    const uint32_t nb_before = L->num_blocks;
    integrate_launch(L, va, cfg, changed_out);
    L->stage_meta();
    host_trace_mark("launched");
    host_trace_dev(ctx, "kernels");
    ctx->sync_status(true);
    L->adopt_meta();
    if (integrate_finish(L, va, changed_out, nb_before)) return;
  }
  throw Error(VXM_ERR_INTERNAL, "integrate: pool growth did not converge");
}

}  // namespace vxm
