// Synthetic inputs (host, OpenMP) — see include/voxmap_b200_synth.h.
// Arithmetic follows the reference's expressions in the pinned association
// order of oracle/eigen_shim (3-term sums a0 + (a1 + a2)) so the rendered
// frames match the reference's render_depth bit-for-bit (tests check this).
#include <algorithm>
#include <cmath>
#include <limits>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "voxmap_b200_synth.h"

namespace {

struct V3 {
  double x, y, z;
};
inline V3 add(V3 a, V3 b) { return {a.x + b.x, a.y + b.y, a.z + b.z}; }
inline V3 sub(V3 a, V3 b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }
inline V3 mul(double s, V3 a) { return {s * a.x, s * a.y, s * a.z}; }
inline double sum3(double a0, double a1, double a2) { return a0 + (a1 + a2); }
inline double dot(V3 a, V3 b) { return sum3(a.x * b.x, a.y * b.y, a.z * b.z); }
inline double norm(V3 a) { return std::sqrt(dot(a, a)); }
inline V3 normalized(V3 a) {
  const double z = dot(a, a);
  return z > 0.0 ? V3{a.x / std::sqrt(z), a.y / std::sqrt(z), a.z / std::sqrt(z)} : a;
}
inline V3 cross(V3 a, V3 b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
inline V3 rot(const double* R, V3 p) {  // row-major R * p
  return {sum3(R[0] * p.x, R[1] * p.y, R[2] * p.z), sum3(R[3] * p.x, R[4] * p.y, R[5] * p.z),
          sum3(R[6] * p.x, R[7] * p.y, R[8] * p.z)};
}

struct Prim {
  int kind;  // 0 sphere, 1 box, 2 plane
  V3 a, b;   // sphere: center,(r,_,_); box: min,max; plane: point,normal
  double r;
};

}  // namespace

struct vxm_scene {
  std::string name;
  std::vector<Prim> prims;
  V3 lo{0, 0, 0}, hi{0, 0, 0};

  // ScenePrimitive::sdf — scene.cpp:56-72
  static double prim_sdf(const Prim& p, V3 q) {
    switch (p.kind) {
      case 0:
        return norm(sub(q, p.a)) - p.r;
      case 1: {
        const V3 mid = mul(0.5, add(p.a, p.b));
        const V3 half = mul(0.5, sub(p.b, p.a));
        const V3 d = sub(q, mid);
        const V3 e = {std::abs(d.x) - half.x, std::abs(d.y) - half.y, std::abs(d.z) - half.z};
        const V3 o = {std::max(e.x, 0.0), std::max(e.y, 0.0), std::max(e.z, 0.0)};
        const double outside = norm(o);
        const double mx = std::max(e.x, std::max(e.y, e.z));
        const double inside = std::min(mx, 0.0);
        return outside + inside;
      }
      default:
        return dot(p.b, sub(q, p.a));
    }
  }
  // SyntheticScene::sdf — scene.cpp:104-110
  double sdf(V3 q) const {
    double best = std::numeric_limits<double>::infinity();
    for (const Prim& p : prims) best = std::min(best, prim_sdf(p, q));
    return best;
  }
  void plane(V3 point, V3 n) {  // make_plane — scene.cpp:91-102
    const double nn = norm(n);
    prims.push_back({2, point, {n.x / nn, n.y / nn, n.z / nn}, 0.0});
  }
  void room_shell(V3 l, V3 h) {  // add_room_shell — scene.cpp:31-41
    for (int axis = 0; axis < 3; ++axis) {
      V3 n{0, 0, 0};
      (axis == 0 ? n.x : axis == 1 ? n.y : n.z) = 1.0;
      plane(l, n);
      plane(h, {-n.x, -n.y, -n.z});
    }
    lo = l;
    hi = h;
  }
  void box(V3 a, V3 b) { prims.push_back({1, a, b, 0.0}); }
  void sphere(V3 c, double r) { prims.push_back({0, c, {0, 0, 0}, r}); }
};

namespace {

// Deterministic, platform-independent generator for the builder scenes.
struct SplitMix {
  uint64_t s;
  uint64_t next() {
    uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  double uni(double a, double b) { return a + (b - a) * double(next() >> 11) * 0x1.0p-53; }
};

constexpr double kPi = 3.14159265358979323846;
constexpr double kHitEpsilon = 1e-4;  // render.cpp:23
constexpr int kMaxSteps = 20000;      // render.cpp:24

// trace — render.cpp:28-39
double trace(const vxm_scene& s, V3 o, V3 d, double t_max) {
  double t = 0.0;
  for (int step = 0; step < kMaxSteps && t <= t_max; ++step) {
    const double dist = s.sdf(add(o, mul(t, d)));
    if (dist < kHitEpsilon) return t;
    t += dist;
  }
  return -1.0;
}

}  // namespace

extern "C" {

vxm_status vxm_synth_scene_create(const char* name_c, vxm_scene** out) {
  const std::string name = name_c ? name_c : "";
  auto* s = new vxm_scene();
  s->name = name;
  if (name == "sphere_in_box") {  // scene.cpp:127-129
    s->room_shell({0, 0, 0}, {3.0, 3.0, 2.5});
    s->sphere({1.5, 1.5, 1.25}, 0.5);
  } else if (name == "room") {  // scene.cpp:130-134
    s->room_shell({0, 0, 0}, {4.0, 3.0, 2.5});
    s->box({1.4, 0.7, 0.0}, {2.0, 1.3, 0.8});
    s->box({2.9, 2.0, 0.0}, {3.2, 2.3, 2.5});
    s->sphere({1.0, 2.2, 0.5}, 0.35);
  } else if (name == "corridor") {  // scene.cpp:135-139
    s->room_shell({0, 0, 0}, {8.0, 2.0, 2.2});
    s->box({2.0, 0.0, 0.0}, {2.6, 0.9, 1.3});
    s->box({4.6, 1.1, 0.0}, {5.2, 2.0, 1.5});
    s->sphere({6.4, 1.0, 0.55}, 0.35);
  } else if (name == "lidar_yard") {
    // C3 (builder-defined; the reference has no 100 m scene): ground plane +
    // 40 boxes 3-15 m wide, 4-20 m tall and 8 spheres in a 200 m x 200 m
    // yard, kept clear of the r = 70 m orbit so the sensor never embeds.
    s->plane({0, 0, 0}, {0, 0, 1});
    SplitMix rng{7};
    int placed = 0;
    while (placed < 40) {
      const double cx = rng.uni(-95, 95), cy = rng.uni(-95, 95);
      const double w = rng.uni(3, 15), d = rng.uni(3, 15), h = rng.uni(4, 20);
      const double rr = std::sqrt(cx * cx + cy * cy);
      if (std::abs(rr - 70.0) < 0.5 * std::max(w, d) + 4.0) continue;
      s->box({cx - 0.5 * w, cy - 0.5 * d, 0.0}, {cx + 0.5 * w, cy + 0.5 * d, h});
      ++placed;
    }
    placed = 0;
    while (placed < 8) {
      const double cx = rng.uni(-90, 90), cy = rng.uni(-90, 90), r = rng.uni(1, 4);
      if (std::abs(std::sqrt(cx * cx + cy * cy) - 70.0) < r + 4.0) continue;
      s->sphere({cx, cy, r}, r);
      ++placed;
    }
    s->lo = {-100, -100, 0};
    s->hi = {100, 100, 3.6};
  } else if (name == "building") {
    // C4 (builder-defined): a 24 m x 16 m x 3 m floor with interior walls
    // (boxes) forming 6 rooms joined by doorways, plus furniture.
    s->room_shell({0, 0, 0}, {24.0, 16.0, 3.0});
    const double t = 0.15;
    for (double x : {8.0, 16.0}) {  // walls along y with doorways
      s->box({x - t, 0.0, 0.0}, {x + t, 3.5, 3.0});
      s->box({x - t, 4.7, 0.0}, {x + t, 11.3, 3.0});
      s->box({x - t, 12.5, 0.0}, {x + t, 16.0, 3.0});
    }
    s->box({0.0, 8.0 - t, 0.0}, {2.5, 8.0 + t, 3.0});  // wall along x
    s->box({3.7, 8.0 - t, 0.0}, {10.5, 8.0 + t, 3.0});
    s->box({11.7, 8.0 - t, 0.0}, {18.5, 8.0 + t, 3.0});
    s->box({19.7, 8.0 - t, 0.0}, {24.0, 8.0 + t, 3.0});
    SplitMix rng{11};
    for (int i = 0; i < 18; ++i) {
      const int room = i % 6;
      const double x0 = 8.0 * (room % 3), y0 = 8.0 * (room / 3);
      const double cx = x0 + rng.uni(1.5, 6.5), cy = y0 + rng.uni(1.5, 6.5);
      if (i % 3 == 2) {
        s->sphere({cx, cy, 0.4}, 0.4);
      } else {
        const double w = rng.uni(0.4, 1.6), d = rng.uni(0.4, 1.2), h = rng.uni(0.5, 1.2);
        s->box({cx - 0.5 * w, cy - 0.5 * d, 0.0}, {cx + 0.5 * w, cy + 0.5 * d, h});
      }
    }
  } else {
    delete s;
    return VXM_ERR_INVALID_ARGUMENT;
  }
  *out = s;
  return VXM_OK;
}

void vxm_synth_scene_destroy(vxm_scene* s) { delete s; }

void vxm_synth_scene_bbox(const vxm_scene* s, double* b) {
  b[0] = s->lo.x; b[1] = s->lo.y; b[2] = s->lo.z;
  b[3] = s->hi.x; b[4] = s->hi.y; b[5] = s->hi.z;
}

double vxm_synth_scene_sdf(const vxm_scene* s, const double p[3]) { return s->sdf({p[0], p[1], p[2]}); }

// orbit_pose — dataset.cpp:334-367
vxm_status vxm_synth_orbit_pose(const vxm_scene* s, int lidar, int frame, int total, vxm_pose* out) {
  if (total < 1) return VXM_ERR_INVALID_ARGUMENT;
  const V3 center = mul(0.5, add(s->lo, s->hi));
  const V3 ext = sub(s->hi, s->lo);
  const double theta = 2.0 * kPi * frame / static_cast<double>(total);
  const V3 t = add(center, {0.35 * ext.x * std::cos(theta), 0.35 * ext.y * std::sin(theta),
                            0.12 * ext.z * std::sin(2.0 * theta)});
  out->t[0] = t.x;
  out->t[1] = t.y;
  out->t[2] = t.z;
  double* R = out->R;
  if (lidar) {
    // AngleAxisd(yaw, UnitZ).toRotationMatrix() (Eigen's formula)
    const double yaw = std::atan2(center.y - t.y, center.x - t.x);
    const double sn = std::sin(yaw), c = std::cos(yaw);
    const V3 axis{0, 0, 1};
    const V3 sin_axis = mul(sn, axis);
    const V3 cos1 = mul(1.0 - c, axis);
    double tmp = cos1.x * axis.y;
    R[1] = tmp - sin_axis.z;
    R[3] = tmp + sin_axis.z;
    tmp = cos1.x * axis.z;
    R[2] = tmp + sin_axis.y;
    R[6] = tmp - sin_axis.y;
    tmp = cos1.y * axis.z;
    R[5] = tmp - sin_axis.x;
    R[7] = tmp + sin_axis.x;
    R[0] = cos1.x * axis.x + c;
    R[4] = cos1.y * axis.y + c;
    R[8] = cos1.z * axis.z + c;
    return VXM_OK;
  }
  const V3 forward = normalized(sub(center, t));
  const V3 up = std::abs(forward.z) > 0.99 ? V3{1, 0, 0} : V3{0, 0, 1};
  const V3 right = normalized(cross(forward, up));
  const V3 down = cross(forward, right);
  R[0] = right.x; R[3] = right.y; R[6] = right.z;
  R[1] = down.x;  R[4] = down.y;  R[7] = down.z;
  R[2] = forward.x; R[5] = forward.y; R[8] = forward.z;
  return VXM_OK;
}

// render_depth (camera) — render.cpp:43-64
vxm_status vxm_synth_render_camera(const vxm_scene* s, const vxm_pose* T, const vxm_camera* cam,
                                   float* out) {
  const int W = cam->width, H = cam->height;
  std::fill(out, out + size_t(W) * H, 0.0f);
  const V3 origin{T->t[0], T->t[1], T->t[2]};
  if (s->sdf(origin) < kHitEpsilon) return VXM_OK;
#pragma omp parallel for schedule(dynamic, 4)
  for (int row = 0; row < H; ++row) {
    for (int col = 0; col < W; ++col) {
      const V3 dir_s = normalized({((col + 0.5) - cam->cu) / cam->fu, ((row + 0.5) - cam->cv) / cam->fv, 1.0});
      const double t_max = cam->max_depth / dir_s.z;
      const double t = trace(*s, origin, rot(T->R, dir_s), t_max);
      if (t >= 0.0) out[size_t(row) * W + col] = static_cast<float>(t * dir_s.z);
    }
  }
  return VXM_OK;
}

// render_depth (lidar) — render.cpp:66-86
vxm_status vxm_synth_render_lidar(const vxm_scene* s, const vxm_pose* T, const vxm_lidar* li,
                                  float* out) {
  const int W = li->num_azimuth, H = li->num_elevation;
  std::fill(out, out + size_t(W) * H, 0.0f);
  const V3 origin{T->t[0], T->t[1], T->t[2]};
  if (s->sdf(origin) < kHitEpsilon) return VXM_OK;
  const double raz = li->azimuth_fov / li->num_azimuth;
  const double rel = li->elevation_fov / li->num_elevation;
#pragma omp parallel for schedule(dynamic, 1)
  for (int row = 0; row < H; ++row) {
    for (int col = 0; col < W; ++col) {
      const double az = li->azimuth_start + (col + 0.5) * raz;
      const double polar = li->elevation_start + (row + 0.5) * rel;
      const double sp = std::sin(polar);
      const V3 dir_s{std::cos(az) * sp, std::sin(az) * sp, std::cos(polar)};
      const double t = trace(*s, origin, rot(T->R, dir_s), li->max_range);
      if (t >= li->min_range) out[size_t(row) * W + col] = static_cast<float>(t);
    }
  }
  return VXM_OK;
}

// SphereWorld dense TSDF — fixtures.hpp:34-98 (add branch of random_edit)
vxm_status vxm_synth_sphere_world(int side, double vs, double trunc, unsigned seed, int n_spheres,
                                  vxm_grid_index* keys, vxm_tsdf_voxel* voxels) {
  if (side <= 0 || side % 8) return VXM_ERR_INVALID_ARGUMENT;
  const double E = side * vs;
  std::mt19937 rng(seed);
  std::uniform_real_distribution<double> pos(0.15 * E, 0.85 * E);
  std::uniform_real_distribution<double> rad(0.08 * E, 0.25 * E);
  struct S {
    V3 c;
    double r;
  };
  std::vector<S> sph;
  for (int i = 0; i < n_spheres; ++i) {
    const double cx = pos(rng), cy = pos(rng), cz = pos(rng);
    sph.push_back({{cx, cy, cz}, rad(rng)});
  }
  const int nb = side / 8;
  const int64_t total = int64_t(nb) * nb * nb;
#pragma omp parallel for schedule(static)
  for (int64_t b = 0; b < total; ++b) {
    // x-slowest block order (sorted GridIndex order)
    const int bx = int(b / (int64_t(nb) * nb)), by = int((b / nb) % nb), bz = int(b % nb);
    if (keys) keys[b] = {bx, by, bz};
    if (!voxels) continue;
    for (int lin = 0; lin < 512; ++lin) {
      const int vx = lin & 7, vy = (lin >> 3) & 7, vz = lin >> 6;
      const V3 c{(double(bx * 8 + vx) + 0.5) * vs, (double(by * 8 + vy) + 0.5) * vs,
                 (double(bz * 8 + vz) + 0.5) * vs};
      double d = 1e9;
      for (const S& s : sph) d = std::min(d, norm(sub(c, s.c)) - s.r);
      vxm_tsdf_voxel& v = voxels[b * 512 + lin];
      v.distance = static_cast<float>(std::clamp(d, -trunc, trunc));
      v.weight = 1.0f;
    }
  }
  return VXM_OK;
}

}  // extern "C"
