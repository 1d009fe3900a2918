// TEST INFRASTRUCTURE ONLY — never linked into or called by the product.
//
// extern "C" driver over the reference's OWN sources (/root/reference/proj/src,
// compiled unmodified with -Dvoxmap=voxmap_ref against oracle/eigen_shim by
// oracle/Makefile into oracle/_ref/libvoxmap_ref.so).  Only tests/, smoke()
// and bench.py's reference/cpu_baseline legs load it, as the checker and as
// the timed CPU baseline ("cpu_baseline.kind": "reference").
//
// It exposes the reference API calls used for parity and timing:
//   integrate_depth            proj/src/integrate/integrator.cpp:162-175
//   reference_integrate_depth  proj/src/reference/reference.cpp:334-354
//   blocks_in_view             proj/src/sensor/view.cpp:61-111
//   update_esdf / mark_sites / clear_invalid / lower_esdf
//                              proj/src/esdf/integrator.cpp:417-572
//   query_batch / reference_query_batch
//                              proj/src/query/query.cpp:147-161, reference.cpp:378-386
//   render_depth / orbit_pose  proj/src/io/render.cpp:43-86, dataset.cpp:309-367
//                              (+ builder scenes from the reference's primitives and the
//                              C5 SphereWorld volume: the reference arm's inputs)
//   brute_force_esdf / compare_esdf / esdf_identical
//                              proj/src/eval/oracle.cpp:26-151
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <random>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "voxmap/core/layer.hpp"
#include "voxmap/core/voxels.hpp"
#include "voxmap/esdf/integrator.hpp"
#include "voxmap/core/serialization.hpp"
#include "voxmap/eval/oracle.hpp"
#include "voxmap/integrate/integrator.hpp"
#include "voxmap/io/dataset.hpp"
#include "voxmap/io/render.hpp"
#include "voxmap/io/scene.hpp"
#include "voxmap/mesh/marching_cubes.hpp"
#include "voxmap/mesh/mesh_layer.hpp"
#include "voxmap/mesh/ply.hpp"
#include "voxmap/query/query.hpp"
#include "voxmap/reference/reference.hpp"
#include "voxmap/sensor/view.hpp"
#include "voxmap_b200.h"

namespace vr = voxmap_ref;

namespace {

thread_local std::string g_err;

struct RefLayer {
  int type;
  vr::Layer<vr::TsdfVoxel>* tsdf = nullptr;
  vr::Layer<vr::EsdfVoxel>* esdf = nullptr;
  vr::Layer<vr::OccupancyVoxel>* occ = nullptr;
  vr::Layer<vr::ColorVoxel>* color = nullptr;
  ~RefLayer() {
    delete tsdf;
    delete esdf;
    delete occ;
    delete color;
  }
};

struct RefState {
  vr::EsdfUpdateState st;
};

template <typename F>
int guard(F&& f) {
  try {
    f();
    return VXM_OK;
  } catch (const vr::InvalidPoseError& e) {
    g_err = e.what();
    return VXM_ERR_INVALID_POSE;
  } catch (const vr::MapCapacityError& e) {
    g_err = e.what();
    return VXM_ERR_CAPACITY;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return VXM_ERR_INVALID_ARGUMENT;
  } catch (const std::exception& e) {
    g_err = e.what();
    return VXM_ERR_INTERNAL;
  }
}

vr::Pose to_pose(const vxm_pose* p) {
  vr::Pose T;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) T.R(r, c) = p->R[r * 3 + c];
  for (int i = 0; i < 3; ++i) T.t[i] = p->t[i];
  return T;
}
void from_pose(const vr::Pose& T, vxm_pose* p) {
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) p->R[r * 3 + c] = T.R(r, c);
  for (int i = 0; i < 3; ++i) p->t[i] = T.t[i];
}
vr::CameraIntrinsics to_cam(const vxm_camera* c) {
  vr::CameraIntrinsics k;
  k.fu = c->fu; k.fv = c->fv; k.cu = c->cu; k.cv = c->cv;
  k.width = c->width; k.height = c->height; k.max_depth = c->max_depth;
  return k;
}
vr::LidarIntrinsics to_lidar(const vxm_lidar* l) {
  vr::LidarIntrinsics k;
  k.num_azimuth = l->num_azimuth; k.num_elevation = l->num_elevation;
  k.azimuth_start = l->azimuth_start; k.elevation_start = l->elevation_start;
  k.azimuth_fov = l->azimuth_fov; k.elevation_fov = l->elevation_fov;
  k.min_range = l->min_range; k.max_range = l->max_range;
  return k;
}
vr::IntegratorConfig to_icfg(const vxm_integrator_config* c) {
  vr::IntegratorConfig k;
  k.truncation = c->truncation;
  k.max_weight = c->max_weight;
  k.weighting = c->weighting == VXM_WEIGHT_INVERSE_SQUARE ? vr::WeightMode::kInverseSquareDepth
                                                          : vr::WeightMode::kConstant;
  k.max_integration_distance = c->max_integration_distance;
  k.camera_sample = c->camera_sample == VXM_SAMPLE_LINEAR
                        ? vr::DepthSampleMode::kLinearForegroundSafe
                        : vr::DepthSampleMode::kNearest;
  k.lidar_sample = c->lidar_sample == VXM_SAMPLE_LINEAR
                       ? vr::DepthSampleMode::kLinearForegroundSafe
                       : vr::DepthSampleMode::kNearest;
  k.max_sample_gap = c->max_sample_gap;
  k.view_pixel_subsample = c->view_pixel_subsample;
  k.hit_log_odds = c->hit_log_odds;
  k.miss_log_odds = c->miss_log_odds;
  k.log_odds_min = c->log_odds_min;
  k.log_odds_max = c->log_odds_max;
  k.parallel = c->parallel != 0;
  return k;
}
vr::EsdfConfig to_ecfg(const vxm_esdf_config* c) {
  vr::EsdfConfig k;
  k.site_threshold = c->site_threshold;
  k.occupied_log_odds_threshold = c->occupied_log_odds_threshold;
  k.max_distance = c->max_distance;
  k.parallel = c->parallel != 0;
  return k;
}
vr::DepthImage to_depth(const float* d, int w, int h) {
  vr::DepthImage img(w, h);
  std::memcpy(img.data.data(), d, sizeof(float) * size_t(w) * h);
  return img;
}
void emit(const std::vector<vr::GridIndex>& v, vxm_grid_index** out, uint64_t* n) {
  *n = v.size();
  *out = static_cast<vxm_grid_index*>(std::malloc(sizeof(vxm_grid_index) * (v.size() + 1)));
  for (size_t i = 0; i < v.size(); ++i) (*out)[i] = {v[i].x, v[i].y, v[i].z};
}
std::vector<vr::GridIndex> to_list(const vxm_grid_index* k, uint64_t n) {
  std::vector<vr::GridIndex> v(n);
  for (uint64_t i = 0; i < n; ++i) v[i] = {k[i].x, k[i].y, k[i].z};
  return v;
}

template <typename V>
void export_layer(const vr::Layer<V>& L, vxm_grid_index* keys, void* voxels) {
  const auto idx = L.sorted_indices();
  for (size_t i = 0; i < idx.size(); ++i) {
    keys[i] = {idx[i].x, idx[i].y, idx[i].z};
    if (voxels)
      std::memcpy(static_cast<char*>(voxels) + i * sizeof(V) * vr::kVoxelsPerBlock,
                  L.block_ptr(idx[i])->voxels.data(), sizeof(V) * vr::kVoxelsPerBlock);
  }
}

}  // namespace

extern "C" {

const char* vxr_last_error() { return g_err.c_str(); }
void vxr_free(void* p) { std::free(p); }

int vxr_layer_create(int type, double vs, uint64_t max_blocks, void** out) {
  return guard([&] {
    auto* L = new RefLayer{type};
    const size_t mb = max_blocks ? size_t(max_blocks) : size_t{1} << 30;
    try {
      if (type == VXM_LAYER_TSDF) L->tsdf = new vr::Layer<vr::TsdfVoxel>(vs, mb);
      else if (type == VXM_LAYER_OCCUPANCY) L->occ = new vr::Layer<vr::OccupancyVoxel>(vs, mb);
      else if (type == VXM_LAYER_COLOR) L->color = new vr::Layer<vr::ColorVoxel>(vs, mb);
      else L->esdf = new vr::Layer<vr::EsdfVoxel>(vs, mb);
    } catch (...) {
      delete L;
      throw;
    }
    *out = L;
  });
}
void vxr_layer_destroy(void* h) { delete static_cast<RefLayer*>(h); }
uint64_t vxr_layer_num_blocks(void* h) {
  auto* L = static_cast<RefLayer*>(h);
  return L->tsdf    ? L->tsdf->num_blocks()
         : L->occ   ? L->occ->num_blocks()
         : L->color ? L->color->num_blocks()
                    : L->esdf->num_blocks();
}
int vxr_layer_export(void* h, vxm_grid_index* keys, void* voxels) {
  return guard([&] {
    auto* L = static_cast<RefLayer*>(h);
    if (L->tsdf) export_layer(*L->tsdf, keys, voxels);
    else if (L->occ) export_layer(*L->occ, keys, voxels);
    else if (L->color) export_layer(*L->color, keys, voxels);
    else export_layer(*L->esdf, keys, voxels);
  });
}
int vxr_layer_write_blocks(void* h, const vxm_grid_index* keys, uint64_t n, const void* voxels) {
  return guard([&] {
    auto* L = static_cast<RefLayer*>(h);
    for (uint64_t i = 0; i < n; ++i) {
      const vr::GridIndex g{keys[i].x, keys[i].y, keys[i].z};
      if (L->tsdf)
        std::memcpy(L->tsdf->get_or_allocate(g).voxels.data(),
                    static_cast<const char*>(voxels) + i * 4096, 4096);
      else if (L->occ)
        std::memcpy(L->occ->get_or_allocate(g).voxels.data(),
                    static_cast<const char*>(voxels) + i * 2048, 2048);
      else if (L->color)
        std::memcpy(L->color->get_or_allocate(g).voxels.data(),
                    static_cast<const char*>(voxels) + i * 4096, 4096);
      else
        std::memcpy(L->esdf->get_or_allocate(g).voxels.data(),
                    static_cast<const char*>(voxels) + i * 6144, 6144);
    }
  });
}

int vxr_blocks_in_view_camera(const vxm_pose* T, const vxm_camera* cam, const float* depth, int w,
                              int h, double block_size, const vxm_view_config* vc,
                              vxm_grid_index** out, uint64_t* n) {
  return guard([&] {
    const vr::ViewConfig cfg{vc->max_integration_distance, vc->truncation, vc->pixel_subsample};
    emit(vr::blocks_in_view(to_pose(T), to_cam(cam), to_depth(depth, w, h), block_size, cfg), out,
         n);
  });
}
int vxr_blocks_in_view_lidar(const vxm_pose* T, const vxm_lidar* li, const float* depth, int w,
                             int h, double block_size, const vxm_view_config* vc,
                             vxm_grid_index** out, uint64_t* n) {
  return guard([&] {
    const vr::ViewConfig cfg{vc->max_integration_distance, vc->truncation, vc->pixel_subsample};
    emit(vr::blocks_in_view(to_pose(T), to_lidar(li), to_depth(depth, w, h), block_size, cfg), out,
         n);
  });
}

// serial != 0 selects the serial restatement reference_integrate_depth.
int vxr_integrate_camera(void* h, const float* depth, int w, int hh, const vxm_pose* T,
                         const vxm_camera* cam, const vxm_integrator_config* c, int serial,
                         vxm_grid_index** out, uint64_t* n) {
  return guard([&] {
    auto* L = static_cast<RefLayer*>(h);
    const auto img = to_depth(depth, w, hh);
    if (L->occ)  // Layer<OccupancyVoxel> overload (integrator.cpp:176-182)
      emit(serial ? vr::reference_integrate_depth(*L->occ, img, to_pose(T), to_cam(cam), to_icfg(c))
                  : vr::integrate_depth(*L->occ, img, to_pose(T), to_cam(cam), to_icfg(c)),
           out, n);
    else
      emit(serial ? vr::reference_integrate_depth(*L->tsdf, img, to_pose(T), to_cam(cam), to_icfg(c))
                  : vr::integrate_depth(*L->tsdf, img, to_pose(T), to_cam(cam), to_icfg(c)),
           out, n);
  });
}
int vxr_integrate_lidar(void* h, const float* depth, int w, int hh, const vxm_pose* T,
                        const vxm_lidar* li, const vxm_integrator_config* c, int serial,
                        vxm_grid_index** out, uint64_t* n) {
  return guard([&] {
    auto* L = static_cast<RefLayer*>(h);
    const auto img = to_depth(depth, w, hh);
    if (L->occ)  // integrator.cpp:183-189
      emit(serial
               ? vr::reference_integrate_depth(*L->occ, img, to_pose(T), to_lidar(li), to_icfg(c))
               : vr::integrate_depth(*L->occ, img, to_pose(T), to_lidar(li), to_icfg(c)),
           out, n);
    else
      emit(serial
               ? vr::reference_integrate_depth(*L->tsdf, img, to_pose(T), to_lidar(li), to_icfg(c))
               : vr::integrate_depth(*L->tsdf, img, to_pose(T), to_lidar(li), to_icfg(c)),
           out, n);
  });
}

int vxr_update_esdf(void* esdf, void* tsdf, const vxm_grid_index* upd, uint64_t nu,
                    const vxm_esdf_config* c, vxm_grid_index** out, uint64_t* n) {
  return guard([&] {
    auto* E = static_cast<RefLayer*>(esdf);
    auto* T = static_cast<RefLayer*>(tsdf);
    if (T->occ)  // Layer<OccupancyVoxel> overload (esdf/integrator.cpp:574-579)
      emit(vr::update_esdf(*E->esdf, *T->occ, to_list(upd, nu), to_ecfg(c)), out, n);
    else
      emit(vr::update_esdf(*E->esdf, *T->tsdf, to_list(upd, nu), to_ecfg(c)), out, n);
  });
}

void* vxr_state_create() { return new RefState; }
void vxr_state_destroy(void* s) { delete static_cast<RefState*>(s); }
int vxr_state_get(void* s, int which, vxm_grid_index** out, uint64_t* n) {
  return guard([&] {
    auto& st = static_cast<RefState*>(s)->st;
    emit(which == 0 ? st.indices_to_update
                    : which == 1 ? st.indices_to_clear : st.cleared_indices,
         out, n);
  });
}
int vxr_state_set(void* s, int which, const vxm_grid_index* k, uint64_t n) {
  return guard([&] {
    auto& st = static_cast<RefState*>(s)->st;
    (which == 0 ? st.indices_to_update
                : which == 1 ? st.indices_to_clear : st.cleared_indices) = to_list(k, n);
  });
}
int vxr_mark_sites(void* esdf, void* tsdf, const vxm_grid_index* upd, uint64_t nu,
                   const vxm_esdf_config* c, void* s, vxm_grid_index** out, uint64_t* n) {
  return guard([&] {
    std::vector<vr::GridIndex> changed;
    auto* T = static_cast<RefLayer*>(tsdf);
    if (T->occ)
      vr::mark_sites(*static_cast<RefLayer*>(esdf)->esdf, *T->occ, to_list(upd, nu), to_ecfg(c),
                     &static_cast<RefState*>(s)->st, &changed);
    else
      vr::mark_sites(*static_cast<RefLayer*>(esdf)->esdf, *T->tsdf, to_list(upd, nu), to_ecfg(c),
                     &static_cast<RefState*>(s)->st, &changed);
    emit(changed, out, n);
  });
}
int vxr_clear_invalid(void* esdf, const vxm_esdf_config* c, void* s, vxm_grid_index** out,
                      uint64_t* n) {
  return guard([&] {
    std::vector<vr::GridIndex> changed;
    vr::clear_invalid(*static_cast<RefLayer*>(esdf)->esdf, to_ecfg(c),
                      &static_cast<RefState*>(s)->st, &changed);
    emit(changed, out, n);
  });
}
int vxr_lower_esdf(void* esdf, void* s, const vxm_esdf_config* c, int* rounds,
                   vxm_grid_index** out, uint64_t* n) {
  return guard([&] {
    std::vector<vr::GridIndex> changed;
    *rounds = vr::lower_esdf(*static_cast<RefLayer*>(esdf)->esdf, static_cast<RefState*>(s)->st,
                             to_ecfg(c), &changed);
    emit(changed, out, n);
  });
}

int vxr_query_batch(void* esdf, const double* xyz, uint64_t n, int want_gradient,
                    const vxm_query_config* qc, int serial, vxm_query_result* out) {
  return guard([&] {
    std::vector<Eigen::Vector3d> pts(n);
    for (uint64_t i = 0; i < n; ++i) pts[i] = Eigen::Vector3d(xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2]);
    vr::QueryConfig cfg;
    cfg.interpolate = qc->interpolate != 0;
    cfg.parallel = qc->parallel != 0;
    const auto& E = *static_cast<RefLayer*>(esdf)->esdf;
    const auto res = serial ? vr::reference_query_batch(E, pts, want_gradient != 0, cfg)
                            : vr::query_batch(E, pts, want_gradient != 0, cfg);
    for (uint64_t i = 0; i < n; ++i) {
      out[i].known = res[i].known;
      out[i].pad_ = 0;
      out[i].distance = res[i].distance;
      for (int a = 0; a < 3; ++a) out[i].gradient[a] = res[i].gradient[a];
    }
  });
}

// Scenes / rendering / trajectories (input generators of the reference).
}  // extern "C"

namespace {

// Deterministic generator of the builder scenes (same stream as
// paper_2311_00626_b200/csrc/synth.cpp; tests pin the rendered frames equal).
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

// add_room_shell (scene.cpp:31-41 is file-local, restated with the public make_plane)
void room_shell(vr::SyntheticScene& sc, const Eigen::Vector3d& lo, const Eigen::Vector3d& hi) {
  for (int axis = 0; axis < 3; ++axis) {
    Eigen::Vector3d n = Eigen::Vector3d::Zero();
    n[axis] = 1.0;
    sc.primitives.push_back(vr::make_plane(lo, n));
    sc.primitives.push_back(vr::make_plane(hi, -n));
  }
  sc.bbox_min = lo;
  sc.bbox_max = hi;
}

// make_scene (scene.cpp:124-144) plus the builder scenes of configs the
// reference has no scene for, assembled from the reference's own primitives
// (make_box / make_sphere / make_plane, scene.cpp:56-102): "lidar_yard" (C3)
// and "building" (C4).
vr::SyntheticScene ref_scene(const std::string& name) {
  if (name == "lidar_yard") {
    vr::SyntheticScene sc;
    sc.name = name;
    sc.primitives.push_back(vr::make_plane({0, 0, 0}, {0, 0, 1}));
    SplitMix rng{7};
    int placed = 0;
    while (placed < 40) {
      const double cx = rng.uni(-95, 95), cy = rng.uni(-95, 95);
      const double w = rng.uni(3, 15), d = rng.uni(3, 15), h = rng.uni(4, 20);
      const double rr = std::sqrt(cx * cx + cy * cy);
      if (std::abs(rr - 70.0) < 0.5 * std::max(w, d) + 4.0) continue;
      sc.primitives.push_back(vr::make_box({cx - 0.5 * w, cy - 0.5 * d, 0.0}, {cx + 0.5 * w, cy + 0.5 * d, h}));
      ++placed;
    }
    placed = 0;
    while (placed < 8) {
      const double cx = rng.uni(-90, 90), cy = rng.uni(-90, 90), r = rng.uni(1, 4);
      if (std::abs(std::sqrt(cx * cx + cy * cy) - 70.0) < r + 4.0) continue;
      sc.primitives.push_back(vr::make_sphere({cx, cy, r}, r));
      ++placed;
    }
    sc.bbox_min = {-100, -100, 0};
    sc.bbox_max = {100, 100, 3.6};
    return sc;
  }
  if (name == "building") {
    vr::SyntheticScene sc;
    sc.name = name;
    room_shell(sc, {0, 0, 0}, {24.0, 16.0, 3.0});
    const double t = 0.15;
    for (double x : {8.0, 16.0}) {
      sc.primitives.push_back(vr::make_box({x - t, 0.0, 0.0}, {x + t, 3.5, 3.0}));
      sc.primitives.push_back(vr::make_box({x - t, 4.7, 0.0}, {x + t, 11.3, 3.0}));
      sc.primitives.push_back(vr::make_box({x - t, 12.5, 0.0}, {x + t, 16.0, 3.0}));
    }
    sc.primitives.push_back(vr::make_box({0.0, 8.0 - t, 0.0}, {2.5, 8.0 + t, 3.0}));
    sc.primitives.push_back(vr::make_box({3.7, 8.0 - t, 0.0}, {10.5, 8.0 + t, 3.0}));
    sc.primitives.push_back(vr::make_box({11.7, 8.0 - t, 0.0}, {18.5, 8.0 + t, 3.0}));
    sc.primitives.push_back(vr::make_box({19.7, 8.0 - t, 0.0}, {24.0, 8.0 + t, 3.0}));
    SplitMix rng{11};
    for (int i = 0; i < 18; ++i) {
      const int room = i % 6;
      const double x0 = 8.0 * (room % 3), y0 = 8.0 * (room / 3);
      const double cx = x0 + rng.uni(1.5, 6.5), cy = y0 + rng.uni(1.5, 6.5);
      if (i % 3 == 2) {
        sc.primitives.push_back(vr::make_sphere({cx, cy, 0.4}, 0.4));
      } else {
        const double w = rng.uni(0.4, 1.6), d = rng.uni(0.4, 1.2), h = rng.uni(0.5, 1.2);
        sc.primitives.push_back(vr::make_box({cx - 0.5 * w, cy - 0.5 * d, 0.0}, {cx + 0.5 * w, cy + 0.5 * d, h}));
      }
    }
    return sc;
  }
  return vr::make_scene(name);
}

}  // namespace

extern "C" {

int vxr_orbit_pose(const char* scene, int lidar, int k, int total, vxm_pose* out) {
  return guard([&] {
    const auto sc = ref_scene(scene);
    from_pose(vr::orbit_pose(sc, lidar ? vr::SensorKind::kLidar : vr::SensorKind::kCamera, k, total),
              out);
  });
}
int vxr_render_depth_camera(const char* scene, const vxm_pose* T, const vxm_camera* cam,
                            float* out) {
  return guard([&] {
    const auto img = vr::render_depth(ref_scene(scene), to_pose(T), to_cam(cam));
    std::memcpy(out, img.data.data(), sizeof(float) * img.data.size());
  });
}
int vxr_render_depth_lidar(const char* scene, const vxm_pose* T, const vxm_lidar* li, float* out) {
  return guard([&] {
    const auto img = vr::render_depth(ref_scene(scene), to_pose(T), to_lidar(li));
    std::memcpy(out, img.data.data(), sizeof(float) * img.data.size());
  });
}
// SphereWorld-style dense TSDF of config C5 (tests/fixtures.hpp:34-98, the
// add branch of random_edit): n spheres from std::mt19937(seed), distance =
// float(clamp(min_i(|c - c_i| - r_i), +-trunc)) at each voxel centre
// (indexing.hpp:113-119), weight 1; blocks in sorted (x-slowest) order.
int vxr_sphere_world(int side, double vs, double trunc, unsigned seed, int n_spheres,
                     vxm_grid_index* keys, vxm_tsdf_voxel* voxels) {
  return guard([&] {
    if (side <= 0 || side % 8) throw std::invalid_argument("sphere_world: side must be a multiple of 8");
    const double E = side * vs;
    std::mt19937 rng(seed);
    std::uniform_real_distribution<double> pos(0.15 * E, 0.85 * E);
    std::uniform_real_distribution<double> rad(0.08 * E, 0.25 * E);
    std::vector<std::pair<Eigen::Vector3d, double>> sph;
    for (int i = 0; i < n_spheres; ++i) {
      const double cx = pos(rng), cy = pos(rng), cz = pos(rng);
      sph.push_back({Eigen::Vector3d(cx, cy, cz), rad(rng)});
    }
    const int nb = side / 8;
    const int64_t total = int64_t(nb) * nb * nb;
#pragma omp parallel for schedule(static)
    for (int64_t b = 0; b < total; ++b) {
      const vr::GridIndex g{int(b / (int64_t(nb) * nb)), int((b / nb) % nb), int(b % nb)};
      if (keys) keys[b] = {g.x, g.y, g.z};
      if (!voxels) continue;
      for (int lin = 0; lin < 512; ++lin) {
        const Eigen::Vector3d c = vr::voxel_center(g, vr::voxel_index_from_linear(lin), vs);
        double d = 1e9;
        for (const auto& s : sph) d = std::min(d, (c - s.first).norm() - s.second);
        voxels[b * 512 + lin].distance = static_cast<float>(std::clamp(d, -trunc, trunc));
        voxels[b * 512 + lin].weight = 1.0f;
      }
    }
  });
}
void vxr_default_camera(int w, int h, vxm_camera* out) {
  const auto c = vr::default_camera_intrinsics(w, h);
  *out = {c.fu, c.fv, c.cu, c.cv, c.width, c.height, c.max_depth};
}
void vxr_default_lidar(int na, int ne, vxm_lidar* out) {
  const auto l = vr::default_lidar_intrinsics(na, ne);
  *out = {l.num_azimuth, l.num_elevation, l.azimuth_start, l.elevation_start,
          l.azimuth_fov,  l.elevation_fov, l.min_range,     l.max_range};
}
int vxr_pose_valid(const vxm_pose* T) { return to_pose(T).valid() ? 1 : 0; }
void vxr_pose_inverse(const vxm_pose* T, vxm_pose* out) { from_pose(to_pose(T).inverse(), out); }

// ESDF oracle utilities.
int vxr_brute_force_esdf(void* esdf, const vxm_esdf_config* c, void** out) {
  return guard([&] {
    auto* L = new RefLayer{VXM_LAYER_ESDF};
    try {
      L->esdf = new vr::Layer<vr::EsdfVoxel>(
          vr::brute_force_esdf(*static_cast<RefLayer*>(esdf)->esdf, to_ecfg(c)));
    } catch (...) {
      delete L;
      throw;
    }
    *out = L;
  });
}
// stats: compared, exact, within_one_voxel, flag_mismatches (uint64) + max_abs_error (double)
int vxr_compare_esdf(void* a, void* b, uint64_t* stats4, double* max_abs) {
  return guard([&] {
    const auto cmp = vr::compare_esdf(*static_cast<RefLayer*>(a)->esdf,
                                      *static_cast<RefLayer*>(b)->esdf);
    stats4[0] = cmp.compared;
    stats4[1] = cmp.exact;
    stats4[2] = cmp.within_one_voxel;
    stats4[3] = cmp.flag_mismatches;
    *max_abs = cmp.max_abs_error;
  });
}

// save_snapshot / load_snapshot (core/serialization.cpp:88-158) on a cake
// that borrows the driver's layers.
int vxr_snapshot_save(const char* path, double vs, void* tsdf, void* occ, void* color, void* esdf) {
  return guard([&] {
    vr::LayerCake cake(vs);
    if (tsdf) cake.tsdf.reset(static_cast<RefLayer*>(tsdf)->tsdf);
    if (occ) cake.occupancy.reset(static_cast<RefLayer*>(occ)->occ);
    if (color) cake.color.reset(static_cast<RefLayer*>(color)->color);
    if (esdf) cake.esdf.reset(static_cast<RefLayer*>(esdf)->esdf);
    const auto release = [&] {
      cake.tsdf.release();
      cake.occupancy.release();
      cake.color.release();
      cake.esdf.release();
    };
    try {
      vr::save_snapshot(cake, path);
    } catch (...) {
      release();
      throw;
    }
    release();
  });
}
int vxr_snapshot_load(const char* path, double* vs, void** tsdf, void** occ, void** color,
                      void** esdf) {
  return guard([&] {
    vr::LayerCake cake = vr::load_snapshot(path);
    *vs = cake.voxel_size;
    *tsdf = *occ = *color = *esdf = nullptr;
    if (cake.color) {
      auto* L = new RefLayer{VXM_LAYER_COLOR};
      L->color = cake.color.release();
      *color = L;
    }
    if (cake.tsdf) *tsdf = new RefLayer{VXM_LAYER_TSDF, cake.tsdf.release(), nullptr};
    if (cake.occupancy) {
      auto* L = new RefLayer{VXM_LAYER_OCCUPANCY};
      L->occ = cake.occupancy.release();
      *occ = L;
    }
    if (cake.esdf) *esdf = new RefLayer{VXM_LAYER_ESDF, nullptr, cake.esdf.release()};
  });
}

// ---- color + meshing (integrator.cpp:191-273, marching_cubes.cpp:95-242, ply.cpp) ----
vr::ColorImage to_color(const uint8_t* rgb, int w, int h) {
  vr::ColorImage img(w, h);
  std::memcpy(img.data.data(), rgb, size_t(w) * h * 3);
  return img;
}
int vxr_integrate_color(void* color, const uint8_t* rgb, int w, int h, const float* depth,
                        const vxm_pose* T, const vxm_camera* cam, void* tsdf,
                        const vxm_integrator_config* c, vxm_grid_index** out, uint64_t* n) {
  return guard([&] {
    emit(vr::integrate_color(*static_cast<RefLayer*>(color)->color, to_color(rgb, w, h),
                             to_depth(depth, w, h), to_pose(T), to_cam(cam),
                             *static_cast<RefLayer*>(tsdf)->tsdf, to_icfg(c)),
         out, n);
  });
}
int vxr_render_color_camera(const char* scene, const vxm_pose* T, const vxm_camera* cam, uint8_t* out) {
  return guard([&] {
    const auto img = vr::render_color(vr::make_scene(scene), to_pose(T), to_cam(cam));
    std::memcpy(out, img.data.data(), img.data.size() * 3);
  });
}
const int8_t* vxr_mc_tri_table() { return &vr::mc::kTriTable[0][0]; }

void* vxr_mesh_create(double vs) { return new vr::MeshLayer(vs); }
void vxr_mesh_destroy(void* m) { delete static_cast<vr::MeshLayer*>(m); }
uint64_t vxr_mesh_num_blocks(void* m) { return static_cast<vr::MeshLayer*>(m)->num_blocks(); }
void vxr_mesh_keys(void* m, vxm_grid_index* keys) {
  const auto idx = static_cast<vr::MeshLayer*>(m)->sorted_indices();
  for (size_t i = 0; i < idx.size(); ++i) keys[i] = {idx[i].x, idx[i].y, idx[i].z};
}
// Pointers into the MeshBlock's arrays (valid until the block is re-meshed).
int vxr_mesh_block_get(void* m, const vxm_grid_index* g, uint64_t* nv, uint64_t* nt,
                       const float** verts, const float** normals, const uint8_t** colors,
                       uint64_t* ncolors, const uint32_t** tris) {
  return guard([&] {
    const vr::MeshBlock* b = static_cast<vr::MeshLayer*>(m)->block_ptr({g->x, g->y, g->z});
    if (!b) throw std::invalid_argument("mesh block not present");
    static_assert(sizeof(Eigen::Vector3f) == 12 && sizeof(std::array<uint32_t, 3>) == 12);
    *nv = b->vertices.size();
    *nt = b->triangles.size();
    *ncolors = b->colors.size();
    *verts = b->vertices.empty() ? nullptr : b->vertices[0].data();
    *normals = b->normals.empty() ? nullptr : b->normals[0].data();
    *colors = b->colors.empty() ? nullptr : b->colors[0].data();
    *tris = b->triangles.empty() ? nullptr : b->triangles[0].data();
  });
}
int vxr_update_mesh(void* m, void* tsdf, const vxm_grid_index* upd, uint64_t nu, float min_weight,
                    void* color, vxm_grid_index** out, uint64_t* n) {
  return guard([&] {
    vr::MeshConfig cfg;
    cfg.min_weight = min_weight;
    emit(vr::update_mesh(*static_cast<vr::MeshLayer*>(m), *static_cast<RefLayer*>(tsdf)->tsdf,
                         to_list(upd, nu), cfg,
                         color ? static_cast<RefLayer*>(color)->color : nullptr),
         out, n);
  });
}
int vxr_mesh_block(void* m, void* tsdf, const vxm_grid_index* g, float min_weight, void* color) {
  return guard([&] {
    vr::MeshConfig cfg;
    cfg.min_weight = min_weight;
    const vr::GridIndex k{g->x, g->y, g->z};
    static_cast<vr::MeshLayer*>(m)->get_or_create(k) = vr::mesh_block(
        *static_cast<RefLayer*>(tsdf)->tsdf, k, cfg,
        color ? static_cast<RefLayer*>(color)->color : nullptr);
  });
}
int vxr_save_mesh_ply(void* m, const char* path) {
  return guard([&] { vr::save_mesh_ply(*static_cast<vr::MeshLayer*>(m), path); });
}

}  // extern "C"
