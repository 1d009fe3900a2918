// C++ facade parity test (GPU): the reference's C++ API shape through
// include/voxmap_b200/voxmap.hpp, checked bit-for-bit against the C oracle
// (oracle/voxmap_oracle.c).  Mirrors proj/tests/integrate_test.cpp:225-363 and
// esdf_test.cpp:232-269, 377-398.  Exit code 0 = pass.
#include <cstdio>
#include <cstring>
#include <vector>

#include "voxmap_b200/voxmap.hpp"
#include "voxmap_b200_synth.h"
#include "voxmap_oracle.h"

namespace vb = voxmap_b200;

static int failures = 0;
#define CHECK(cond)                                                      \
  do {                                                                   \
    if (!(cond)) {                                                       \
      std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      ++failures;                                                        \
    }                                                                    \
  } while (0)

static vb::Pose pose_of(const vxm_pose& p) {
  vb::Pose T;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) T.R(r, c) = p.R[3 * r + c];
  T.t = {p.t[0], p.t[1], p.t[2]};
  return T;
}

static std::vector<vb::GridIndex> oracle_list(vxm_grid_index* p, uint64_t n) {
  std::vector<vb::GridIndex> v = vb::from_c(p, n);
  vxo_free(p);
  return v;
}

template <typename V>
static bool same_layer(const vb::Layer<V>& g, const vxo_layer* o) {
  const auto keys = g.sorted_indices();
  const uint64_t n = vxo_layer_num_blocks(o);
  if (keys.size() != n) return false;
  std::vector<vxm_grid_index> ok(n);
  std::vector<V> ov(n * 512);
  vxo_layer_export(o, ok.data(), ov.data());
  for (uint64_t i = 0; i < n; ++i) {
    if (keys[i].x != ok[i].x || keys[i].y != ok[i].y || keys[i].z != ok[i].z) return false;
    const auto* b = g.block_ptr(keys[i]);
    if (!b || std::memcmp(b->voxels.data(), ov.data() + i * 512, sizeof(V) * 512) != 0) return false;
  }
  return true;
}

// Index algebra KATs — core_test.cpp:30-71 (host inline, no device).
static void index_kats() {
  const double vs = 0.05;
  vb::GridIndex g;
  vb::VoxelIndex v;
  vb::position_to_indices({0.0, 0.0, 0.0}, vs, &g, &v);
  CHECK((g == vb::GridIndex{0, 0, 0}) && (v == vb::VoxelIndex{0, 0, 0}));
  vb::position_to_indices({-0.01, 0.0, 0.0}, vs, &g, &v);
  CHECK((g == vb::GridIndex{-1, 0, 0}) && (v == vb::VoxelIndex{7, 0, 0}));
  vb::position_to_indices({0.43, 0.05, -0.40}, vs, &g, &v);
  CHECK((g == vb::GridIndex{1, 0, -1}) && (v == vb::VoxelIndex{0, 1, 0}));
  const vb::Vec3 c0 = vb::voxel_center({0, 0, 0}, {0, 0, 0}, vs);
  CHECK(c0.x == 0.025 && c0.y == 0.025 && c0.z == 0.025);
  const vb::Vec3 cn = vb::voxel_center({-1, 0, 0}, {7, 0, 0}, vs);
  CHECK(cn.x == -0.025 && cn.y == 0.025 && cn.z == 0.025);
  unsigned st = 7;
  auto rnd = [&st](int lo, int hi) {
    st = st * 1103515245u + 12345u;
    return lo + int((st >> 8) % unsigned(hi - lo + 1));
  };
  for (int i = 0; i < 1000; ++i) {
    const vb::GridIndex gg{rnd(-50, 50), rnd(-50, 50), rnd(-50, 50)};
    const vb::VoxelIndex vv{rnd(0, 7), rnd(0, 7), rnd(0, 7)};
    vb::position_to_indices(vb::voxel_center(gg, vv, vs), vs, &g, &v);
    CHECK(g == gg && v == vv);
    CHECK(vb::voxel_index_from_linear(vb::linear_voxel_index(vv)) == vv);
    CHECK(vb::local_voxel_of_global(vb::global_voxel_index(gg, vv)) == vv);
    CHECK(vb::block_of_global_voxel(vb::global_voxel_index(gg, vv)) == gg);
  }
}

int main() {
  index_kats();
  vxm_scene* scene = nullptr;
  vxm_synth_scene_create("sphere_in_box", &scene);
  vb::CameraIntrinsics cam;
  cam.width = 160;
  cam.height = 120;
  cam.fu = cam.fv = cam.cu = 80.0;
  cam.cv = 60.0;
  cam.max_depth = 10.0;
  const vxm_camera cam_c = cam.c();
  vb::IntegratorConfig cfg;
  cfg.truncation = 0.2;
  const vxm_integrator_config cfg_c = cfg.c();
  vb::EsdfConfig ecfg;
  ecfg.site_threshold = 0.05;
  const vxm_esdf_config ecfg_c = ecfg.c();

  vb::Layer<vb::TsdfVoxel> tsdf(0.05);
  vb::Layer<vb::EsdfVoxel> esdf(0.05);
  vxo_layer *otsdf = nullptr, *oesdf = nullptr;
  vxo_layer_create(VXM_LAYER_TSDF, 0.05, 0, &otsdf);
  vxo_layer_create(VXM_LAYER_ESDF, 0.05, 0, &oesdf);

  for (int k = 0; k < 3; ++k) {  // integrate_test.cpp:243-261 shape
    vxm_pose p;
    vxm_synth_orbit_pose(scene, 0, k, 8, &p);
    vb::DepthImage depth(cam.width, cam.height);
    vxm_synth_render_camera(scene, &p, &cam_c, depth.data.data());
    const auto a = vb::integrate_depth(tsdf, depth, pose_of(p), cam, cfg);
    vxm_grid_index* ob = nullptr;
    uint64_t on = 0;
    vxo_integrate_camera(otsdf, depth.data.data(), depth.width, depth.height, &p, &cam_c, &cfg_c, &ob, &on);
    const auto b = oracle_list(ob, on);
    CHECK(!a.empty());
    CHECK(a == b);
    const auto ea = vb::update_esdf(esdf, tsdf, a, ecfg);
    const auto bc = vb::to_c(b);
    vxo_update_esdf(oesdf, otsdf, bc.data(), bc.size(), &ecfg_c, &ob, &on);
    CHECK(ea == oracle_list(ob, on));
  }
  CHECK(same_layer(tsdf, otsdf));
  CHECK(same_layer(esdf, oesdf));

  // Host writes through block_ptr() are seen by the next device operation
  // (Layer handles stay valid, layer.hpp:44-46).
  {
    const auto keys = tsdf.sorted_indices();
    auto* blk = tsdf.block_ptr(keys.front());
    CHECK(blk != nullptr);
    blk->voxels[0].distance = 0.0f;
    blk->voxels[0].weight = 1.0f;
    CHECK(tsdf.block_ptr(keys.front())->voxels[0].weight == 1.0f);
    const vb::Layer<vb::TsdfVoxel> copy = tsdf.clone();
    CHECK(copy.block_ptr(keys.front())->voxels[0].weight == 1.0f);
  }

  // Errors map onto the reference's exception types (integrate_test.cpp:447-488).
  {
    vb::Layer<vb::TsdfVoxel> layer(0.05);
    vb::DepthImage wrong(32, 48);
    vb::CameraIntrinsics c64 = cam;
    c64.width = 64;
    c64.height = 48;
    bool threw = false;
    try {
      vb::integrate_depth(layer, wrong, vb::Pose::identity(), c64, cfg);
    } catch (const std::invalid_argument&) {
      threw = true;
    }
    CHECK(threw);
    vb::Pose bad;
    bad.R(0, 0) = 2.0;
    threw = false;
    try {
      vb::DepthImage d(64, 48);
      vb::integrate_depth(layer, d, bad, c64, cfg);
    } catch (const vb::InvalidPoseError&) {
      threw = true;
    }
    CHECK(threw);
    CHECK(layer.num_blocks() == 0);
  }

  // Queries (query.cpp production order) — bitwise vs the oracle.
  {
    std::vector<vb::Vec3> pts;
    std::vector<double> flat;
    for (int i = 0; i < 500; ++i) {
      const vb::Vec3 q{0.1 + 0.0057 * i, 0.3 + 0.0041 * i, 0.2 + 0.0033 * i};
      pts.push_back(q);
      flat.insert(flat.end(), {q.x, q.y, q.z});
    }
    vb::QueryConfig qc;
    const auto got = vb::query_batch(esdf, pts, true, qc);
    std::vector<vxm_query_result> want(pts.size());
    const vxm_query_config qcc{1, 1};
    vxo_query_batch(oesdf, flat.data(), pts.size(), 1, &qcc, want.data());
    int known = 0;
    for (size_t i = 0; i < pts.size(); ++i) {
      CHECK(got[i].known == (want[i].known != 0));
      CHECK(got[i].distance == want[i].distance);
      CHECK(got[i].gradient.x == want[i].gradient[0] && got[i].gradient.y == want[i].gradient[1] &&
            got[i].gradient.z == want[i].gradient[2]);
      known += got[i].known;
    }
    CHECK(known > 50);
  }

  // snapshots (core/serialization.hpp:29-35): save -> load round trip
  {
    const std::string path = "/tmp/vxm_facade_test.vxlf";
    vb::LayerCake cake(tsdf.voxel_size());
    cake.tsdf = std::make_unique<vb::Layer<vb::TsdfVoxel>>(tsdf.clone());
    cake.esdf = std::make_unique<vb::Layer<vb::EsdfVoxel>>(esdf.clone());
    vb::save_snapshot(cake, path);
    vb::LayerCake back = vb::load_snapshot(path);
    CHECK(back.voxel_size == tsdf.voxel_size());
    CHECK(back.tsdf && back.esdf);
    auto same = [](const auto& a, const auto& b) {
      const auto ka = a.sorted_indices(), kb = b.sorted_indices();
      if (ka != kb) return false;
      for (const auto& g : ka)
        if (std::memcmp(a.block_ptr(g)->voxels.data(), b.block_ptr(g)->voxels.data(),
                        sizeof(a.block_ptr(g)->voxels)) != 0)
          return false;
      return true;
    };
    CHECK(same(*back.tsdf, tsdf));
    CHECK(same(*back.esdf, esdf));
    CHECK(same_layer(*back.esdf, oesdf));
    bool threw = false;
    try {
      vb::load_snapshot("/tmp/does-not-exist.vxlf");
    } catch (const vb::IoError&) {
      threw = true;
    }
    CHECK(threw);
    std::remove(path.c_str());
  }

  // Occupancy overloads (integrator.cpp:176-189, esdf/integrator.cpp:574-579)
  // and the cake's occupancy layer in a snapshot.
  {
    vb::Layer<vb::OccupancyVoxel> occ(0.05);
    vb::Layer<vb::EsdfVoxel> oesdf2(0.05);
    vxo_layer *oocc = nullptr, *oe2 = nullptr;
    vxo_layer_create(VXM_LAYER_OCCUPANCY, 0.05, 0, &oocc);
    vxo_layer_create(VXM_LAYER_ESDF, 0.05, 0, &oe2);
    for (int k = 0; k < 3; ++k) {
      vxm_pose p;
      vxm_synth_orbit_pose(scene, 0, k, 8, &p);
      vb::DepthImage depth(cam.width, cam.height);
      vxm_synth_render_camera(scene, &p, &cam_c, depth.data.data());
      const auto a = vb::integrate_depth(occ, depth, pose_of(p), cam, cfg);
      vxm_grid_index* ob = nullptr;
      uint64_t on = 0;
      vxo_integrate_camera(oocc, depth.data.data(), depth.width, depth.height, &p, &cam_c, &cfg_c, &ob, &on);
      const auto b = oracle_list(ob, on);
      CHECK(!a.empty());
      CHECK(a == b);
      const auto ea = vb::update_esdf(oesdf2, occ, a, ecfg);
      const auto bc = vb::to_c(b);
      vxo_update_esdf(oe2, oocc, bc.data(), bc.size(), &ecfg_c, &ob, &on);
      CHECK(ea == oracle_list(ob, on));
    }
    CHECK(same_layer(occ, oocc));
    {  // voxel_ptr (layer.hpp:88-96): the block's voxel or nullptr
      const auto keys = occ.sorted_indices();
      const vb::GlobalVoxelIndex gv = vb::global_voxel_index(keys.front(), {3, 4, 5});
      const vb::OccupancyVoxel* p = occ.voxel_ptr(gv);
      CHECK(p != nullptr && p == &occ.block_ptr(keys.front())->voxel({3, 4, 5}));
      CHECK(occ.voxel_ptr(vb::GlobalVoxelIndex{1 << 24, 0, 0}) == nullptr);
    }
    CHECK(same_layer(oesdf2, oe2));
    const std::string path = "/tmp/vxm_facade_test_occ.vxlf";
    vb::LayerCake cake(0.05);
    cake.occupancy = std::make_unique<vb::Layer<vb::OccupancyVoxel>>(occ.clone());
    vb::save_snapshot(cake, path);
    vb::LayerCake back = vb::load_snapshot(path);
    CHECK(!back.tsdf && back.occupancy && !back.esdf);
    CHECK(back.occupancy && same_layer(*back.occupancy, oocc));
    std::remove(path.c_str());
    vxo_layer_destroy(oocc);
    vxo_layer_destroy(oe2);
  }

  // A writable handle kept across device operations (layer.hpp:44-46): the
  // reference's host blocks ARE the map, so a write through a handle taken
  // before integrate_depth and made after it must persist and compose voxel
  // by voxel with the integration's own changes.  The oracle does the same
  // writes on its own layer.
  {
    vb::Layer<vb::TsdfVoxel> t2(0.05);
    vxo_layer* o2 = nullptr;
    vxo_layer_create(VXM_LAYER_TSDF, 0.05, 0, &o2);
    auto frame = [&](int k) {
      vxm_pose p;
      vxm_synth_orbit_pose(scene, 0, k, 8, &p);
      vb::DepthImage depth(cam.width, cam.height);
      vxm_synth_render_camera(scene, &p, &cam_c, depth.data.data());
      const auto a = vb::integrate_depth(t2, depth, pose_of(p), cam, cfg);
      vxm_grid_index* ob = nullptr;
      uint64_t on = 0;
      vxo_integrate_camera(o2, depth.data.data(), depth.width, depth.height, &p, &cam_c, &cfg_c, &ob, &on);
      CHECK(a == oracle_list(ob, on));
      return a;
    };
    auto oracle_write = [&](const vb::GridIndex& g, int lin, vb::TsdfVoxel v) {
      const uint64_t n = vxo_layer_num_blocks(o2);
      std::vector<vxm_grid_index> ok(n);
      std::vector<vb::TsdfVoxel> ov(n * 512);
      vxo_layer_export(o2, ok.data(), ov.data());
      for (uint64_t i = 0; i < n; ++i)
        if (ok[i].x == g.x && ok[i].y == g.y && ok[i].z == g.z) {
          ov[i * 512 + lin] = v;
          vxo_layer_write_blocks(o2, &ok[i], 1, ov.data() + i * 512);
        }
    };
    const auto first = frame(0);
    CHECK(!first.empty());
    const vb::GridIndex g = first[first.size() / 2];
    vb::VoxelBlock<vb::TsdfVoxel>* h = t2.block_ptr(g);  // kept across the frames below
    CHECK(h != nullptr);
    const auto second = frame(1);                         // device op (may change block g)
    const vb::TsdfVoxel w1{0.0625f, 3.0f};
    h->voxels[7] = w1;                                    // write AFTER the device op
    oracle_write(g, 7, w1);
    const auto third = frame(2);                          // must see the write
    const vb::TsdfVoxel w2{-0.03125f, 5.0f};
    h->voxels[300] = w2;
    oracle_write(g, 300, w2);
    CHECK(t2.block_ptr(g) == h);                          // the handle stays valid
    CHECK(std::memcmp(&h->voxels[300], &w2, sizeof w2) == 0);
    CHECK(same_layer(t2, o2));
    vxo_layer_destroy(o2);
  }

  vxo_layer_destroy(otsdf);
  vxo_layer_destroy(oesdf);
  vxm_synth_scene_destroy(scene);
  std::printf("facade_test: %s (%d failures)\n", failures ? "FAIL" : "PASS", failures);
  return failures ? 1 : 0;
}
