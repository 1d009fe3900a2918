// voxmap_b200 C++ facade: the reference's C++ mapper API (namespace voxmap,
// /root/reference/proj/include) re-exposed over the C-ABI of libvoxmap_b200.
//
// A user of the reference switches by including this header instead of the
// voxmap headers and linking libvoxmap_b200.so.  Names, argument meaning and
// error behaviour follow the reference:
//   Layer<TsdfVoxel/EsdfVoxel>  core/layer.hpp:47-125 (device-resident; host
//                               block_ptr()/voxel_ptr() go through a lazy mirror)
//   integrate_depth             integrate/integrator.hpp:36-45
//   blocks_in_view              sensor/view.hpp:38-48
//   update_esdf, mark_sites, clear_invalid, lower_esdf, EsdfUpdateState
//                               esdf/integrator.hpp:67-120
//   query_batch                 query/query.hpp:59-62
//   InvalidPoseError, MapCapacityError, std::invalid_argument
// Eigen types in the reference signatures become small POD vectors here
// (Vec3 / Mat3); everything else is field-for-field identical.
#pragma once

#include <algorithm>
#include <array>
#include <cmath>
#include <compare>
#include <cstdint>
#include <cstring>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <unordered_map>
#include <vector>

#include "voxmap_b200.h"

namespace voxmap_b200 {

inline constexpr int kVoxelsPerSide = 8;
inline constexpr int kVoxelsPerBlock = 512;

// ---- errors (sensor/pose.hpp:23-26, core/layer.hpp:28-31) ----------------------
class InvalidPoseError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class MapCapacityError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class DeviceError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};
class IoError : public std::runtime_error {  // core/serialization.hpp:24-27
 public:
  using std::runtime_error::runtime_error;
};

inline void check(vxm_status s) {
  if (s == VXM_OK) return;
  const std::string msg = vxm_last_error();
  switch (s) {
    case VXM_ERR_INVALID_POSE: throw InvalidPoseError(msg);
    case VXM_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case VXM_ERR_CAPACITY: throw MapCapacityError(msg);
    case VXM_ERR_IO: throw IoError(msg);
    default: throw DeviceError(msg);
  }
}

// ---- core types (core/indexing.hpp, core/voxels.hpp) ----------------------------
struct GridIndex {
  int32_t x = 0, y = 0, z = 0;
  friend auto operator<=>(const GridIndex&, const GridIndex&) = default;
};
struct Vec3 {
  double x = 0, y = 0, z = 0;
  double& operator[](int i) { return i == 0 ? x : (i == 1 ? y : z); }
  double operator[](int i) const { return i == 0 ? x : (i == 1 ? y : z); }
  bool operator==(const Vec3&) const = default;
};

// ---- index algebra (core/indexing.hpp:33-139) --------------
struct VoxelIndex {  // voxel inside a block, 0..7 per axis
  int32_t x = 0, y = 0, z = 0;
  friend auto operator<=>(const VoxelIndex&, const VoxelIndex&) = default;
};
struct GlobalVoxelIndex {  // voxel in the whole map
  int64_t x = 0, y = 0, z = 0;
  friend auto operator<=>(const GlobalVoxelIndex&, const GlobalVoxelIndex&) = default;
};
// x-fastest linear index inside a block: x + 8 (y + 8 z)
inline int linear_voxel_index(const VoxelIndex& v) {
  return v.x + kVoxelsPerSide * (v.y + kVoxelsPerSide * v.z);
}
inline VoxelIndex voxel_index_from_linear(int lin) {
  const int x = lin % kVoxelsPerSide, r = lin / kVoxelsPerSide;
  return VoxelIndex{x, r % kVoxelsPerSide, r / kVoxelsPerSide};
}
// floor(a / 8), also for negative a
inline int64_t floor_div_side(int64_t a) {
  return a >= 0 ? a / kVoxelsPerSide : -((kVoxelsPerSide - 1 - a) / kVoxelsPerSide);
}
inline GlobalVoxelIndex global_voxel_index(const GridIndex& g, const VoxelIndex& v) {
  return GlobalVoxelIndex{int64_t(g.x) * kVoxelsPerSide + v.x, int64_t(g.y) * kVoxelsPerSide + v.y,
                          int64_t(g.z) * kVoxelsPerSide + v.z};
}
inline GridIndex block_of_global_voxel(const GlobalVoxelIndex& gv) {
  return GridIndex{int32_t(floor_div_side(gv.x)), int32_t(floor_div_side(gv.y)),
                   int32_t(floor_div_side(gv.z))};
}
inline VoxelIndex local_voxel_of_global(const GlobalVoxelIndex& gv) {
  const GridIndex b = block_of_global_voxel(gv);
  return VoxelIndex{int32_t(gv.x - int64_t(b.x) * kVoxelsPerSide), int32_t(gv.y - int64_t(b.y) * kVoxelsPerSide),
                    int32_t(gv.z - int64_t(b.z) * kVoxelsPerSide)};
}
// global voxel containing a metric position: floor(p / voxel_size) per axis
inline GlobalVoxelIndex position_to_global_voxel(const Vec3& p, double voxel_size) {
  return GlobalVoxelIndex{int64_t(std::floor(p.x / voxel_size)), int64_t(std::floor(p.y / voxel_size)),
                          int64_t(std::floor(p.z / voxel_size))};
}
inline void position_to_indices(const Vec3& p, double voxel_size, GridIndex* block, VoxelIndex* voxel) {
  const GlobalVoxelIndex gv = position_to_global_voxel(p, voxel_size);
  *block = block_of_global_voxel(gv);
  *voxel = local_voxel_of_global(gv);
}
inline GridIndex position_to_block_index(const Vec3& p, double voxel_size) {
  return block_of_global_voxel(position_to_global_voxel(p, voxel_size));
}
// voxel centre: ((8 g + v) + 0.5) * voxel_size, the reference's association
inline Vec3 voxel_center(const GridIndex& g, const VoxelIndex& v, double voxel_size) {
  return Vec3{(double(g.x) * kVoxelsPerSide + v.x + 0.5) * voxel_size,
              (double(g.y) * kVoxelsPerSide + v.y + 0.5) * voxel_size,
              (double(g.z) * kVoxelsPerSide + v.z + 0.5) * voxel_size};
}
inline Vec3 global_voxel_center(const GlobalVoxelIndex& gv, double voxel_size) {
  return Vec3{(double(gv.x) + 0.5) * voxel_size, (double(gv.y) + 0.5) * voxel_size,
              (double(gv.z) + 0.5) * voxel_size};
}
inline Vec3 block_origin(const GridIndex& g, double voxel_size) {
  const double edge = kVoxelsPerSide * voxel_size;
  return Vec3{g.x * edge, g.y * edge, g.z * edge};
}
struct TsdfVoxel {
  float distance = 0.0f;
  float weight = 0.0f;
};
struct OccupancyVoxel {  // core/voxels.hpp:28-32
  float log_odds = 0.0f;
};
struct ColorVoxel {  // core/voxels.hpp:34-41
  uint8_t r = 0, g = 0, b = 0, reserved = 0;
  float weight = 0.0f;
};
struct EsdfVoxel {
  static constexpr uint8_t kObserved = 1, kSite = 2, kInside = 4;
  int32_t squared_distance = 0;
  int16_t parent_x = 0, parent_y = 0, parent_z = 0;
  uint8_t flags = 0, reserved = 0;
  bool observed() const { return flags & kObserved; }
  bool is_site() const { return flags & kSite; }
  bool inside() const { return flags & kInside; }
  bool has_parent() const { return parent_x || parent_y || parent_z; }
  friend bool operator==(const EsdfVoxel&, const EsdfVoxel&) = default;
};
static_assert(sizeof(TsdfVoxel) == sizeof(vxm_tsdf_voxel) && sizeof(EsdfVoxel) == sizeof(vxm_esdf_voxel) &&
              sizeof(OccupancyVoxel) == sizeof(vxm_occupancy_voxel) &&
              sizeof(ColorVoxel) == sizeof(vxm_color_voxel));

template <typename V>
struct VoxelBlock {
  std::array<V, kVoxelsPerBlock> voxels{};
  V& voxel(const VoxelIndex& v) { return voxels[size_t(linear_voxel_index(v))]; }
  const V& voxel(const VoxelIndex& v) const { return voxels[size_t(linear_voxel_index(v))]; }
};

template <typename V>
struct LayerTraits;
template <>
struct LayerTraits<TsdfVoxel> {
  static constexpr vxm_layer_type type = VXM_LAYER_TSDF;
};
template <>
struct LayerTraits<EsdfVoxel> {
  static constexpr vxm_layer_type type = VXM_LAYER_ESDF;
};
template <>
struct LayerTraits<OccupancyVoxel> {
  static constexpr vxm_layer_type type = VXM_LAYER_OCCUPANCY;
};
template <>
struct LayerTraits<ColorVoxel> {
  static constexpr vxm_layer_type type = VXM_LAYER_COLOR;
};

struct GridHash {
  size_t operator()(const GridIndex& g) const {  // indexing.hpp:146-154
    return size_t((uint64_t(uint32_t(g.x)) * 73856093ull) ^ (uint64_t(uint32_t(g.y)) * 19349669ull) ^
                  (uint64_t(uint32_t(g.z)) * 83492791ull));
  }
};

// ---- context --------------------------------------------------------------------
// One CUDA device + stream.  default_context() serves the common case.
class Context {
 public:
  explicit Context(int device = 0) { check(vxm_context_create(device, &h_)); }
  ~Context() { vxm_context_destroy(h_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  vxm_context* handle() const { return h_; }

 private:
  vxm_context* h_ = nullptr;
};

inline Context& default_context() {
  static Context ctx(0);
  return ctx;
}

// Block list result helper.
class BlockList {
 public:
  explicit BlockList(Context& ctx) { check(vxm_blocklist_create(ctx.handle(), &h_)); }
  ~BlockList() { vxm_blocklist_destroy(h_); }
  BlockList(const BlockList&) = delete;
  vxm_blocklist* handle() const { return h_; }
  std::vector<GridIndex> to_vector() const {
    const vxm_grid_index* p = nullptr;
    uint64_t n = 0;
    check(vxm_blocklist_host(h_, &p, &n));
    std::vector<GridIndex> out(n);
    for (uint64_t i = 0; i < n; ++i) out[i] = {p[i].x, p[i].y, p[i].z};
    return out;
  }

 private:
  vxm_blocklist* h_ = nullptr;
};

// ---- Layer<V> — core/layer.hpp:47-125 ---------------------------------------------
// Blocks live on the device.  Host reads (block_ptr/voxel_ptr/clone) sync a
// lazy host mirror whose block addresses never change (handles stay valid, as
// layer.hpp:44-46 promises).  A block handed out through a non-const accessor
// stays "writable" for the layer's lifetime: before every device operation
// (and every mirror refresh) each writable block is compared with the bytes
// last exchanged with the device; voxels the caller changed since are merged
// into the device's current block voxel by voxel, so writes through a kept
// handle persist across device operations exactly as writes into the
// reference's host blocks do.
template <typename V>
class Layer {
 public:
  using BlockType = VoxelBlock<V>;

  explicit Layer(double voxel_size, size_t max_blocks = size_t{1} << 30,
                 Context& ctx = default_context())
      : ctx_(&ctx) {
    check(vxm_layer_create(ctx.handle(), LayerTraits<V>::type, voxel_size, max_blocks, &h_));
    voxel_size_ = voxel_size;
    max_blocks_ = max_blocks;
  }
  // Adopts a C-ABI layer handle (e.g. from vxm_snapshot_load).
  Layer(vxm_layer* adopt, double voxel_size, Context& ctx)
      : h_(adopt), ctx_(&ctx), voxel_size_(voxel_size), max_blocks_(size_t{1} << 30) {}
  ~Layer() {
    if (h_) vxm_layer_destroy(h_);
  }
  Layer(Layer&& o) noexcept { *this = std::move(o); }
  Layer& operator=(Layer&& o) noexcept {
    std::swap(h_, o.h_);
    std::swap(ctx_, o.ctx_);
    std::swap(voxel_size_, o.voxel_size_);
    std::swap(max_blocks_, o.max_blocks_);
    std::swap(mirror_, o.mirror_);
    std::swap(mirror_valid_, o.mirror_valid_);
    std::swap(writable_, o.writable_);
    return *this;
  }

  double voxel_size() const { return voxel_size_; }
  double block_size() const { return voxel_size_ * kVoxelsPerSide; }
  // The C-ABI handle, with host-side edits uploaded first.
  vxm_layer* c_handle() const {
    flush();
    return h_;
  }
  size_t num_blocks() const {
    flush();
    uint64_t n = 0;
    check(vxm_layer_num_blocks(h_, &n));
    return n;
  }
  bool has_block(const GridIndex& g) const {
    flush();
    uint8_t out = 0;
    const vxm_grid_index k{g.x, g.y, g.z};
    check(vxm_layer_has_blocks(h_, &k, 1, &out));
    return out != 0;
  }
  const BlockType* block_ptr(const GridIndex& g) const {
    sync_mirror();
    auto it = mirror_.find(g);
    return it == mirror_.end() ? nullptr : it->second.get();
  }
  BlockType* block_ptr(const GridIndex& g) {
    sync_mirror();
    auto it = mirror_.find(g);
    if (it == mirror_.end()) return nullptr;
    make_writable(g, *it->second);
    return it->second.get();
  }
  BlockType& get_or_allocate(const GridIndex& g) {
    sync_mirror();
    auto it = mirror_.find(g);
    if (it == mirror_.end()) {
      const BlockType zero{};
      const vxm_grid_index k{g.x, g.y, g.z};
      check(vxm_layer_write_blocks(h_, &k, 1, zero.voxels.data()));
      it = mirror_.emplace(g, std::make_unique<BlockType>()).first;
    }
    make_writable(g, *it->second);
    return *it->second;
  }
  // voxel lookup by global voxel index; nullptr when the block is absent (layer.hpp:88-96)
  const V* voxel_ptr(const GlobalVoxelIndex& gv) const {
    const BlockType* b = block_ptr(block_of_global_voxel(gv));
    return b ? &b->voxel(local_voxel_of_global(gv)) : nullptr;
  }
  V* voxel_ptr(const GlobalVoxelIndex& gv) {
    BlockType* b = block_ptr(block_of_global_voxel(gv));
    return b ? &b->voxel(local_voxel_of_global(gv)) : nullptr;
  }
  std::vector<GridIndex> sorted_indices() const {
    flush();
    const size_t n = num_blocks();
    std::vector<vxm_grid_index> k(n);
    check(vxm_layer_export(h_, k.data(), nullptr, n));
    std::vector<GridIndex> out(n);
    for (size_t i = 0; i < n; ++i) out[i] = {k[i].x, k[i].y, k[i].z};
    return out;
  }
  Layer clone() const {
    flush();
    vxm_layer* c = nullptr;
    check(vxm_layer_clone(h_, &c));
    Layer out;
    out.h_ = c;
    out.ctx_ = ctx_;
    out.voxel_size_ = voxel_size_;
    out.max_blocks_ = max_blocks_;
    return out;
  }

  // --- device interop (used by the free functions below) ---
  vxm_layer* device() const {
    flush();
    mirror_valid_ = false;  // the device op may change any block
    return h_;
  }
  Context& context() const { return *ctx_; }

 private:
  Layer() = default;
  void make_writable(const GridIndex& g, const BlockType& b) {
    writable_.try_emplace(g, b);  // base = the bytes the mirror holds now (device-equal)
  }
  // Uploads what the caller wrote through writable handles since the last
  // exchange.  Mirror valid: no device op since, so the device block equals
  // the base and the host block is uploaded whole.  Mirror stale: the device
  // may have changed the block, so the caller's changed voxels are merged
  // into the device's current bytes (and the handle sees the merge).
  void flush() const {
    std::vector<vxm_grid_index> keys;
    std::vector<V> vox;
    std::vector<const GridIndex*> gs;
    for (auto& kv : writable_) {
      const BlockType& host = *mirror_.at(kv.first);
      if (std::memcmp(host.voxels.data(), kv.second.voxels.data(), sizeof(host.voxels)) == 0) continue;
      gs.push_back(&kv.first);
    }
    if (gs.empty()) return;
    for (const GridIndex* g : gs) {
      BlockType& host = *mirror_.at(*g);
      BlockType& base = writable_.at(*g);
      const vxm_grid_index k{g->x, g->y, g->z};
      if (!mirror_valid_) {  // three-way merge against the device's current block
        BlockType dev;
        check(vxm_layer_read_blocks(h_, &k, 1, dev.voxels.data(), nullptr));
        for (int v = 0; v < kVoxelsPerBlock; ++v)
          if (std::memcmp(&host.voxels[v], &base.voxels[v], sizeof(V)) != 0) dev.voxels[v] = host.voxels[v];
        host = dev;
      }
      base = host;
      keys.push_back(k);
      vox.insert(vox.end(), host.voxels.begin(), host.voxels.end());
    }
    check(vxm_layer_write_blocks(h_, keys.data(), keys.size(), vox.data()));
  }
  void sync_mirror() const {
    if (mirror_valid_) return;
    flush();
    uint64_t n = 0;
    check(vxm_layer_num_blocks(h_, &n));
    std::vector<vxm_grid_index> k(n);
    std::vector<V> vox(n * kVoxelsPerBlock);
    check(vxm_layer_export(h_, k.data(), vox.data(), n));
    for (uint64_t i = 0; i < n; ++i) {
      const GridIndex g{k[i].x, k[i].y, k[i].z};
      auto& slot = mirror_[g];  // existing blocks keep their address (handles stay valid)
      if (!slot) slot = std::make_unique<BlockType>();
      std::memcpy(slot->voxels.data(), vox.data() + i * kVoxelsPerBlock, sizeof(V) * kVoxelsPerBlock);
      auto w = writable_.find(g);
      if (w != writable_.end()) w->second = *slot;
    }
    mirror_valid_ = true;
  }

  vxm_layer* h_ = nullptr;
  Context* ctx_ = nullptr;
  double voxel_size_ = 0.0;
  size_t max_blocks_ = 0;
  mutable std::unordered_map<GridIndex, std::unique_ptr<BlockType>, GridHash> mirror_;
  mutable bool mirror_valid_ = false;
  // blocks handed out writable -> the bytes last exchanged with the device
  mutable std::unordered_map<GridIndex, BlockType, GridHash> writable_;
};

// ---- sensors / configs ---------------------------------------------------------
struct Mat3 {
  double m[3][3] = {{1, 0, 0}, {0, 1, 0}, {0, 0, 1}};
  double& operator()(int r, int c) { return m[r][c]; }
  double operator()(int r, int c) const { return m[r][c]; }
};
struct Pose {  // sensor/pose.hpp:30-60
  Mat3 R;
  Vec3 t;
  static Pose identity() { return Pose{}; }
  vxm_pose c() const {
    vxm_pose p;
    for (int r = 0; r < 3; ++r)
      for (int cc = 0; cc < 3; ++cc) p.R[3 * r + cc] = R(r, cc);
    p.t[0] = t.x;
    p.t[1] = t.y;
    p.t[2] = t.z;
    return p;
  }
  bool valid() const {
    const vxm_pose p = c();
    return vxm_pose_valid(&p) != 0;
  }
  Pose inverse() const {
    const vxm_pose p = c();
    vxm_pose o;
    vxm_pose_inverse(&p, &o);
    Pose out;
    for (int r = 0; r < 3; ++r)
      for (int cc = 0; cc < 3; ++cc) out.R(r, cc) = o.R[3 * r + cc];
    out.t = {o.t[0], o.t[1], o.t[2]};
    return out;
  }
};
struct CameraIntrinsics {  // sensor/camera.hpp:24-31
  double fu = 0, fv = 0, cu = 0, cv = 0;
  int width = 0, height = 0;
  double max_depth = 0;
  vxm_camera c() const { return {fu, fv, cu, cv, width, height, max_depth}; }
};
struct LidarIntrinsics {  // sensor/lidar.hpp:27-38
  int num_azimuth = 0, num_elevation = 0;
  double azimuth_start = 0, elevation_start = 0, azimuth_fov = 2 * 3.14159265358979323846,
         elevation_fov = 0, min_range = 0, max_range = 0;
  vxm_lidar c() const {
    return {num_azimuth, num_elevation, azimuth_start, elevation_start,
            azimuth_fov, elevation_fov, min_range,     max_range};
  }
};
struct DepthImage {  // sensor/image.hpp:27-39
  int width = 0, height = 0;
  std::vector<float> data;
  DepthImage() = default;
  DepthImage(int w, int h) : width(w), height(h), data(size_t(w) * h, 0.0f) {}
  float& at(int col, int row) { return data[size_t(row) * width + col]; }
  float at(int col, int row) const { return data[size_t(row) * width + col]; }
};
enum class WeightMode { kConstant, kInverseSquareDepth };
enum class DepthSampleMode { kNearest, kLinearForegroundSafe };
struct IntegratorConfig {  // integrate/config.hpp:38-56
  double truncation = 0.2;
  float max_weight = 100.0f;
  WeightMode weighting = WeightMode::kConstant;
  double max_integration_distance = 5.0;
  DepthSampleMode camera_sample = DepthSampleMode::kNearest;
  DepthSampleMode lidar_sample = DepthSampleMode::kLinearForegroundSafe;
  float max_sample_gap = 0.2f;
  int view_pixel_subsample = 8;
  bool parallel = true;
  vxm_integrator_config c() const {
    vxm_integrator_config k;
    vxm_integrator_config_default(&k);
    k.truncation = truncation;
    k.max_weight = max_weight;
    k.weighting = weighting == WeightMode::kInverseSquareDepth ? VXM_WEIGHT_INVERSE_SQUARE
                                                               : VXM_WEIGHT_CONSTANT;
    k.max_integration_distance = max_integration_distance;
    k.camera_sample = camera_sample == DepthSampleMode::kNearest ? VXM_SAMPLE_NEAREST : VXM_SAMPLE_LINEAR;
    k.lidar_sample = lidar_sample == DepthSampleMode::kNearest ? VXM_SAMPLE_NEAREST : VXM_SAMPLE_LINEAR;
    k.max_sample_gap = max_sample_gap;
    k.view_pixel_subsample = view_pixel_subsample;
    k.parallel = parallel;
    return k;
  }
};
struct ViewConfig {  // sensor/view.hpp:27-31
  double max_integration_distance = 5.0;
  double truncation = 0.2;
  int pixel_subsample = 8;
};
struct EsdfConfig {  // esdf/integrator.hpp:30-40
  double site_threshold = 0.05;
  float occupied_log_odds_threshold = 0.0f;
  double max_distance = 2.0;
  bool parallel = true;
  vxm_esdf_config c() const {
    return {site_threshold, occupied_log_odds_threshold, max_distance, parallel ? 1 : 0};
  }
};
struct QueryConfig {  // query/query.hpp:41-49
  bool interpolate = true;
  bool parallel = true;
};
struct QueryResult {  // query/query.hpp:30-39
  bool known = false;
  double distance = 0.0;
  Vec3 gradient;
  bool operator==(const QueryResult&) const = default;
};

inline std::vector<vxm_grid_index> to_c(const std::vector<GridIndex>& v) {
  std::vector<vxm_grid_index> out(v.size());
  for (size_t i = 0; i < v.size(); ++i) out[i] = {v[i].x, v[i].y, v[i].z};
  return out;
}
inline std::vector<GridIndex> from_c(const vxm_grid_index* p, uint64_t n) {
  std::vector<GridIndex> out(n);
  for (uint64_t i = 0; i < n; ++i) out[i] = {p[i].x, p[i].y, p[i].z};
  return out;
}

// ---- integrate/integrator.hpp:36-55 (TSDF and occupancy overloads) ---------------
template <typename V>
concept SourceVoxel = std::is_same_v<V, TsdfVoxel> || std::is_same_v<V, OccupancyVoxel>;

template <SourceVoxel V>
inline std::vector<GridIndex> integrate_depth(Layer<V>& layer, const DepthImage& depth,
                                              const Pose& T_LS, const CameraIntrinsics& camera,
                                              const IntegratorConfig& cfg) {
  const vxm_pose p = T_LS.c();
  const vxm_camera cam = camera.c();
  const vxm_integrator_config k = cfg.c();
  BlockList out(layer.context());
  check(vxm_integrate_depth_camera(layer.device(), depth.data.data(), depth.width, depth.height, &p,
                                   &cam, &k, out.handle()));
  return out.to_vector();
}
template <SourceVoxel V>
inline std::vector<GridIndex> integrate_depth(Layer<V>& layer, const DepthImage& depth,
                                              const Pose& T_LS, const LidarIntrinsics& lidar,
                                              const IntegratorConfig& cfg) {
  const vxm_pose p = T_LS.c();
  const vxm_lidar li = lidar.c();
  const vxm_integrator_config k = cfg.c();
  BlockList out(layer.context());
  check(vxm_integrate_depth_lidar(layer.device(), depth.data.data(), depth.width, depth.height, &p,
                                  &li, &k, out.handle()));
  return out.to_vector();
}

// ---- sensor/view.hpp:38-48 ----------------------------------------------------------
inline std::vector<GridIndex> blocks_in_view(const Pose& T_LS, const CameraIntrinsics& camera,
                                             const DepthImage& depth, double block_size,
                                             const ViewConfig& cfg, Context& ctx = default_context()) {
  const vxm_pose p = T_LS.c();
  const vxm_camera cam = camera.c();
  const vxm_view_config v{cfg.max_integration_distance, cfg.truncation, cfg.pixel_subsample};
  BlockList out(ctx);
  check(vxm_blocks_in_view_camera(ctx.handle(), &p, &cam, depth.data.data(), depth.width,
                                  depth.height, block_size, &v, out.handle()));
  return out.to_vector();
}
inline std::vector<GridIndex> blocks_in_view(const Pose& T_LS, const LidarIntrinsics& lidar,
                                             const DepthImage& depth, double block_size,
                                             const ViewConfig& cfg, Context& ctx = default_context()) {
  const vxm_pose p = T_LS.c();
  const vxm_lidar li = lidar.c();
  const vxm_view_config v{cfg.max_integration_distance, cfg.truncation, cfg.pixel_subsample};
  BlockList out(ctx);
  check(vxm_blocks_in_view_lidar(ctx.handle(), &p, &li, depth.data.data(), depth.width,
                                 depth.height, block_size, &v, out.handle()));
  return out.to_vector();
}

// ---- esdf/integrator.hpp:67-120 -------------------------------------------------------
struct EsdfUpdateState {
  std::vector<GridIndex> indices_to_update, indices_to_clear, cleared_indices;
};

namespace detail {
struct StateHandle {
  vxm_esdf_state* h = nullptr;
  explicit StateHandle(const EsdfUpdateState& s) {
    check(vxm_esdf_state_create(&h));
    const auto a = to_c(s.indices_to_update), b = to_c(s.indices_to_clear), c = to_c(s.cleared_indices);
    check(vxm_esdf_state_set(h, 0, a.data(), a.size()));
    check(vxm_esdf_state_set(h, 1, b.data(), b.size()));
    check(vxm_esdf_state_set(h, 2, c.data(), c.size()));
  }
  void copy_to(EsdfUpdateState* s) const {
    const vxm_grid_index* p = nullptr;
    uint64_t n = 0;
    check(vxm_esdf_state_get(h, 0, &p, &n));
    s->indices_to_update = from_c(p, n);
    check(vxm_esdf_state_get(h, 1, &p, &n));
    s->indices_to_clear = from_c(p, n);
    check(vxm_esdf_state_get(h, 2, &p, &n));
    s->cleared_indices = from_c(p, n);
  }
  ~StateHandle() { vxm_esdf_state_destroy(h); }
};
}  // namespace detail

template <SourceVoxel V>
inline void mark_sites(Layer<EsdfVoxel>& esdf, const Layer<V>& source,
                       const std::vector<GridIndex>& updated_blocks, const EsdfConfig& cfg,
                       EsdfUpdateState* state, std::vector<GridIndex>* changed) {
  detail::StateHandle st(*state);
  const auto u = to_c(updated_blocks);
  const vxm_esdf_config k = cfg.c();
  BlockList out(esdf.context());
  check(vxm_esdf_mark_sites(esdf.device(), source.device(), u.data(), u.size(), &k, st.h,
                            out.handle()));
  st.copy_to(state);
  const auto c = out.to_vector();
  changed->insert(changed->end(), c.begin(), c.end());
}
inline void clear_invalid(Layer<EsdfVoxel>& esdf, const EsdfConfig& cfg, EsdfUpdateState* state,
                          std::vector<GridIndex>* changed) {
  detail::StateHandle st(*state);
  const vxm_esdf_config k = cfg.c();
  BlockList out(esdf.context());
  check(vxm_esdf_clear_invalid(esdf.device(), &k, st.h, out.handle()));
  st.copy_to(state);
  const auto c = out.to_vector();
  changed->insert(changed->end(), c.begin(), c.end());
}
inline int lower_esdf(Layer<EsdfVoxel>& esdf, const EsdfUpdateState& state, const EsdfConfig& cfg,
                      std::vector<GridIndex>* changed) {
  detail::StateHandle st(state);
  const vxm_esdf_config k = cfg.c();
  BlockList out(esdf.context());
  int rounds = 0;
  check(vxm_esdf_lower(esdf.device(), st.h, &k, out.handle(), &rounds));
  const auto c = out.to_vector();
  changed->insert(changed->end(), c.begin(), c.end());
  return rounds;
}
template <SourceVoxel V>
inline std::vector<GridIndex> update_esdf(Layer<EsdfVoxel>& esdf, const Layer<V>& source,
                                          const std::vector<GridIndex>& updated_blocks,
                                          const EsdfConfig& cfg) {
  const auto u = to_c(updated_blocks);
  const vxm_esdf_config k = cfg.c();
  BlockList out(esdf.context());
  check(vxm_update_esdf(esdf.device(), source.device(), u.data(), u.size(), &k, out.handle()));
  return out.to_vector();
}
inline double esdf_distance(const EsdfVoxel& v, double voxel_size) {  // esdf/integrator.hpp:59-63
  const double d = std::sqrt(static_cast<double>(v.squared_distance)) * voxel_size;
  return v.inside() ? -d : d;
}

// ---- query/query.hpp:59-62 ----------------------------------------------------------
inline std::vector<QueryResult> query_batch(const Layer<EsdfVoxel>& esdf,
                                            const std::vector<Vec3>& points, bool want_gradient,
                                            const QueryConfig& cfg = {}) {
  std::vector<double> xyz(points.size() * 3);
  for (size_t i = 0; i < points.size(); ++i) {
    xyz[3 * i] = points[i].x;
    xyz[3 * i + 1] = points[i].y;
    xyz[3 * i + 2] = points[i].z;
  }
  std::vector<vxm_query_result> r(points.size());
  const vxm_query_config k{cfg.interpolate ? 1 : 0, cfg.parallel ? 1 : 0};
  check(vxm_query_batch(esdf.device(), xyz.data(), points.size(), want_gradient ? 1 : 0, &k, r.data()));
  std::vector<QueryResult> out(points.size());
  for (size_t i = 0; i < points.size(); ++i) {
    out[i].known = r[i].known != 0;
    out[i].distance = r[i].distance;
    out[i].gradient = {r[i].gradient[0], r[i].gradient[1], r[i].gradient[2]};
  }
  return out;
}

// ---- color fusion (integrate/integrator.hpp:57-66) ----------------------------------
struct ColorImage {  // sensor/image.hpp:41-55
  int width = 0, height = 0;
  std::vector<std::array<uint8_t, 3>> data;
  ColorImage() = default;
  ColorImage(int w, int h) : width(w), height(h), data(size_t(w) * h) {}
  std::array<uint8_t, 3>& at(int col, int row) { return data[size_t(row) * width + col]; }
  const std::array<uint8_t, 3>& at(int col, int row) const { return data[size_t(row) * width + col]; }
};
inline std::vector<GridIndex> integrate_color(Layer<ColorVoxel>& color_layer, const ColorImage& color,
                                              const DepthImage& depth, const Pose& T_LS,
                                              const CameraIntrinsics& camera,
                                              const Layer<TsdfVoxel>& tsdf_layer,
                                              const IntegratorConfig& cfg) {
  const vxm_pose p = T_LS.c();
  const vxm_camera cam = camera.c();
  const vxm_integrator_config k = cfg.c();
  BlockList out(color_layer.context());
  check(vxm_integrate_color(color_layer.device(), color.data.empty() ? nullptr : color.data[0].data(),
                            color.width, color.height, depth.data.data(), depth.width, depth.height,
                            &p, &cam, tsdf_layer.device(), &k, out.handle()));
  return out.to_vector();
}

// ---- meshing (mesh/marching_cubes.hpp, mesh_layer.hpp, ply.hpp) ---------------------
struct MeshConfig {  // marching_cubes.hpp:24-33
  float min_weight = 1e-4f;
  bool parallel = true;
  vxm_mesh_config c() const { return {min_weight, parallel ? 1 : 0}; }
};
struct MeshBlock {  // mesh_layer.hpp:16-25
  std::vector<std::array<float, 3>> vertices, normals;
  std::vector<std::array<uint8_t, 3>> colors;
  std::vector<std::array<uint32_t, 3>> triangles;
  bool empty() const { return triangles.empty(); }
};
// MeshLayer (mesh_layer.hpp:27-66) over the library's mesh layer; block_ptr
// copies the block out (stable until the next call on the same block).
class MeshLayer {
 public:
  explicit MeshLayer(double voxel_size, Context& ctx = default_context()) : ctx_(&ctx) {
    check(vxm_mesh_layer_create(ctx.handle(), voxel_size, &h_));
  }
  ~MeshLayer() { vxm_mesh_layer_destroy(h_); }
  MeshLayer(const MeshLayer&) = delete;
  MeshLayer& operator=(const MeshLayer&) = delete;
  double voxel_size() const { return vxm_mesh_layer_voxel_size(h_); }
  size_t num_blocks() const { return size_t(vxm_mesh_layer_num_blocks(h_)); }
  std::vector<GridIndex> sorted_indices() const {
    std::vector<vxm_grid_index> k(num_blocks());
    check(vxm_mesh_layer_sorted_indices(h_, k.data(), k.size()));
    return from_c(k.data(), k.size());
  }
  const MeshBlock* block_ptr(const GridIndex& g) const {
    const vxm_grid_index k{g.x, g.y, g.z};
    vxm_mesh_block_view v{};
    int found = 0;
    check(vxm_mesh_layer_block(h_, &k, &v, &found));
    if (!found) return nullptr;
    MeshBlock& b = cache_[g];
    b.vertices.resize(v.n_vertices);
    b.normals.resize(v.n_vertices);
    b.colors.resize(v.n_colors);
    b.triangles.resize(v.n_triangles);
    if (v.n_vertices) {
      std::memcpy(b.vertices.data(), v.vertices, 12 * v.n_vertices);
      std::memcpy(b.normals.data(), v.normals, 12 * v.n_vertices);
    }
    if (v.n_colors) std::memcpy(b.colors.data(), v.colors, 3 * v.n_colors);
    if (v.n_triangles) std::memcpy(b.triangles.data(), v.triangles, 12 * v.n_triangles);
    return &b;
  }
  void erase(const GridIndex& g) {
    const vxm_grid_index k{g.x, g.y, g.z};
    check(vxm_mesh_layer_erase(h_, &k));
    cache_.erase(g);
  }
  vxm_mesh_layer* handle() const { return h_; }
  Context& context() const { return *ctx_; }

 private:
  vxm_mesh_layer* h_ = nullptr;
  Context* ctx_;
  mutable std::unordered_map<GridIndex, MeshBlock, GridHash> cache_;
};
inline MeshBlock mesh_block(const Layer<TsdfVoxel>& tsdf, const GridIndex& g, const MeshConfig& cfg = {},
                            const Layer<ColorVoxel>* color = nullptr) {
  MeshLayer tmp(tsdf.voxel_size(), tsdf.context());
  const vxm_grid_index k{g.x, g.y, g.z};
  const vxm_mesh_config c = cfg.c();
  check(vxm_mesh_block(tmp.handle(), tsdf.device(), &k, &c, color ? color->device() : nullptr));
  return *tmp.block_ptr(g);
}
inline std::vector<GridIndex> update_mesh(MeshLayer& mesh, const Layer<TsdfVoxel>& tsdf,
                                          const std::vector<GridIndex>& updated_blocks,
                                          const MeshConfig& cfg = {},
                                          const Layer<ColorVoxel>* color = nullptr) {
  const auto u = to_c(updated_blocks);
  const vxm_mesh_config c = cfg.c();
  BlockList out(mesh.context());
  check(vxm_update_mesh(mesh.handle(), tsdf.device(), u.data(), u.size(), &c,
                        color ? color->device() : nullptr, out.handle()));
  return out.to_vector();
}
inline void save_mesh_ply(const MeshLayer& mesh, const std::string& path) {
  check(vxm_save_mesh_ply(mesh.handle(), path.c_str()));
}

// ---- snapshots (core/layer_cake.hpp:27-57, core/serialization.hpp:29-35) --------
// The LayerCake's voxel layers (TSDF, occupancy, color, ESDF).
struct LayerCake {
  explicit LayerCake(double vs) : voxel_size(vs) {}
  double voxel_size;
  std::unique_ptr<Layer<TsdfVoxel>> tsdf;
  std::unique_ptr<Layer<OccupancyVoxel>> occupancy;
  std::unique_ptr<Layer<ColorVoxel>> color;
  std::unique_ptr<Layer<EsdfVoxel>> esdf;
  Layer<ColorVoxel>& require_color() {
    if (!color) color = std::make_unique<Layer<ColorVoxel>>(voxel_size);
    return *color;
  }
  Layer<TsdfVoxel>& require_tsdf() {
    if (!tsdf) tsdf = std::make_unique<Layer<TsdfVoxel>>(voxel_size);
    return *tsdf;
  }
  Layer<OccupancyVoxel>& require_occupancy() {
    if (!occupancy) occupancy = std::make_unique<Layer<OccupancyVoxel>>(voxel_size);
    return *occupancy;
  }
  Layer<EsdfVoxel>& require_esdf() {
    if (!esdf) esdf = std::make_unique<Layer<EsdfVoxel>>(voxel_size);
    return *esdf;
  }
};

inline void save_snapshot(const LayerCake& cake, const std::string& path) {
  check(vxm_snapshot_save_layers(path.c_str(), cake.voxel_size,
                                 cake.tsdf ? cake.tsdf->c_handle() : nullptr,
                                 cake.occupancy ? cake.occupancy->c_handle() : nullptr,
                                 cake.color ? cake.color->c_handle() : nullptr,
                                 cake.esdf ? cake.esdf->c_handle() : nullptr));
}

inline LayerCake load_snapshot(const std::string& path, Context& ctx = default_context()) {
  double vs = 0.0;
  vxm_layer *t = nullptr, *o = nullptr, *cl = nullptr, *e = nullptr;
  check(vxm_snapshot_load_layers(ctx.handle(), path.c_str(), &vs, &t, &o, &cl, &e));
  LayerCake cake(vs);
  if (t) cake.tsdf = std::make_unique<Layer<TsdfVoxel>>(t, vs, ctx);
  if (o) cake.occupancy = std::make_unique<Layer<OccupancyVoxel>>(o, vs, ctx);
  if (cl) cake.color = std::make_unique<Layer<ColorVoxel>>(cl, vs, ctx);
  if (e) cake.esdf = std::make_unique<Layer<EsdfVoxel>>(e, vs, ctx);
  return cake;
}

}  // namespace voxmap_b200
