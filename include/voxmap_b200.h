/*
 * voxmap_b200 — C-ABI of the B200-native per-frame map update
 * (block allocation -> TSDF projective integration -> ESDF -> query).
 *
 * This is the drop-in boundary that replaces the reference's C++ mapper API
 * in /root/reference/proj/include (namespace voxmap).  Every entry point names
 * the reference interface it replaces (file:line under proj/).  The C++
 * facade in include/voxmap_b200/voxmap.hpp re-exposes the reference's
 * signatures (Layer<V>, integrate_depth, update_esdf, query_batch, ...) on
 * top of these functions; INTEGRATION.md shows the binding.
 *
 * Conventions
 *   - Plain C types only: pointers + sizes, POD config structs mirroring the
 *     reference's config structs field for field.
 *   - Every function returns vxm_status; on failure vxm_last_error() holds a
 *     message.  Status codes map 1:1 onto the reference's exception types
 *     (InvalidPoseError, std::invalid_argument, MapCapacityError).
 *   - Host-pointer entry points are synchronous (they return the reference's
 *     by-value results).  *_device entry points take device pointers, are
 *     stream-ordered on the context's stream, and report errors at
 *     vxm_context_synchronize().
 *   - There is no CPU fallback: without a usable sm_100 device every compute
 *     entry point fails with VXM_ERR_CUDA.
 */
#ifndef VOXMAP_B200_H_
#define VOXMAP_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status ----------------------------------------------------------- */
typedef enum {
  VXM_OK = 0,
  VXM_ERR_INVALID_POSE = 1,     /* voxmap::InvalidPoseError      pose.hpp:23-26   */
  VXM_ERR_INVALID_ARGUMENT = 2, /* std::invalid_argument                         */
  VXM_ERR_CAPACITY = 3,         /* voxmap::MapCapacityError      layer.hpp:28-31  */
  VXM_ERR_CUDA = 4,             /* device missing / CUDA runtime failure         */
  VXM_ERR_INTERNAL = 5,
  VXM_ERR_IO = 6                /* voxmap::IoError          serialization.hpp:24-27 */
} vxm_status;

/* ---- POD mirrors of the reference types -------------------------------- */
/* GridIndex (core/indexing.hpp:33-39): lexicographic (x, y, z) order. */
typedef struct { int32_t x, y, z; } vxm_grid_index;

/* TsdfVoxel (core/voxels.hpp:22-26), 8 bytes. */
typedef struct { float distance, weight; } vxm_tsdf_voxel;

/* OccupancyVoxel (core/voxels.hpp:28-32), 4 bytes: log-odds, 0 = unobserved prior. */
typedef struct { float log_odds; } vxm_occupancy_voxel;

/* ColorVoxel (core/voxels.hpp:34-41), 8 bytes. */
typedef struct {
  uint8_t r, g, b, reserved;
  float weight;
} vxm_color_voxel;

/* EsdfVoxel (core/voxels.hpp:48-68), 12 bytes, same byte layout. */
typedef struct {
  int32_t squared_distance;
  int16_t parent_x, parent_y, parent_z;
  uint8_t flags; /* 1 observed, 2 site, 4 inside */
  uint8_t reserved;
} vxm_esdf_voxel;

enum { VXM_ESDF_OBSERVED = 1, VXM_ESDF_SITE = 2, VXM_ESDF_INSIDE = 4 };
enum { VXM_VOXELS_PER_SIDE = 8, VXM_VOXELS_PER_BLOCK = 512 };

/* Layer voxel type: Layer<TsdfVoxel>, Layer<EsdfVoxel>, Layer<OccupancyVoxel>. */
typedef enum {
  VXM_LAYER_TSDF = 0,
  VXM_LAYER_ESDF = 1,
  VXM_LAYER_OCCUPANCY = 2,
  VXM_LAYER_COLOR = 3
} vxm_layer_type;

/* CameraIntrinsics (sensor/camera.hpp:24-31). */
typedef struct {
  double fu, fv, cu, cv;
  int32_t width, height;
  double max_depth;
} vxm_camera;

/* LidarIntrinsics (sensor/lidar.hpp:27-38). */
typedef struct {
  int32_t num_azimuth, num_elevation;
  double azimuth_start, elevation_start, azimuth_fov, elevation_fov;
  double min_range, max_range;
} vxm_lidar;

/* Pose (sensor/pose.hpp:30-60): p_parent = R * p_child + t, R row-major. */
typedef struct { double R[9]; double t[3]; } vxm_pose;

enum { VXM_WEIGHT_CONSTANT = 0, VXM_WEIGHT_INVERSE_SQUARE = 1 };
enum { VXM_SAMPLE_NEAREST = 0, VXM_SAMPLE_LINEAR = 1 };

/* IntegratorConfig (integrate/config.hpp:38-56). */
typedef struct {
  double truncation;
  float max_weight;
  int32_t weighting;
  double max_integration_distance;
  int32_t camera_sample;
  int32_t lidar_sample;
  float max_sample_gap;
  int32_t view_pixel_subsample;
  float hit_log_odds, miss_log_odds, log_odds_min, log_odds_max;
  int32_t parallel; /* accepted, ignored */
} vxm_integrator_config;

/* ViewConfig (sensor/view.hpp:27-31). */
typedef struct {
  double max_integration_distance;
  double truncation;
  int32_t pixel_subsample;
} vxm_view_config;

/* EsdfConfig (esdf/integrator.hpp:30-40). */
typedef struct {
  double site_threshold;
  float occupied_log_odds_threshold;
  double max_distance;
  int32_t parallel; /* accepted, ignored */
} vxm_esdf_config;

/* QueryConfig (query/query.hpp:41-49) and QueryResult (:30-39). */
typedef struct { int32_t interpolate; int32_t parallel; } vxm_query_config;
typedef struct {
  int32_t known;
  int32_t pad_;
  double distance;
  double gradient[3];
} vxm_query_result;

/* Reference defaults (config.hpp, esdf/integrator.hpp, query.hpp). */
void vxm_integrator_config_default(vxm_integrator_config* cfg);
void vxm_esdf_config_default(vxm_esdf_config* cfg);
void vxm_query_config_default(vxm_query_config* cfg);

/* ---- opaque handles ---------------------------------------------------- */
typedef struct vxm_context vxm_context;     /* device + stream + scratch       */
typedef struct vxm_layer vxm_layer;         /* Layer<V> (core/layer.hpp:47-125) */
typedef struct vxm_blocklist vxm_blocklist; /* std::vector<GridIndex> result    */
typedef struct vxm_esdf_state vxm_esdf_state; /* EsdfUpdateState (esdf/integrator.hpp:67-74) */

const char* vxm_last_error(void);
const char* vxm_version(void);

/* Context: one CUDA device + one stream.  Calls on a context are serialized. */
vxm_status vxm_context_create(int device, vxm_context** out);
void vxm_context_destroy(vxm_context* ctx);
vxm_status vxm_context_synchronize(vxm_context* ctx);
/* Block-coordinate sharding: this context owns blocks with
 * floor(g.x / slab) mod world == rank.  world = 1 (default) owns everything. */
vxm_status vxm_context_set_shard(vxm_context* ctx, int rank, int world, int slab);
/* Kernel launches issued by this context since creation (bench evidence). */
uint64_t vxm_context_launch_count(const vxm_context* ctx);
/* The context's cudaStream_t (as an integer handle) for external event timing. */
uint64_t vxm_context_stream(const vxm_context* ctx);

/* Work counters accumulated by the device passes (algorithmic-bytes model of
 * SURVEY §8(d)); reset with vxm_context_reset_stats. */
typedef struct {
  uint64_t integrate_calls, candidate_blocks, new_blocks, changed_blocks;
  uint64_t voxels_read, voxels_updated, depth_pixels;
  uint64_t esdf_calls, esdf_blocks, effective_blocks, esdf_new_blocks;
  uint64_t lower_rounds, dirty_blocks_after_round1, pair_exchanges, compared_blocks;
  uint64_t reserved[8];
} vxm_stats;
vxm_status vxm_context_stats(vxm_context* ctx, vxm_stats* out);
void vxm_context_reset_stats(vxm_context* ctx);
/* Per-kernel CUDA-event timing on the context stream (off by default). */
vxm_status vxm_context_set_profiling(vxm_context* ctx, int enable);
/* Accumulated device time (ms) and launch count of one instrumented kernel
 * ("k_integrate", "k_lower", "k_dilate_alloc", "k_rays", "k_mark", ...). */
vxm_status vxm_context_kernel_time(vxm_context* ctx, const char* kernel, double* ms,
                                   uint64_t* launches);
/* Diagnostics (parity tests): the LiDAR projection's angles exactly as
 * k_integrate computes them for p = (x, y, z) in the sensor frame —
 * azimuth = atan2(y, x) and polar = acos(z / |p|) of LidarIntrinsics::project
 * (lidar.hpp:43-55) — for n points (xyz: n x 3 doubles, host memory). */
vxm_status vxm_diag_lidar_angles(vxm_context* ctx, const double* xyz, uint64_t n, double* azimuth,
                                 double* polar);
void vxm_context_reset_kernel_times(vxm_context* ctx);

/* ---- block lists ------------------------------------------------------- */
vxm_status vxm_blocklist_create(vxm_context* ctx, vxm_blocklist** out);
void vxm_blocklist_destroy(vxm_blocklist* list);
/* Host view (downloads if the list was produced by a *_device call). */
vxm_status vxm_blocklist_host(vxm_blocklist* list, const vxm_grid_index** data, uint64_t* n);
/* Replace contents with a host array (uploads). */
vxm_status vxm_blocklist_assign(vxm_blocklist* list, const vxm_grid_index* data, uint64_t n);

/* ---- layers (core/layer.hpp) -------------------------------------------- */
/* Layer(double voxel_size, size_t max_blocks) — layer.hpp:52-57. */
vxm_status vxm_layer_create(vxm_context* ctx, vxm_layer_type type, double voxel_size,
                            uint64_t max_blocks, vxm_layer** out);
void vxm_layer_destroy(vxm_layer* layer);
double vxm_layer_voxel_size(const vxm_layer* layer);
/* num_blocks() — layer.hpp:61. */
vxm_status vxm_layer_num_blocks(vxm_layer* layer, uint64_t* out);
/* Pre-sizes the device block pool for n blocks (capped at max_blocks) so that
 * later frames do not pay pool growth; no effect on results.  (The reference
 * allocates per block; nvblox pre-sizes its GPU hash the same way.) */
vxm_status vxm_layer_reserve(vxm_layer* layer, uint64_t n_blocks);
/* has_block() for a batch of keys — layer.hpp:63. out[i] = 0/1. */
vxm_status vxm_layer_has_blocks(vxm_layer* layer, const vxm_grid_index* keys, uint64_t n,
                                uint8_t* out);
/* sorted_indices() + block bytes — layer.hpp:109-117 (and block_ptr()).
 * keys_out gets num_blocks sorted keys; voxels_out (may be NULL) gets the
 * blocks' bytes in the same order (512 voxels each). */
vxm_status vxm_layer_export(vxm_layer* layer, vxm_grid_index* keys_out, void* voxels_out,
                            uint64_t capacity);
/* Read specific blocks (block_ptr) — missing blocks are zero-filled, found[i]=0. */
vxm_status vxm_layer_read_blocks(vxm_layer* layer, const vxm_grid_index* keys, uint64_t n,
                                 void* voxels_out, uint8_t* found);
/* get_or_allocate + overwrite bytes (host writes through block_ptr). */
vxm_status vxm_layer_write_blocks(vxm_layer* layer, const vxm_grid_index* keys, uint64_t n,
                                  const void* voxels);
/* clone() — layer.hpp:98-105. */
vxm_status vxm_layer_clone(vxm_layer* src, vxm_layer** out);

/* ---- view candidates (sensor/view.hpp:38-48, view.cpp:61-111) ---------- */
vxm_status vxm_blocks_in_view_camera(vxm_context* ctx, const vxm_pose* T_LS, const vxm_camera* cam,
                                     const float* depth, int width, int height, double block_size,
                                     const vxm_view_config* cfg, vxm_blocklist* out);
vxm_status vxm_blocks_in_view_lidar(vxm_context* ctx, const vxm_pose* T_LS, const vxm_lidar* lidar,
                                    const float* depth, int width, int height, double block_size,
                                    const vxm_view_config* cfg, vxm_blocklist* out);

/* ---- page-locked host buffers ------------------------------------------- */
/* Host memory the DMA engines read at full PCIe rate (cudaHostAlloc), for
 * depth / color frames handed to the host-buffer entry points (any host
 * pointer works; pageable or differently registered memory uploads slower). */
vxm_status vxm_host_alloc(uint64_t bytes, void** out);
void vxm_host_free(void* p);

/* ---- depth integration (integrate/integrator.hpp:36-55) ----------------- */
/* integrate_depth(Layer<TsdfVoxel>&, DepthImage, Pose T_LS, CameraIntrinsics,
 * IntegratorConfig) — integrator.cpp:162-168; with an occupancy layer, the
 * Layer<OccupancyVoxel>& overload (integrator.cpp:176-189: occupancy_update,
 * updates.hpp:59-72).  The layer's type selects the overload.  changed_out
 * receives the sorted changed-block list.  Validates before mutating
 * (integrator.cpp:26-34). */
vxm_status vxm_integrate_depth_camera(vxm_layer* layer, const float* depth, int width, int height,
                                      const vxm_pose* T_LS, const vxm_camera* cam,
                                      const vxm_integrator_config* cfg, vxm_blocklist* changed_out);
/* LidarIntrinsics overload — integrator.cpp:169-175. */
vxm_status vxm_integrate_depth_lidar(vxm_layer* layer, const float* depth, int width, int height,
                                     const vxm_pose* T_LS, const vxm_lidar* lidar,
                                     const vxm_integrator_config* cfg, vxm_blocklist* changed_out);
/* Device-resident variants: depth is a device pointer, changed_out stays on
 * the device (read it with vxm_blocklist_host).  Errors surface at
 * vxm_context_synchronize(). */
vxm_status vxm_integrate_depth_camera_device(vxm_layer* layer, const float* depth_dev, int width,
                                             int height, const vxm_pose* T_LS,
                                             const vxm_camera* cam,
                                             const vxm_integrator_config* cfg,
                                             vxm_blocklist* changed_out);
vxm_status vxm_integrate_depth_lidar_device(vxm_layer* layer, const float* depth_dev, int width,
                                            int height, const vxm_pose* T_LS,
                                            const vxm_lidar* lidar,
                                            const vxm_integrator_config* cfg,
                                            vxm_blocklist* changed_out);

/* ---- color fusion (integrate/integrator.hpp:57-66, integrator.cpp:191-273) -- */
/* integrate_color(Layer<ColorVoxel>&, ColorImage, DepthImage, Pose T_LS,
 * CameraIntrinsics, const Layer<TsdfVoxel>&, IntegratorConfig): fuses an RGB
 * image (host, row-major width x height x 3) into the voxels of the TSDF
 * surface band (weight > 0, |distance| <= truncation); color blocks are
 * allocated only where the TSDF block holds band voxels.  The depth image
 * (host) selects the candidate blocks.  Errors as the reference (before any
 * mutation): degenerate pose, color size != intrinsics, depth size mismatch. */
vxm_status vxm_integrate_color(vxm_layer* color, const uint8_t* rgb, int width, int height,
                               const float* depth, int depth_width, int depth_height,
                               const vxm_pose* T_LS, const vxm_camera* cam, vxm_layer* tsdf,
                               const vxm_integrator_config* cfg, vxm_blocklist* changed_out);

/* ---- meshing (mesh/marching_cubes.hpp:24-78, mesh_layer.hpp, ply.hpp) ---- */
/* MeshConfig (marching_cubes.hpp:24-33). */
typedef struct {
  float min_weight; /* corners with weight below this leave a cube inactive */
  int32_t parallel; /* accepted, ignored */
} vxm_mesh_config;
void vxm_mesh_config_default(vxm_mesh_config* cfg);
/* MeshLayer (mesh_layer.hpp:27-66): per-block meshes, host-resident (the
 * device computes them).  A block view's arrays stay valid until the block is
 * re-meshed or the layer destroyed. */
typedef struct vxm_mesh_layer vxm_mesh_layer;
typedef struct {
  uint64_t n_vertices, n_triangles, n_colors; /* n_colors: 0 or n_vertices */
  const float* vertices;     /* 3 per vertex, metres, layer frame */
  const float* normals;      /* 3 per vertex, unit, along +gradient */
  const uint8_t* colors;     /* 3 per vertex (when meshed with a color layer) */
  const uint32_t* triangles; /* 3 block-local vertex indices per triangle */
} vxm_mesh_block_view;
vxm_status vxm_mesh_layer_create(vxm_context* ctx, double voxel_size, vxm_mesh_layer** out);
void vxm_mesh_layer_destroy(vxm_mesh_layer* mesh);
double vxm_mesh_layer_voxel_size(const vxm_mesh_layer* mesh);
uint64_t vxm_mesh_layer_num_blocks(const vxm_mesh_layer* mesh);
/* sorted_indices (mesh_layer.hpp:47-55) into keys_out[capacity]. */
vxm_status vxm_mesh_layer_sorted_indices(const vxm_mesh_layer* mesh, vxm_grid_index* keys_out,
                                         uint64_t capacity);
/* block_ptr (mesh_layer.hpp:37-40): *found = 0 when absent. */
vxm_status vxm_mesh_layer_block(const vxm_mesh_layer* mesh, const vxm_grid_index* g,
                                vxm_mesh_block_view* out, int* found);
vxm_status vxm_mesh_layer_erase(vxm_mesh_layer* mesh, const vxm_grid_index* g);
/* mesh_block (marching_cubes.cpp:95-209), stored into mesh at g (as
 * get_or_create(g) = mesh_block(...)).  VXM_ERR_INVALID_ARGUMENT when the TSDF
 * block is not allocated.  color may be NULL (no vertex colors). */
vxm_status vxm_mesh_block(vxm_mesh_layer* mesh, vxm_layer* tsdf, const vxm_grid_index* g,
                          const vxm_mesh_config* cfg, vxm_layer* color);
/* update_mesh (marching_cubes.cpp:211-242): re-meshes every allocated block of
 * updated U its -x/-y/-z neighbours; remeshed_out gets those targets (sorted). */
vxm_status vxm_update_mesh(vxm_mesh_layer* mesh, vxm_layer* tsdf, const vxm_grid_index* updated,
                           uint64_t n, const vxm_mesh_config* cfg, vxm_layer* color,
                           vxm_blocklist* remeshed_out);
vxm_status vxm_update_mesh_list(vxm_mesh_layer* mesh, vxm_layer* tsdf, vxm_blocklist* updated,
                                const vxm_mesh_config* cfg, vxm_layer* color,
                                vxm_blocklist* remeshed_out);
/* save_mesh_ply (ply.cpp:33-105): binary little-endian PLY, blocks in sorted
 * order, byte-identical to the reference's.  VXM_ERR_IO when it cannot write. */
vxm_status vxm_save_mesh_ply(const vxm_mesh_layer* mesh, const char* path);

/* ---- replay (io/pipeline.hpp:27-72, pipeline.cpp:54-148) ------------------- */
/* ReplayConfig (pipeline.hpp:27-36). */
typedef struct {
  double voxel_size;
  int32_t update_every;  /* derive ESDF + mesh every this many frames (+ after the last) */
  vxm_integrator_config integrator;
  vxm_esdf_config esdf;
  int32_t use_occupancy; /* fuse occupancy instead of the TSDF (pipeline.cpp:73-77, 95-101) */
  int32_t with_color;    /* fuse color (camera datasets only, pipeline.cpp:111-117) */
  vxm_mesh_config mesh;
} vxm_replay_config;
/* FrameTiming: wall-clock ms per stage of one frame (0 when skipped). */
typedef struct {
  int32_t frame;
  double tsdf_ms, color_ms, esdf_ms, mesh_ms;
} vxm_frame_timing;
/* ReplayResult's LayerCake (pipeline.hpp:54-57): the layers replay created
 * (NULL when never required, as the reference's lazily created layers). */
typedef struct {
  vxm_layer* source;     /* TSDF, or occupancy with use_occupancy */
  vxm_layer* esdf;
  vxm_layer* color;
  vxm_mesh_layer* mesh;
} vxm_replay_result;
/* make_replay_config (pipeline.cpp:46-52): truncation 4 voxels, site threshold 1. */
void vxm_replay_config_make(double voxel_size, vxm_replay_config* out);
/* replay (pipeline.cpp:54-148) over in-memory frames: n_frames depth images
 * (host, n_frames x height x width, row-major) with their poses, and for the
 * camera optionally their color images (host, n_frames x height x width x 3, or
 * NULL: frames without color).  Integrates every frame (and its color with
 * with_color) and, every update_every frames and after the last one, folds the
 * blocks changed since the previous update into the ESDF and (TSDF source) the
 * mesh.  timings has n_frames entries.  Errors as the reference: no frames,
 * update_every < 1, color with occupancy or LiDAR -> VXM_ERR_INVALID_ARGUMENT. */
vxm_status vxm_replay_camera(vxm_context* ctx, const vxm_replay_config* cfg, const vxm_camera* cam,
                             int n_frames, int width, int height, const float* depth,
                             const uint8_t* rgb, const vxm_pose* poses, vxm_replay_result* out,
                             vxm_frame_timing* timings);
vxm_status vxm_replay_lidar(vxm_context* ctx, const vxm_replay_config* cfg, const vxm_lidar* lidar,
                            int n_frames, int width, int height, const float* depth,
                            const vxm_pose* poses, vxm_replay_result* out,
                            vxm_frame_timing* timings);

/* ---- snapshots (core/serialization.hpp:29-35, FORMATS.md "VXLF") -------- */
/* save_snapshot (serialization.cpp:88-110): VXLF v1, little-endian; layers in
 * the reference's order (tsdf, then esdf), blocks in sorted GridIndex order, so
 * equal maps give byte-identical files.  Either layer may be NULL; both must
 * have `voxel_size`.  Errors: VXM_ERR_IO (cannot open / write failed). */
vxm_status vxm_snapshot_save(const char* path, double voxel_size, vxm_layer* tsdf, vxm_layer* esdf);
/* load_snapshot (serialization.cpp:112-158): creates the layers found in the
 * file on `ctx` (NULL when absent).  VXM_ERR_IO on bad magic, unsupported
 * version, invalid voxel size, truncated payload, voxel size mismatch, unknown
 * layer name, and for the occupancy / color layers this library does not
 * implement (out of scope). */
vxm_status vxm_snapshot_load(vxm_context* ctx, const char* path, double* voxel_size_out,
                             vxm_layer** tsdf_out, vxm_layer** esdf_out);
/* The same over the LayerCake's tsdf / occupancy / color / esdf layers
 * (layer_cake.hpp:29-33; written in the reference's order tsdf, occupancy,
 * color, esdf).  Any layer argument may be NULL; a NULL out pointer makes a
 * file holding that layer fail with VXM_ERR_IO. */
vxm_status vxm_snapshot_save_layers(const char* path, double voxel_size, vxm_layer* tsdf,
                                    vxm_layer* occupancy, vxm_layer* color, vxm_layer* esdf);
vxm_status vxm_snapshot_load_layers(vxm_context* ctx, const char* path, double* voxel_size_out,
                                    vxm_layer** tsdf_out, vxm_layer** occupancy_out,
                                    vxm_layer** color_out, vxm_layer** esdf_out);

/* ---- block-sharded ESDF ------------------------------------ */
/* One update_esdf (esdf/integrator.cpp:365-413) over a map sharded by block x:
 * shard p of n_shards (its own context — same GPU or another — configured with
 * vxm_context_set_shard(ctx, p, n_shards, slab)) owns the blocks with
 * floor(x / slab) mod n_shards == p, holds them in esdf[p] / tsdf[p] and passes
 * its changed TSDF list updated[p].  Each lowering round the shards exchange
 * their slab-boundary x-faces (peer copies) and agree on termination.  The union
 * of esdf[] and of changed_out[] equals update_esdf over the union map,
 * bit-for-bit. */
vxm_status vxm_update_esdf_sharded(int n_shards, vxm_layer* const* esdf, vxm_layer* const* tsdf,
                                   vxm_blocklist* const* updated, const vxm_esdf_config* cfg,
                                   vxm_blocklist* const* changed_out);

/* The same update as steps, for one process per shard (the caller moves the
 * exchange buffers between neighbours and reduces the flags / counts, e.g. with
 * NCCL through torch.distributed — paper_2311_00626_b200/dist.py):
 *   begin(union of all shards' updated lists) -> local any_update;   OR-reduce
 *   if the OR is set: plan -> n_boundary;   all-gather n_boundary
 *     exchange_buffers(n of the -x neighbour (rank-1), n of the +x one (rank+1))
 *     for round = 1, 2, ...: sweep(round); send `send` to both neighbours, receive
 *       the -x neighbour's into recv_left and the +x one's into recv_right;
 *       border(round) -> next_dirty;  sum-reduce; stop at 0
 *   finish(lowered = the OR) -> changed blocks; frees the handle.
 * sweep() and border(next_dirty = NULL) only ENQUEUE on the context stream
 * (vxm_context_stream): a collective enqueued on that stream after sweep()
 * sees the packed send buffer, and border() after it sees the received
 * snapshots, without a host synchronisation.  border() with a non-NULL
 * next_dirty also waits and returns the count; next_count() gives the device
 * address (uint32) that border(round) writes the count to, for an on-device
 * reduction. */
typedef struct vxm_shard_update vxm_shard_update;
vxm_status vxm_shard_update_begin(vxm_layer* esdf, vxm_layer* tsdf, vxm_blocklist* updated_union,
                                  const vxm_esdf_config* cfg, vxm_shard_update** out,
                                  int* local_any_update);
vxm_status vxm_shard_update_plan(vxm_shard_update* su, uint32_t* n_boundary);
vxm_status vxm_shard_update_exchange_buffers(vxm_shard_update* su, uint32_t n_left, uint32_t n_right,
                                             void** send, uint64_t* send_bytes, void** recv_left,
                                             uint64_t* recv_left_bytes, void** recv_right,
                                             uint64_t* recv_right_bytes);
vxm_status vxm_shard_update_sweep(vxm_shard_update* su, uint32_t round);
vxm_status vxm_shard_update_border(vxm_shard_update* su, uint32_t round, uint32_t* next_dirty);
vxm_status vxm_shard_update_next_count(vxm_shard_update* su, uint32_t round, void** device_u32);
/* Fused alternative to the round loop above (one persistent kernel per rank,
 * the faces written straight into the neighbours' receive buffers over peer
 * memory, system-scope flags and a count board for termination — no host step
 * per round): after exchange_buffers(), ipc_handles() writes this rank's three
 * CUDA IPC handles (3 x 64 bytes; it also clears the rank's mailbox, so every
 * rank must call it before the all-gather, which is the barrier); the caller
 * all-gathers them (world x 192 bytes in rank order) into lower_fused(), which
 * enqueues the whole lowering; then finish(lowered = 1).  ranks_on_device: the
 * ranks sharing this GPU (their kernels split its SMs; all ranks' kernels must
 * run concurrently).  2..8 ranks. */
vxm_status vxm_shard_update_ipc_handles(vxm_shard_update* su, void* handles_out);
vxm_status vxm_shard_update_lower_fused(vxm_shard_update* su, const void* all_handles, int ranks_on_device);
vxm_status vxm_shard_update_finish(vxm_shard_update* su, int lowered, vxm_blocklist* changed_out);
void vxm_shard_update_destroy(vxm_shard_update* su);

/* ---- fused frame update (replay pipeline step) ---------------------------- */
/* One frame of the replay pipeline (pipeline.cpp:95-108: integrate the frame,
 * then update the ESDF from its changed blocks) on a device-resident depth
 * image, with ONE host round trip for both halves.  Same results as
 * vxm_integrate_depth_*_device followed by vxm_update_esdf_list; both changed
 * lists stay on the device.  `esdf` may be NULL (integration only; ecfg and
 * esdf_changed are then ignored).  The ESDF half's argument errors (layer
 * types, voxel-size mismatch) are reported before the TSDF is touched. */
vxm_status vxm_update_frame_camera_device(vxm_layer* tsdf, vxm_layer* esdf, const float* depth_dev,
                                          int width, int height, const vxm_pose* T_LS,
                                          const vxm_camera* cam, const vxm_integrator_config* icfg,
                                          const vxm_esdf_config* ecfg, vxm_blocklist* tsdf_changed,
                                          vxm_blocklist* esdf_changed);
vxm_status vxm_update_frame_lidar_device(vxm_layer* tsdf, vxm_layer* esdf, const float* depth_dev,
                                         int width, int height, const vxm_pose* T_LS,
                                         const vxm_lidar* lidar, const vxm_integrator_config* icfg,
                                         const vxm_esdf_config* ecfg, vxm_blocklist* tsdf_changed,
                                         vxm_blocklist* esdf_changed);

/* ---- ESDF (esdf/integrator.hpp:81-120) ---------------------------------- */
/* update_esdf(Layer<EsdfVoxel>&, const Layer<TsdfVoxel>&, updated, EsdfConfig)
 * — esdf/integrator.cpp:365-413, 567-572.  `tsdf` may be an occupancy layer:
 * the Layer<OccupancyVoxel> overload (:574-579, OccupancyClassifier :200-266).
 * The same holds for vxm_update_esdf_list, vxm_esdf_mark_sites and the
 * frame step (vxm_update_frame_*); the sharded update takes TSDF sources. */
vxm_status vxm_update_esdf(vxm_layer* esdf, vxm_layer* tsdf, const vxm_grid_index* updated,
                           uint64_t n, const vxm_esdf_config* cfg, vxm_blocklist* changed_out);
/* Same, with the updated list taken from a (device-resident) block list,
 * e.g. the changed_out of a previous integrate call. */
vxm_status vxm_update_esdf_list(vxm_layer* esdf, vxm_layer* tsdf, vxm_blocklist* updated,
                                const vxm_esdf_config* cfg, vxm_blocklist* changed_out);

/* Phase API (esdf/integrator.hpp:76-107), used directly by the reference's tests. */
vxm_status vxm_esdf_state_create(vxm_esdf_state** out);
void vxm_esdf_state_destroy(vxm_esdf_state* st);
/* Which: 0 indices_to_update, 1 indices_to_clear, 2 cleared_indices. */
vxm_status vxm_esdf_state_get(vxm_esdf_state* st, int which, const vxm_grid_index** data,
                              uint64_t* n);
vxm_status vxm_esdf_state_set(vxm_esdf_state* st, int which, const vxm_grid_index* data,
                              uint64_t n);
/* mark_sites — esdf/integrator.cpp:417-431 (TSDF or occupancy source). changed is appended. */
vxm_status vxm_esdf_mark_sites(vxm_layer* esdf, vxm_layer* tsdf, const vxm_grid_index* updated,
                               uint64_t n, const vxm_esdf_config* cfg, vxm_esdf_state* st,
                               vxm_blocklist* changed);
/* clear_invalid — esdf/integrator.cpp:433-486. */
vxm_status vxm_esdf_clear_invalid(vxm_layer* esdf, const vxm_esdf_config* cfg, vxm_esdf_state* st,
                                  vxm_blocklist* changed);
/* lower_esdf — esdf/integrator.cpp:488-565; *rounds receives the round count. */
vxm_status vxm_esdf_lower(vxm_layer* esdf, vxm_esdf_state* st, const vxm_esdf_config* cfg,
                          vxm_blocklist* changed, int* rounds);

/* ---- queries (query/query.hpp:59-62, query.cpp:147-161) ----------------- */
vxm_status vxm_query_batch(vxm_layer* esdf, const double* xyz, uint64_t n, int want_gradient,
                           const vxm_query_config* cfg, vxm_query_result* out);

/* ---- host utilities ----------------------------------------------------- */
/* Pose::valid() (pose.hpp:42-50) and Pose::inverse() (:52). */
int vxm_pose_valid(const vxm_pose* T);
void vxm_pose_inverse(const vxm_pose* T, vxm_pose* out);

#ifdef __cplusplus
}
#endif
#endif /* VOXMAP_B200_H_ */
