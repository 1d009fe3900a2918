/*
 * voxmap_b200 synthetic inputs (host only, OpenMP): analytic SDF scenes,
 * sphere-traced depth frames and orbit trajectories, following the
 * reference's input generators so benchmarks and tests can build the
 * BASELINE.json configurations without the reference:
 *   make_scene      proj/src/io/scene.cpp:124-144  ("sphere_in_box", "room", "corridor")
 *   render_depth    proj/src/io/render.cpp:43-86
 *   orbit_pose      proj/src/io/dataset.cpp:334-367
 * plus builder-defined scenes for configs the reference has no scene for
 * ("lidar_yard": C3, 200 m ground plane + boxes; "building": C4 multi-room)
 * and the SphereWorld-style dense TSDF volume of config C5
 * (proj/tests/fixtures.hpp:34-98).
 */
#ifndef VOXMAP_B200_SYNTH_H_
#define VOXMAP_B200_SYNTH_H_

#include "voxmap_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct vxm_scene vxm_scene;

vxm_status vxm_synth_scene_create(const char* name, vxm_scene** out);
void vxm_synth_scene_destroy(vxm_scene* s);
/* bbox_min[3], bbox_max[3] */
void vxm_synth_scene_bbox(const vxm_scene* s, double* bbox6);
double vxm_synth_scene_sdf(const vxm_scene* s, const double p[3]);
vxm_status vxm_synth_orbit_pose(const vxm_scene* s, int lidar, int frame, int total,
                                vxm_pose* out);
/* out: height x width floats, row-major */
vxm_status vxm_synth_render_camera(const vxm_scene* s, const vxm_pose* T_WS, const vxm_camera* cam,
                                   float* out);
vxm_status vxm_synth_render_lidar(const vxm_scene* s, const vxm_pose* T_WS, const vxm_lidar* li,
                                  float* out);
/* Dense SphereWorld TSDF (C5): side_voxels^3 voxels (side multiple of 8),
 * n_spheres drawn from std::mt19937(seed) as (cx, cy, cz, r) with
 * cx,cy,cz ~ U[0.15E, 0.85E], r ~ U[0.08E, 0.25E], E = side * vs.  Writes
 * (side/8)^3 block keys (x-slowest order) and their voxels (distance =
 * float(clamp(sdf, +-trunc)), weight = 1).  keys may be NULL. */
vxm_status vxm_synth_sphere_world(int side_voxels, double vs, double trunc, unsigned seed,
                                  int n_spheres, vxm_grid_index* keys, vxm_tsdf_voxel* voxels);

#ifdef __cplusplus
}
#endif
#endif
