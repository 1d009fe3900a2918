/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle for the per-frame map update.
 *
 * A plain-C restatement of the reference's hot path (SURVEY.md §8(a) rows
 * a1-a11), written from the reference sources' semantics with file:line
 * citations into /root/reference/proj.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load it; the product (libvoxmap_b200)
 * never links or calls it.
 *
 * Parity pinning: the restatement is checked bit-for-bit against the
 * reference's own sources compiled in oracle/_ref (tests/test_oracle_vs_ref.py)
 * and against the reference tests' known-answer vectors (tests/golden/).
 * The reference's Eigen association order is pinned by oracle/eigen_shim
 * (Eigen3 is absent from this image); see DESIGN.md §Oracle.
 */
#ifndef VOXMAP_ORACLE_H_
#define VOXMAP_ORACLE_H_

#include <stdint.h>

#include "voxmap_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct vxo_layer vxo_layer;
typedef struct vxo_state vxo_state;

const char* vxo_last_error(void);
void vxo_free(void* p);

int vxo_layer_create(int type, double voxel_size, uint64_t max_blocks, vxo_layer** out);
void vxo_layer_destroy(vxo_layer* L);
uint64_t vxo_layer_num_blocks(const vxo_layer* L);
/* Sorted keys (+ block bytes when voxels != NULL). */
int vxo_layer_export(const vxo_layer* L, vxm_grid_index* keys, void* voxels);
int vxo_layer_write_blocks(vxo_layer* L, const vxm_grid_index* keys, uint64_t n,
                           const void* voxels);

/* Host-side pose helpers with the pinned association order. */
int vxo_pose_valid(const vxm_pose* T);
void vxo_pose_inverse(const vxm_pose* T, vxm_pose* out);

/* Results are malloc'ed arrays; free with vxo_free. */
int vxo_blocks_in_view_camera(const vxm_pose* T, const vxm_camera* cam, const float* depth,
                              int w, int h, double block_size, const vxm_view_config* cfg,
                              vxm_grid_index** out, uint64_t* n);
int vxo_blocks_in_view_lidar(const vxm_pose* T, const vxm_lidar* li, const float* depth, int w,
                             int h, double block_size, const vxm_view_config* cfg,
                             vxm_grid_index** out, uint64_t* n);
int vxo_integrate_camera(vxo_layer* L, const float* depth, int w, int h, const vxm_pose* T,
                         const vxm_camera* cam, const vxm_integrator_config* cfg,
                         vxm_grid_index** out, uint64_t* n);
int vxo_integrate_lidar(vxo_layer* L, const float* depth, int w, int h, const vxm_pose* T,
                        const vxm_lidar* li, const vxm_integrator_config* cfg,
                        vxm_grid_index** out, uint64_t* n);

vxo_state* vxo_state_create(void);
void vxo_state_destroy(vxo_state* s);
int vxo_state_get(vxo_state* s, int which, vxm_grid_index** out, uint64_t* n);
int vxo_state_set(vxo_state* s, int which, const vxm_grid_index* k, uint64_t n);
int vxo_mark_sites(vxo_layer* esdf, const vxo_layer* tsdf, const vxm_grid_index* upd,
                   uint64_t nu, const vxm_esdf_config* cfg, vxo_state* s, vxm_grid_index** out,
                   uint64_t* n);
int vxo_clear_invalid(vxo_layer* esdf, const vxm_esdf_config* cfg, vxo_state* s,
                      vxm_grid_index** out, uint64_t* n);
int vxo_lower_esdf(vxo_layer* esdf, vxo_state* s, const vxm_esdf_config* cfg, int* rounds,
                   vxm_grid_index** out, uint64_t* n);
int vxo_update_esdf(vxo_layer* esdf, const vxo_layer* tsdf, const vxm_grid_index* upd,
                    uint64_t nu, const vxm_esdf_config* cfg, vxm_grid_index** out, uint64_t* n);
int vxo_query_batch(const vxo_layer* esdf, const double* xyz, uint64_t n, int want_gradient,
                    const vxm_query_config* cfg, vxm_query_result* out);

#ifdef __cplusplus
}
#endif
#endif
