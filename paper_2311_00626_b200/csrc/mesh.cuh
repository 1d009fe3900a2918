// Mesh layer (host container of per-block meshes, as the reference's
// MeshLayer, include/voxmap/mesh/mesh_layer.hpp:27-66) and the device
// marching-cubes driver (mesh.cu).
#pragma once

#include <map>
#include <vector>

#include "runtime.cuh"

namespace vxm {

// MeshBlock (mesh_layer.hpp:16-25): block-local vertex indices.
struct MeshBlockH {
  std::vector<float> vertices;     // 3 per vertex (metres, layer frame)
  std::vector<float> normals;      // 3 per vertex
  std::vector<uint8_t> colors;     // 3 per vertex, or empty (no color layer)
  std::vector<uint32_t> triangles; // 3 per triangle
};

struct MeshLayerH {
  Context* ctx = nullptr;
  double vs = 0.0;
  std::map<uint64_t, MeshBlockH> blocks;  // packed-key order == GridIndex order
};

// update_mesh (marching_cubes.cpp:211-242): targets = updated U {-x, -y, -z
// neighbours}, restricted to allocated TSDF blocks, sorted; every target is
// re-meshed (mesh_block, :95-209) and stored.  Returns the targets (host).
std::vector<vxm_grid_index> run_update_mesh(MeshLayerH* M, Layer* T, BlockList* updated,
                                            float min_weight, Layer* color);
// mesh_block for an explicit sorted unique list of allocated blocks.
void run_mesh_blocks(MeshLayerH* M, Layer* T, BlockList* targets, float min_weight, Layer* color);

// color.cu — integrate_color (integrate/integrator.cpp:191-273)
void run_integrate_color(Layer* C, Layer* T, const uint8_t* rgb_host, const ViewArgs& va,
                         const vxm_integrator_config& cfg, BlockList* changed_out);

}  // namespace vxm
