"""B200-native per-frame map update (nvblox / voxmap hot path).

Block allocation -> TSDF / occupancy projective integration -> ESDF -> queries, as
hand-written sm_100a CUDA behind the C-ABI in include/voxmap_b200.h.  The
Python API mirrors the reference's C++ mapper API (see voxmap.py).
"""
from .voxmap import (BlockList, CameraIntrinsics, Context, EsdfConfig, EsdfLayer,  # noqa: F401
                     EsdfUpdateState, IntegratorConfig, InvalidArgumentError, InvalidPoseError,
                     LidarIntrinsics, MapCapacityError, Pose, TsdfLayer, VoxmapCudaError,
                     VoxmapError, blocks_in_view, clear_invalid, default_camera_intrinsics,
                     default_context, default_lidar_intrinsics, esdf_distance, integrate_depth,
                     integrate_depth_device, lib, lower_esdf, mark_sites, query_batch,
                     update_esdf, update_esdf_device, update_frame_device,
                     IoError, save_snapshot, load_snapshot, update_esdf_sharded,
                     make_replay_config, replay, write_timing_csv, OccupancyLayer,
                     ColorLayer, MeshLayer, MeshBlock, integrate_color, mesh_block, update_mesh,
                     save_mesh_ply, replay_cake, HostBuffer, pinned_like,
                     linear_voxel_index, voxel_index_from_linear, global_voxel_index,
                     block_of_global_voxel, local_voxel_of_global, position_to_global_voxel,
                     position_to_indices, voxel_center, block_origin, diag_lidar_angles)
