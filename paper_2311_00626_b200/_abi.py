"""ctypes mirror of include/voxmap_b200.h (POD structs + status codes).

Shared by the product's Python host mirror (paper_2311_00626_b200.voxmap) and
the test-only oracle bindings (oracle/bindings.py).  No logic lives here.
"""
from __future__ import annotations

import ctypes as C
import math

import numpy as np

VXM_OK = 0
VXM_ERR_INVALID_POSE = 1
VXM_ERR_INVALID_ARGUMENT = 2
VXM_ERR_CAPACITY = 3
VXM_ERR_CUDA = 4
VXM_ERR_INTERNAL = 5
VXM_ERR_IO = 6

LAYER_TSDF = 0
LAYER_ESDF = 1
LAYER_OCCUPANCY = 2
LAYER_COLOR = 3

WEIGHT_CONSTANT = 0
WEIGHT_INVERSE_SQUARE = 1
SAMPLE_NEAREST = 0
SAMPLE_LINEAR = 1

VOXELS_PER_SIDE = 8
VOXELS_PER_BLOCK = 512

ESDF_OBSERVED = 1
ESDF_SITE = 2
ESDF_INSIDE = 4

# numpy views of the voxel PODs (core/voxels.hpp:22-68)
TSDF_DTYPE = np.dtype([("distance", "<f4"), ("weight", "<f4")])
ESDF_DTYPE = np.dtype([("squared_distance", "<i4"), ("parent_x", "<i2"), ("parent_y", "<i2"),
                       ("parent_z", "<i2"), ("flags", "u1"), ("reserved", "u1")])
OCCUPANCY_DTYPE = np.dtype([("log_odds", "<f4")])
COLOR_DTYPE = np.dtype([("r", "u1"), ("g", "u1"), ("b", "u1"), ("reserved", "u1"), ("weight", "<f4")])
assert TSDF_DTYPE.itemsize == 8 and ESDF_DTYPE.itemsize == 12 and OCCUPANCY_DTYPE.itemsize == 4
assert COLOR_DTYPE.itemsize == 8


def layer_dtype(kind):
    return {LAYER_TSDF: TSDF_DTYPE, LAYER_ESDF: ESDF_DTYPE, LAYER_OCCUPANCY: OCCUPANCY_DTYPE,
            LAYER_COLOR: COLOR_DTYPE}[kind]


class GridIndex(C.Structure):
    _fields_ = [("x", C.c_int32), ("y", C.c_int32), ("z", C.c_int32)]


class Camera(C.Structure):
    _fields_ = [("fu", C.c_double), ("fv", C.c_double), ("cu", C.c_double), ("cv", C.c_double),
                ("width", C.c_int32), ("height", C.c_int32), ("max_depth", C.c_double)]


class Lidar(C.Structure):
    _fields_ = [("num_azimuth", C.c_int32), ("num_elevation", C.c_int32),
                ("azimuth_start", C.c_double), ("elevation_start", C.c_double),
                ("azimuth_fov", C.c_double), ("elevation_fov", C.c_double),
                ("min_range", C.c_double), ("max_range", C.c_double)]


class PoseC(C.Structure):
    _fields_ = [("R", C.c_double * 9), ("t", C.c_double * 3)]


class IntegratorConfigC(C.Structure):
    _fields_ = [("truncation", C.c_double), ("max_weight", C.c_float), ("weighting", C.c_int32),
                ("max_integration_distance", C.c_double), ("camera_sample", C.c_int32),
                ("lidar_sample", C.c_int32), ("max_sample_gap", C.c_float),
                ("view_pixel_subsample", C.c_int32), ("hit_log_odds", C.c_float),
                ("miss_log_odds", C.c_float), ("log_odds_min", C.c_float),
                ("log_odds_max", C.c_float), ("parallel", C.c_int32)]


class ViewConfigC(C.Structure):
    _fields_ = [("max_integration_distance", C.c_double), ("truncation", C.c_double),
                ("pixel_subsample", C.c_int32)]


class EsdfConfigC(C.Structure):
    _fields_ = [("site_threshold", C.c_double), ("occupied_log_odds_threshold", C.c_float),
                ("max_distance", C.c_double), ("parallel", C.c_int32)]


class MeshConfigC(C.Structure):
    """vxm_mesh_config — MeshConfig (mesh/marching_cubes.hpp:24-33)."""
    _fields_ = [("min_weight", C.c_float), ("parallel", C.c_int32)]


def default_mesh_config(**kw):
    c = MeshConfigC(1e-4, 1)
    for k, v in kw.items():
        setattr(c, k, v)
    return c


class ReplayConfigC(C.Structure):
    """vxm_replay_config — ReplayConfig (io/pipeline.hpp:27-36)."""
    _fields_ = [("voxel_size", C.c_double), ("update_every", C.c_int32),
                ("integrator", IntegratorConfigC), ("esdf", EsdfConfigC),
                ("use_occupancy", C.c_int32), ("with_color", C.c_int32), ("mesh", MeshConfigC)]


class ReplayResultC(C.Structure):
    _fields_ = [("source", C.c_void_p), ("esdf", C.c_void_p), ("color", C.c_void_p),
                ("mesh", C.c_void_p)]


FRAME_TIMING_DTYPE = np.dtype([("frame", "<i4"), ("pad_", "<i4"), ("tsdf_ms", "<f8"),
                               ("color_ms", "<f8"), ("esdf_ms", "<f8"), ("mesh_ms", "<f8")])


class MeshBlockViewC(C.Structure):
    _fields_ = [("n_vertices", C.c_uint64), ("n_triangles", C.c_uint64), ("n_colors", C.c_uint64),
                ("vertices", C.POINTER(C.c_float)), ("normals", C.POINTER(C.c_float)),
                ("colors", C.POINTER(C.c_uint8)), ("triangles", C.POINTER(C.c_uint32))]


class QueryConfigC(C.Structure):
    _fields_ = [("interpolate", C.c_int32), ("parallel", C.c_int32)]


class QueryResultC(C.Structure):
    _fields_ = [("known", C.c_int32), ("pad_", C.c_int32), ("distance", C.c_double),
                ("gradient", C.c_double * 3)]


QUERY_DTYPE = np.dtype([("known", "<i4"), ("pad_", "<i4"), ("distance", "<f8"),
                        ("gradient", "<f8", (3,))])
assert QUERY_DTYPE.itemsize == C.sizeof(QueryResultC)


def quantize_log_odds(value: float) -> float:
    """config.hpp:29-31: nearbyint(double(v) * 4096) / 4096, rounded to float."""
    return float(np.float32(np.rint(float(np.float32(value)) * 4096.0) / 4096.0))


def default_integrator_config(**kw) -> IntegratorConfigC:
    """IntegratorConfig defaults (integrate/config.hpp:38-56)."""
    c = IntegratorConfigC(truncation=0.2, max_weight=100.0, weighting=WEIGHT_CONSTANT,
                          max_integration_distance=5.0, camera_sample=SAMPLE_NEAREST,
                          lidar_sample=SAMPLE_LINEAR, max_sample_gap=0.2, view_pixel_subsample=8,
                          hit_log_odds=quantize_log_odds(0.8473),
                          miss_log_odds=quantize_log_odds(-0.4055), log_odds_min=-5.0,
                          log_odds_max=5.0, parallel=1)
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def default_esdf_config(**kw) -> EsdfConfigC:
    """EsdfConfig defaults (esdf/integrator.hpp:30-40)."""
    c = EsdfConfigC(site_threshold=0.05, occupied_log_odds_threshold=0.0, max_distance=2.0,
                    parallel=1)
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def view_config_from(cfg: IntegratorConfigC) -> ViewConfigC:
    """integrator.cpp:77-78: ViewConfig{max_integration_distance, truncation, subsample}."""
    return ViewConfigC(cfg.max_integration_distance, cfg.truncation, cfg.view_pixel_subsample)


def pose_c(R, t) -> PoseC:
    p = PoseC()
    R = np.asarray(R, dtype=np.float64).reshape(3, 3)
    for i in range(9):
        p.R[i] = float(R.flat[i])
    for i in range(3):
        p.t[i] = float(t[i])
    return p


def pose_arrays(p: PoseC):
    return np.array(list(p.R), dtype=np.float64).reshape(3, 3), np.array(list(p.t))


def keys_array(ptr, n: int) -> np.ndarray:
    """(n, 3) int32 copy of a vxm_grid_index array."""
    if n == 0:
        return np.zeros((0, 3), dtype=np.int32)
    buf = (C.c_int32 * (3 * n)).from_address(C.cast(ptr, C.c_void_p).value)
    return np.frombuffer(buf, dtype=np.int32).reshape(n, 3).copy()


def as_keys(keys) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(keys, dtype=np.int32).reshape(-1, 3))
    return a


def ptr(a: np.ndarray):
    return C.c_void_p(a.ctypes.data) if a is not None and a.size else C.c_void_p(0)


def default_camera(width: int = 640, height: int = 480) -> Camera:
    """default_camera_intrinsics — io/dataset.cpp:309-319."""
    return Camera(width / 2.0, width / 2.0, width / 2.0, height / 2.0, width, height, 10.0)


def default_lidar(num_azimuth: int = 512, num_elevation: int = 32) -> Lidar:
    """default_lidar_intrinsics — io/dataset.cpp:321-332."""
    return Lidar(num_azimuth, num_elevation, -math.pi, 0.5 * math.pi - 0.3, 2.0 * math.pi, 0.6,
                 0.3, 20.0)
