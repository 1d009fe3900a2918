"""Synthetic inputs (include/voxmap_b200_synth.h): scenes, orbit poses,
sphere-traced depth frames, and the dense SphereWorld TSDF of config C5.

Test and bench input generation only: it lives in its own host library
(_lib/libvoxmap_synth.so), not in the product library."""
from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from . import _abi as A
from .voxmap import Pose

SYNTH_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib", "libvoxmap_synth.so")
_synth = None
_synth_lock = threading.Lock()


def lib():
    """Loads libvoxmap_synth.so (the input generator)."""
    global _synth
    with _synth_lock:
        if _synth is None:
            if not os.path.exists(SYNTH_PATH):
                raise ImportError(f"{SYNTH_PATH} missing: run __graft_entry__.build()")
            L = C.CDLL(SYNTH_PATH)
            L.vxm_synth_scene_sdf.restype = C.c_double
            _synth = L
        return _synth


def check(rc):
    if rc != A.VXM_OK:
        raise ValueError(f"synthetic input generator failed (status {rc})")


class Scene:
    """make_scene (io/scene.cpp:124-144) + builder scenes 'lidar_yard', 'building'."""

    def __init__(self, name: str):
        h = C.c_void_p()
        rc = lib().vxm_synth_scene_create(name.encode(), C.byref(h))
        if rc != 0:
            raise ValueError(f"unknown scene {name!r}")
        self.h = h
        self.name = name

    def __del__(self):
        try:
            lib().vxm_synth_scene_destroy(self.h)
        except Exception:
            pass

    @property
    def bbox(self):
        b = (C.c_double * 6)()
        lib().vxm_synth_scene_bbox(self.h, b)
        return np.array(b[:3]), np.array(b[3:])

    def sdf(self, p) -> float:
        a = (C.c_double * 3)(*[float(x) for x in p])
        return float(lib().vxm_synth_scene_sdf(self.h, a))

    def orbit_pose(self, k: int, total: int, lidar: bool = False) -> A.PoseC:
        p = A.PoseC()
        check(lib().vxm_synth_orbit_pose(self.h, C.c_int(int(lidar)), C.c_int(k), C.c_int(total),
                                         C.byref(p)))
        return p

    def render_camera(self, T: A.PoseC, cam: A.Camera) -> np.ndarray:
        out = np.zeros((cam.height, cam.width), np.float32)
        check(lib().vxm_synth_render_camera(self.h, C.byref(T), C.byref(cam), A.ptr(out)))
        return out

    def render_lidar(self, T: A.PoseC, li: A.Lidar) -> np.ndarray:
        out = np.zeros((li.num_elevation, li.num_azimuth), np.float32)
        check(lib().vxm_synth_render_lidar(self.h, C.byref(T), C.byref(li), A.ptr(out)))
        return out


def sphere_world(side: int, vs: float, trunc: float, seed: int = 2311, n_spheres: int = 6):
    """Dense C5 TSDF: (keys (nb^3,3), voxels (nb^3,512) TSDF_DTYPE)."""
    nb = side // 8
    keys = np.zeros((nb ** 3, 3), np.int32)
    vox = np.zeros((nb ** 3, A.VOXELS_PER_BLOCK), A.TSDF_DTYPE)
    check(lib().vxm_synth_sphere_world(C.c_int(side), C.c_double(vs), C.c_double(trunc),
                                       C.c_uint(seed), C.c_int(n_spheres), A.ptr(keys), A.ptr(vox)))
    return keys, vox


__all__ = ["Scene", "sphere_world", "Pose"]
