"""Shared test helpers: synthetic frame sequences and layer comparisons."""
from __future__ import annotations

import numpy as np

from paper_2311_00626_b200 import _abi as A


def camera_frames(scene_name, w, h, n_frames, orbit, start=0):
    from paper_2311_00626_b200 import synth
    S = synth.Scene(scene_name)
    cam = A.default_camera(w, h)
    out = []
    for k in range(start, start + n_frames):
        T = S.orbit_pose(k, orbit)
        out.append((T, S.render_camera(T, cam)))
    return cam, out


def lidar_frames(scene_name, na, ne, n_frames, orbit, max_range=None, start=0):
    from paper_2311_00626_b200 import synth
    S = synth.Scene(scene_name)
    li = A.default_lidar(na, ne)
    if max_range is not None:
        li.max_range = max_range
    out = []
    for k in range(start, start + n_frames):
        T = S.orbit_pose(k, orbit, lidar=True)
        out.append((T, S.render_lidar(T, li)))
    return li, out


def layers_identical(ka, va, kb, vb):
    return np.array_equal(ka, kb) and va.tobytes() == vb.tobytes()


def tsdf_close(va, vb, rtol=1e-5):
    """LiDAR tolerance (integrate_test.cpp:108-113 bound): 1e-5 relative."""
    da, db = va["distance"].astype(np.float64), vb["distance"].astype(np.float64)
    wa, wb = va["weight"].astype(np.float64), vb["weight"].astype(np.float64)
    ok_d = np.abs(da - db) <= rtol * (np.abs(db) + 1e-3)
    ok_w = np.abs(wa - wb) <= rtol * (np.abs(wb) + 1e-3)
    return bool(ok_d.all() and ok_w.all())
