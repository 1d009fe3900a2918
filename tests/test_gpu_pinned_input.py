"""GPU parity: host depth images in page-locked memory vs pageable memory.

integrate_depth (integrator.hpp:34-48) through the host API must give the
same changed lists and layer bytes whether the caller's image is page-locked
(vxm_host_alloc: the e2e bench's frames, a direct DMA) or pageable, and the
same as the oracle; with a pool re-run (the staged image used twice) and
with the host buffer rewritten between calls.  (Measured and not kept: the
view kernels reading a page-locked image over PCIe themselves, overlapping
the transfer with the ray casting — 32-byte tile reads made it slower than
the DMA: C1 e2e 9.8k -> 8.7k frames/s, profiles/r2_ab_host_path.txt.)
"""
import numpy as np
import pytest

from paper_2311_00626_b200 import _abi as A
from tests.helpers import camera_frames, layers_identical, lidar_frames

pytestmark = pytest.mark.gpu


def _run(vx, frames, sensor, cfg, vs, pinned):
    T = vx.TsdfLayer(vs)
    outs = []
    buf = None
    for pose, d in frames:
        d = np.ascontiguousarray(d, np.float32)
        if pinned:
            if buf is None:
                buf = vx.pinned_like(d)  # one buffer, rewritten per frame
            else:
                buf.array[...] = d
            img = buf.array
        else:
            img = d
        outs.append(vx.integrate_depth(T, img, pose, sensor, cfg).copy())
    return T, outs


def test_pinned_camera_matches_pageable_and_oracle(vx, port):
    cam, seq = camera_frames("room", 320, 240, 4, 16)
    cfg = A.default_integrator_config(truncation=0.16)
    Ta, oa = _run(vx, seq, cam, cfg, 0.04, pinned=True)
    Tb, ob = _run(vx, seq, cam, cfg, 0.04, pinned=False)
    To = port.layer(A.LAYER_TSDF, 0.04)
    for (pose, d), a, b in zip(seq, oa, ob):
        assert np.array_equal(a, b)
        assert np.array_equal(a, port.integrate_camera(To, d, pose, cam, cfg))
    assert layers_identical(*Ta.export(), *Tb.export())
    assert layers_identical(*Ta.export(), *To.export())


def test_pinned_lidar_matches_pageable(vx):
    li, seq = lidar_frames("room", 512, 32, 3, 16)
    cfg = A.default_integrator_config(truncation=0.2)
    Ta, oa = _run(vx, seq, li, cfg, 0.05, pinned=True)
    Tb, ob = _run(vx, seq, li, cfg, 0.05, pinned=False)
    for a, b in zip(oa, ob):
        assert np.array_equal(a, b)
    assert layers_identical(*Ta.export(), *Tb.export())


def test_pinned_pool_rerun(vx):
    # >65k new blocks in one LiDAR frame overflow the initial pool: the frame
    # is re-run after growth and the view kernels read the host image again
    li, seq = lidar_frames("lidar_yard", 2048, 64, 1, 100, max_range=100.0)
    cfg = A.default_integrator_config(truncation=0.4, max_integration_distance=100.0)
    Ta, oa = _run(vx, seq, li, cfg, 0.1, pinned=True)
    Tb, ob = _run(vx, seq, li, cfg, 0.1, pinned=False)
    assert np.array_equal(oa[0], ob[0])
    assert Ta.num_blocks() > 65536
    assert layers_identical(*Ta.export(), *Tb.export())


def test_pinned_then_update_esdf(vx):
    # the host-API pair of the bench's e2e path, pinned frames
    cam, seq = camera_frames("room", 320, 240, 3, 16)
    icfg = A.default_integrator_config(truncation=0.16)
    ecfg = A.default_esdf_config(site_threshold=0.04, max_distance=1.0)
    T1, E1 = vx.TsdfLayer(0.04), vx.EsdfLayer(0.04)
    T2, E2 = vx.TsdfLayer(0.04), vx.EsdfLayer(0.04)
    for pose, d in seq:
        d = np.ascontiguousarray(d, np.float32)
        buf = vx.pinned_like(d)
        c1 = vx.integrate_depth(T1, buf.array, pose, cam, icfg)
        e1 = vx.update_esdf(E1, T1, c1, ecfg)
        c2 = vx.integrate_depth(T2, d, pose, cam, icfg)
        e2 = vx.update_esdf(E2, T2, c2, ecfg)
        assert np.array_equal(c1, c2)
        assert np.array_equal(e1, e2)
    assert layers_identical(*E1.export(), *E2.export())
