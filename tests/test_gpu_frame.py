"""GPU parity: the fused per-frame update (vxm_update_frame_*_device).

One replay-pipeline frame (proj/src/pipeline/pipeline.cpp:95-108: integrate,
then update_esdf on the changed blocks) with a single host round trip.  It
must reproduce the two reference calls exactly: same changed lists, same
layer bytes, against the oracle and against the two-call GPU path, including
a frame whose allocations overflow the pre-sized pool (re-run after growth).
"""
import numpy as np
import pytest
import torch

from paper_2311_00626_b200 import _abi as A
from tests.helpers import camera_frames, layers_identical, lidar_frames

pytestmark = pytest.mark.gpu


def _dev(d):
    return torch.from_numpy(np.ascontiguousarray(d, np.float32)).cuda()


def test_update_frame_matches_oracle_camera(vx, port):
    cam, seq = camera_frames("room", 320, 240, 4, 16)
    icfg = A.default_integrator_config(truncation=0.16)
    ecfg = A.default_esdf_config(site_threshold=0.04, max_distance=1.0)
    ctx = vx.default_context()
    T, E = vx.TsdfLayer(0.04), vx.EsdfLayer(0.04)
    To, Eo = port.layer(A.LAYER_TSDF, 0.04), port.layer(A.LAYER_ESDF, 0.04)
    tch, ech = vx.BlockList(ctx), vx.BlockList(ctx)
    for pose, d in seq:
        dd = _dev(d)
        torch.cuda.synchronize()
        vx.update_frame_device(T, E, dd.data_ptr(), d.shape[1], d.shape[0], pose, cam, icfg, ecfg,
                               tch, ech)
        b = port.integrate_camera(To, d, pose, cam, icfg)
        eb = port.update_esdf(Eo, To, b, ecfg)
        assert np.array_equal(tch.numpy(), b)
        assert np.array_equal(ech.numpy(), eb)
    assert layers_identical(*T.export(), *To.export())
    assert layers_identical(*E.export(), *Eo.export())


def test_update_frame_integrate_only(vx):
    cam, seq = camera_frames("sphere_in_box", 160, 120, 3, 8)
    icfg = A.default_integrator_config(truncation=0.2)
    ctx = vx.default_context()
    Ta, Tb = vx.TsdfLayer(0.05), vx.TsdfLayer(0.05)
    ca, cb = vx.BlockList(ctx), vx.BlockList(ctx)
    for pose, d in seq:
        dd = _dev(d)
        torch.cuda.synchronize()
        vx.update_frame_device(Ta, None, dd.data_ptr(), d.shape[1], d.shape[0], pose, cam, icfg,
                               None, ca, None)
        vx.integrate_depth_device(Tb, dd.data_ptr(), d.shape[1], d.shape[0], pose, cam, icfg, cb)
        assert np.array_equal(ca.numpy(), cb.numpy())
    assert layers_identical(*Ta.export(), *Tb.export())


def test_update_frame_pool_rerun_lidar(vx):
    """C3-like LiDAR frame: >65k new blocks in one frame overflow the
    pre-sized pool; the fused call grows it and re-runs, matching the
    two-call path (which does the same inside integrate_depth)."""
    li, seq = lidar_frames("lidar_yard", 2048, 64, 2, 100, max_range=100.0)
    icfg = A.default_integrator_config(truncation=0.4, max_integration_distance=100.0)
    ecfg = A.default_esdf_config(site_threshold=0.1, max_distance=2.0)
    ctx = vx.default_context()
    Ta, Ea = vx.TsdfLayer(0.1), vx.EsdfLayer(0.1)
    Tb, Eb = vx.TsdfLayer(0.1), vx.EsdfLayer(0.1)
    ta, ea = vx.BlockList(ctx), vx.BlockList(ctx)
    for pose, d in seq:
        dd = _dev(d)
        torch.cuda.synchronize()
        vx.update_frame_device(Ta, Ea, dd.data_ptr(), d.shape[1], d.shape[0], pose, li, icfg, ecfg,
                               ta, ea)
        tb = vx.integrate_depth(Tb, d, pose, li, icfg)
        eb = vx.update_esdf(Eb, Tb, tb, ecfg)
        assert np.array_equal(ta.numpy(), tb)
        assert np.array_equal(ea.numpy(), eb)
    assert Ta.num_blocks() > 65536
    assert layers_identical(*Ta.export(), *Tb.export())
    assert layers_identical(*Ea.export(), *Eb.export())


def test_update_frame_rejects_before_mutation(vx):
    cam, seq = camera_frames("sphere_in_box", 160, 120, 1, 8)
    icfg = A.default_integrator_config(truncation=0.2)
    ecfg = A.default_esdf_config(site_threshold=0.05)
    ctx = vx.default_context()
    T, E = vx.TsdfLayer(0.05), vx.EsdfLayer(0.1)  # voxel sizes differ
    pose, d = seq[0]
    dd = _dev(d)
    torch.cuda.synchronize()
    with pytest.raises(vx.InvalidArgumentError):
        vx.update_frame_device(T, E, dd.data_ptr(), d.shape[1], d.shape[0], pose, cam, icfg, ecfg,
                               vx.BlockList(ctx), vx.BlockList(ctx))
    assert T.num_blocks() == 0


def test_update_esdf_host_list_reuse_matches_oracle(vx, port):
    """update_esdf on the host list the last integrate returned reuses its device
    keys; an older (different) list is uploaded — both equal the oracle."""
    from paper_2311_00626_b200 import _abi as A
    from tests.helpers import camera_frames, layers_identical
    cam, seq = camera_frames("sphere_in_box", 160, 120, 3, 8)
    icfg = A.default_integrator_config(truncation=0.2)
    ecfg = A.default_esdf_config(site_threshold=0.05)
    T, E = vx.TsdfLayer(0.05), vx.EsdfLayer(0.05)
    To, Eo = port.layer(A.LAYER_TSDF, 0.05), port.layer(A.LAYER_ESDF, 0.05)
    lists = []
    for pose, d in seq[:2]:
        a = vx.integrate_depth(T, d, pose, cam, icfg)
        assert np.array_equal(a, port.integrate_camera(To, d, pose, cam, icfg))
        lists.append(a)
    # stale list first (uploaded), then the last integrate's list (reused), then a subset
    for u in (lists[0], lists[1], lists[1][: len(lists[1]) // 2]):
        assert np.array_equal(vx.update_esdf(E, T, u, ecfg), port.update_esdf(Eo, To, u, ecfg))
    assert layers_identical(*E.export(), *port.export(Eo))
