"""The lowering kernel without the general sweep format (k_lower_xr
FASTONLY) runs only while every ESDF block is in the compact format: maps
written by the library alone with max_sq <= 510^2.  User-written ESDF data
(layer write_blocks) and larger distance limits keep the general kernel; both
paths stay bit-identical to the oracle (esdf/integrator.cpp:365-413)."""
import numpy as np
import pytest

import paper_2311_00626_b200 as vx
from oracle.bindings import PortOracle
from paper_2311_00626_b200 import _abi as A
from tests.helpers import camera_frames, layers_identical

pytestmark = pytest.mark.gpu


def _run(ecfg, edit=None, n=4):
    port = PortOracle()
    cam, seq = camera_frames("room", 320, 240, n, 16)
    icfg = A.default_integrator_config(truncation=0.16)
    T, E = vx.TsdfLayer(0.04), vx.EsdfLayer(0.04)
    To, Eo = port.layer(A.LAYER_TSDF, 0.04), port.layer(A.LAYER_ESDF, 0.04)
    for i, (pose, d) in enumerate(seq):
        a = vx.integrate_depth(T, d, pose, cam, icfg)
        b = port.integrate_camera(To, d, pose, cam, icfg)
        assert np.array_equal(a, b)
        assert np.array_equal(vx.update_esdf(E, T, a, ecfg), port.update_esdf(Eo, To, b, ecfg)), i
        if edit is not None and i == 1:  # the same user data written into both maps
            k, v = E.export()
            edit(v)
            E.write_blocks(k, v)
            port.write_blocks(Eo, k, v)
    assert layers_identical(*E.export(), *port.export(Eo))


def test_library_only_map():
    _run(A.default_esdf_config(site_threshold=0.04, max_distance=1.0))


def test_user_written_esdf_data_outside_the_compact_format():
    def edit(v):
        flat = v.reshape(-1)
        unobs = np.flatnonzero((flat["flags"] & 1) == 0)[:50]
        assert len(unobs) == 50
        flat["squared_distance"][unobs] = 1 << 30  # >= 2^29: not representable in the compact format
    _run(A.default_esdf_config(site_threshold=0.04, max_distance=1.0), edit)


def test_distance_limit_above_the_compact_range():
    # max_distance / vs = 625 voxels: max_sq = 390625 > 510^2
    _run(A.default_esdf_config(site_threshold=0.04, max_distance=25.0), n=3)
