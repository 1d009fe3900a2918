"""GPU parity at BASELINE.json's larger configurations.

C5 (ESDF full recompute of a dense SphereWorld volume, fixtures.hpp:34-98 /
SURVEY §8(d)) against the reference's own OpenMP code (oracle/_ref) at
256^3, and at the full 512^3 through size-independent properties:
idempotence (a second update with the same input changes nothing,
esdf_test.cpp:308-335) and agreement with the exact Euclidean distance on
sampled voxels (the reference's brute-force bar, eval/oracle.cpp:26-134).

C3 (64 x 2048 LiDAR, 10 cm, 100 m): two frames against the reference —
allocated block sets and observed masks exact, TSDF within the reference's
1e-5 relative bound (integrate_test.cpp:108-113); the ESDF half exact when fed
identical TSDF blocks.
"""
import numpy as np
import pytest

from paper_2311_00626_b200 import _abi as A
from paper_2311_00626_b200 import synth
from tests.helpers import layers_identical, lidar_frames, tsdf_close

pytestmark = pytest.mark.gpu

C5_VS, C5_TRUNC = 0.02, 0.08


def c5_cfg():
    return A.default_esdf_config(site_threshold=0.02, max_distance=2.0)


def test_c5_sphere_world_256_vs_reference(vx, ref):
    keys, vox = synth.sphere_world(256, C5_VS, C5_TRUNC)
    T, E = vx.TsdfLayer(C5_VS), vx.EsdfLayer(C5_VS)
    T.write_blocks(keys, vox)
    a = vx.update_esdf(E, T, keys, c5_cfg())
    To, Eo = ref.layer(A.LAYER_TSDF, C5_VS), ref.layer(A.LAYER_ESDF, C5_VS)
    ref.write_blocks(To, keys, vox)
    b = ref.update_esdf(Eo, To, keys, c5_cfg())
    assert np.array_equal(a, b)
    assert layers_identical(*E.export(), *ref.export(Eo))


def _sites(keys, vox):
    """World voxel coordinates of every site (ESDF flag bit 2)."""
    lin = np.arange(512)
    off = np.stack([lin % 8, (lin // 8) % 8, lin // 64], -1)
    b, v = np.nonzero(vox["flags"] & A.ESDF_SITE)
    return keys[b].astype(np.int64) * 8 + off[v]


def test_c5_sphere_world_512_properties(vx):
    keys, vox = synth.sphere_world(512, C5_VS, C5_TRUNC)
    T, E = vx.TsdfLayer(C5_VS), vx.EsdfLayer(C5_VS)
    T.write_blocks(keys, vox)
    del vox
    cfg = c5_cfg()
    first = vx.update_esdf(E, T, keys, cfg)
    assert len(first) == len(keys)  # every block is new
    # idempotent: same input again -> no site change, nothing lowered
    assert len(vx.update_esdf(E, T, keys, cfg)) == 0
    ek, ev = E.export()
    assert np.array_equal(ek, keys)
    # exact EDT on sampled observed voxels: >= 99% exact, all within one voxel
    from scipy.spatial import cKDTree
    tree = cKDTree(_sites(ek, ev))
    rng = np.random.default_rng(11)
    bi = rng.integers(0, len(ek), 20000)
    vi = rng.integers(0, 512, 20000)
    sel = ((ev["flags"][bi, vi] & A.ESDF_OBSERVED) != 0) & ((ev["flags"][bi, vi] & A.ESDF_SITE) == 0)
    bi, vi = bi[sel], vi[sel]
    pos = ek[bi].astype(np.int64) * 8 + np.stack([vi % 8, (vi // 8) % 8, vi // 64], -1)
    dist, _ = tree.query(pos.astype(np.float64))
    best = np.rint(dist * dist).astype(np.int64)  # integer lattice: exact
    max_sq, cap = 10000, 16
    inside = (ev["flags"][bi, vi] & A.ESDF_INSIDE) != 0
    want = np.minimum(best, np.where(inside, cap, max_sq))
    got = ev["squared_distance"][bi, vi].astype(np.int64)
    exact = got == want
    assert exact.mean() >= 0.99
    assert np.all(np.abs(np.sqrt(got) - np.sqrt(want)) <= 1.0 + 1e-9)


def test_c3_lidar_two_frames_vs_reference(vx, ref):
    li, seq = lidar_frames("lidar_yard", 2048, 64, 2, 100, max_range=100.0)
    icfg = A.default_integrator_config(truncation=0.4, max_integration_distance=100.0)
    ecfg = A.default_esdf_config(site_threshold=0.1, max_distance=2.0)
    T, E = vx.TsdfLayer(0.1), vx.EsdfLayer(0.1)
    To, Eo = ref.layer(A.LAYER_TSDF, 0.1), ref.layer(A.LAYER_ESDF, 0.1)
    Tf = ref.layer(A.LAYER_TSDF, 0.1)  # reference ESDF input = our TSDF bytes
    for pose, d in seq:
        a = vx.integrate_depth(T, d, pose, li, icfg)
        b = ref.integrate_lidar(To, d, pose, li, icfg)
        ka, va = T.export()
        kb, vb = ref.export(To)
        assert np.array_equal(ka, kb)                                # allocated set exact
        assert np.array_equal(va["weight"] > 0, vb["weight"] > 0)   # observed mask exact
        assert tsdf_close(va, vb)
        # changed lists agree up to voxels whose bytes differ in the last ulp
        diff = set(map(tuple, a)) ^ set(map(tuple, b))
        assert len(diff) <= max(1, len(b) // 1000)
        ref.write_blocks(Tf, ka, va)
        ea = vx.update_esdf(E, T, a, ecfg)
        eb = ref.update_esdf(Eo, Tf, a, ecfg)
        assert np.array_equal(ea, eb)
    assert layers_identical(*E.export(), *ref.export(Eo))


def test_c4_building_1cm_two_frames_vs_reference(vx, ref):
    """C4 at 1 cm (building walkthrough, 640x480): camera path bit-exact."""
    from tests.helpers import camera_frames
    cam, seq = camera_frames("building", 640, 480, 2, 100)
    icfg = A.default_integrator_config(truncation=0.04)
    ecfg = A.default_esdf_config(site_threshold=0.01, max_distance=2.0)
    T, E = vx.TsdfLayer(0.01), vx.EsdfLayer(0.01)
    To, Eo = ref.layer(A.LAYER_TSDF, 0.01), ref.layer(A.LAYER_ESDF, 0.01)
    for pose, d in seq:
        a = vx.integrate_depth(T, d, pose, cam, icfg)
        b = ref.integrate_camera(To, d, pose, cam, icfg)
        assert np.array_equal(a, b)
        assert np.array_equal(vx.update_esdf(E, T, a, ecfg), ref.update_esdf(Eo, To, b, ecfg))
    assert layers_identical(*T.export(), *ref.export(To))
    assert layers_identical(*E.export(), *ref.export(Eo))
