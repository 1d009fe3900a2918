"""Occupancy source: occupancy integration and the
occupancy-source ESDF.

Reference: integrate_depth's Layer<OccupancyVoxel> overloads
(proj/src/integrate/integrator.cpp:148-158, 176-189) with occupancy_update
(include/voxmap/integrate/updates.hpp:59-72) and quantize_log_odds
(integrate/config.hpp:29-31); mark_sites / update_esdf from occupancy
(src/esdf/integrator.cpp:200-266 OccupancyClassifier, :425-431, :574-579);
the occupancy layer of the VXLF snapshot (core/serialization.cpp:98-103,
147-148); replay with use_occupancy (io/pipeline.cpp:73-77, 95-101).

CPU: the C restatement (oracle/voxmap_oracle.c) equals the reference's own
build (oracle/_ref) bit for bit, and the reference's occupancy KATs
(esdf_test.cpp:100-123, 271-306, 346-375) hold for both.  GPU: the device
path equals the reference bit for bit for the camera; for LiDAR the allocated
set, the changed lists and every log-odds value agree (the update is a
quantized sum, so it is exact wherever the hit/miss/occlusion decision is).
"""
import numpy as np
import pytest

from paper_2311_00626_b200 import _abi as A
from tests.helpers import camera_frames, layers_identical, lidar_frames

OCC = A.LAYER_OCCUPANCY


def _occ_blocks(n_blocks_side, fill):
    """Keys and voxels of a dense occupancy cube (global voxel g -> fill(g))."""
    keys, vox = [], []
    lin = np.arange(512)
    vx_, vy_, vz_ = lin & 7, (lin >> 3) & 7, lin >> 6
    for bx in range(n_blocks_side):
        for by in range(n_blocks_side):
            for bz in range(n_blocks_side):
                keys.append((bx, by, bz))
                v = np.zeros(512, A.OCCUPANCY_DTYPE)
                v["log_odds"] = fill(8 * bx + vx_, 8 * by + vy_, 8 * bz + vz_)
                vox.append(v)
    order = np.lexsort(np.array(keys).T[::-1])
    return np.array(keys, np.int32)[order], np.stack(vox)[order]


def _single_voxel_world():
    """esdf_test.cpp:271-306: free 32^3 (-1) with one occupied voxel (4) at (16,16,16)."""
    return _occ_blocks(4, lambda x, y, z: np.where((x == 16) & (y == 16) & (z == 16), 4.0, -1.0))


def _wall_world():
    """esdf_test.cpp:346-375: two blocks along x (-1.5) with an L-shaped wall (2.5)."""
    keys = np.array([[0, 0, 0], [1, 0, 0]], np.int32)
    vox = np.zeros((2, 512), A.OCCUPANCY_DTYPE)
    vox["log_odds"] = -1.5

    def put(x, y, z):
        vox[x // 8]["log_odds"][(x % 8) + 8 * (y + 8 * z)] = 2.5
    for x in range(3, 13):
        put(x, 2, 0)
        put(x, 2, 1)
    for y in range(2, 7):
        put(3, y, 0)
        put(3, y, 1)
    return keys, vox


def _exact_single_site(keys, vox_esdf, site, max_sq):
    lin = np.arange(512)
    for k, blk in zip(keys, vox_esdf):
        gx, gy, gz = 8 * k[0] + (lin & 7), 8 * k[1] + ((lin >> 3) & 7), 8 * k[2] + (lin >> 6)
        d2 = (gx - site[0]) ** 2 + (gy - site[1]) ** 2 + (gz - site[2]) ** 2
        if not np.array_equal(blk["squared_distance"], np.minimum(d2, max_sq)):
            return False
    return True


# ---- CPU: the restatement against the reference's own build -------------------

def test_port_occupancy_camera_and_lidar_equal_reference(port, ref):
    """integrate_test.cpp:295-321 'occupancy from camera / lidar frames' plus the
    occupancy ESDF on top, restatement vs the reference build, bit for bit."""
    cfg = A.default_integrator_config(truncation=0.2)
    ecfg = A.default_esdf_config(site_threshold=0.05)
    cam, cseq = camera_frames("sphere_in_box", 160, 120, 3, 8)
    li, lseq = lidar_frames("sphere_in_box", 180, 16, 3, 8)
    for kind, seq, sensor in (("camera", cseq, cam), ("lidar", lseq, li)):
        Lp, Lr = port.layer(OCC, 0.05), ref.layer(OCC, 0.05)
        Ep, Er = port.layer(A.LAYER_ESDF, 0.05), ref.layer(A.LAYER_ESDF, 0.05)
        for T, d in seq:
            if kind == "camera":
                a, b = port.integrate_camera(Lp, d, T, sensor, cfg), ref.integrate_camera(Lr, d, T, sensor, cfg)
            else:
                a, b = port.integrate_lidar(Lp, d, T, sensor, cfg), ref.integrate_lidar(Lr, d, T, sensor, cfg)
            assert len(a) and np.array_equal(a, b), kind
            assert np.array_equal(port.update_esdf(Ep, Lp, a, ecfg), ref.update_esdf(Er, Lr, b, ecfg))
        assert layers_identical(*port.export(Lp), *ref.export(Lr)), kind
        assert layers_identical(*port.export(Ep), *ref.export(Er)), kind
        _, lo = ref.export(Lr)
        q = lo["log_odds"].astype(np.float64) * 4096.0
        assert np.array_equal(q, np.round(q))  # quantized sums (integrate_test.cpp:150-213)
        assert lo["log_odds"].min() >= -5.0 and lo["log_odds"].max() <= 5.0


@pytest.mark.parametrize("oracle_name", ["port", "ref"])
def test_occupancy_esdf_kats(oracle_name, request):
    """esdf_test.cpp:100-123 (site next to free space), 271-306 (single occupied
    voxel in a free 32^3: exact everywhere), 346-375 (L-wall == brute force)."""
    o = request.getfixturevalue(oracle_name)
    cfg = A.default_esdf_config(site_threshold=0.05)
    # isolated occupied voxel inside one observed-free block
    keys = np.array([[0, 0, 0]], np.int32)
    vox = np.full((1, 512), -2.0, np.float32).view(A.OCCUPANCY_DTYPE)
    vox["log_odds"][0, 4 + 8 * (4 + 8 * 4)] = 3.0
    S, E = o.layer(OCC, 0.05), o.layer(A.LAYER_ESDF, 0.05)
    o.write_blocks(S, keys, vox)
    st = o.state()
    o.mark_sites(E, S, keys, cfg, st)
    _, ev = o.export(E)
    f = ev["flags"][0]
    assert f[4 + 8 * (4 + 8 * 4)] == A.ESDF_OBSERVED | A.ESDF_SITE | A.ESDF_INSIDE
    assert f[0] == A.ESDF_OBSERVED
    assert np.array_equal(st.get(0), keys)
    # 32^3 single voxel
    keys, vox = _single_voxel_world()
    S, E = o.layer(OCC, 0.05), o.layer(A.LAYER_ESDF, 0.05)
    o.write_blocks(S, keys, vox)
    o.update_esdf(E, S, keys, cfg)
    ke, ve = o.export(E)
    assert np.array_equal(ke, keys)
    assert _exact_single_site(ke, ve, (16, 16, 16), 1600)
    if oracle_name == "ref":  # brute_force_esdf lives in the reference build
        keys, vox = _wall_world()
        S, E = o.layer(OCC, 0.05), o.layer(A.LAYER_ESDF, 0.05)
        o.write_blocks(S, keys, vox)
        o.update_esdf(E, S, keys, cfg)
        cmp = o.compare_esdf(E, o.brute_force_esdf(E, cfg))
        assert cmp["compared"] == 1024 and cmp["flag_mismatches"] == 0
        assert cmp["exact"] == cmp["compared"]


def test_reference_snapshot_with_occupancy_round_trip(ref, tmp_path):
    """serialization.cpp:98-103, 147-148: the occupancy layer's VXLF record."""
    keys, vox = _wall_world()
    S = ref.layer(OCC, 0.05)
    ref.write_blocks(S, keys, vox)
    p = tmp_path / "o.vxlf"
    ref.save_snapshot(str(p), 0.05, occupancy=S)
    vs, t, o, e = ref.load_snapshot(str(p), with_occupancy=True)
    assert vs == 0.05 and t is None and e is None
    assert layers_identical(*ref.export(S), *ref.export(o))


# ---- GPU: the device path against the reference --------------------------------

@pytest.mark.gpu
@pytest.mark.parametrize("scene,w,h,vs,frames,orbit,trunc", [
    ("sphere_in_box", 160, 120, 0.05, 3, 8, 0.2),
    ("room", 640, 480, 0.02, 3, 100, 0.08),
])
def test_gpu_occupancy_camera_bitwise(vx, ref, scene, w, h, vs, frames, orbit, trunc):
    cam, seq = camera_frames(scene, w, h, frames, orbit)
    cfg = A.default_integrator_config(truncation=trunc)
    ecfg = A.default_esdf_config(site_threshold=vs)
    G, Ge = vx.OccupancyLayer(vs), vx.EsdfLayer(vs)
    R, Re = ref.layer(OCC, vs), ref.layer(A.LAYER_ESDF, vs)
    for T, d in seq:
        a = vx.integrate_depth(G, d, T, cam, cfg)
        b = ref.integrate_camera(R, d, T, cam, cfg)
        assert np.array_equal(a, b)
        assert np.array_equal(vx.update_esdf(Ge, G, a, ecfg), ref.update_esdf(Re, R, b, ecfg))
    assert layers_identical(*G.export(), *ref.export(R))
    assert layers_identical(*Ge.export(), *ref.export(Re))


@pytest.mark.gpu
def test_gpu_occupancy_lidar(vx, ref):
    li, seq = lidar_frames("sphere_in_box", 180, 16, 3, 8)
    cfg = A.default_integrator_config(truncation=0.2)
    ecfg = A.default_esdf_config(site_threshold=0.05)
    G, Ge = vx.OccupancyLayer(0.05), vx.EsdfLayer(0.05)
    R, Re = ref.layer(OCC, 0.05), ref.layer(A.LAYER_ESDF, 0.05)
    for T, d in seq:
        a = vx.integrate_depth(G, d, T, li, cfg)
        b = ref.integrate_lidar(R, d, T, li, cfg)
        assert len(a) and np.array_equal(a, b)
        assert np.array_equal(vx.update_esdf(Ge, G, a, ecfg), ref.update_esdf(Re, R, b, ecfg))
    ka, va = G.export()
    kb, vb = ref.export(R)
    assert np.array_equal(ka, kb)
    assert np.array_equal(va["log_odds"], vb["log_odds"])
    assert layers_identical(*Ge.export(), *ref.export(Re))


@pytest.mark.gpu
def test_gpu_occupancy_esdf_kats(vx, ref):
    cfg = A.default_esdf_config(site_threshold=0.05)
    keys, vox = _single_voxel_world()
    S, E = vx.OccupancyLayer(0.05), vx.EsdfLayer(0.05)
    S.write_blocks(keys, vox)
    vx.update_esdf(E, S, keys, cfg)
    ke, ve = E.export()
    assert np.array_equal(ke, keys) and _exact_single_site(ke, ve, (16, 16, 16), 1600)
    keys, vox = _wall_world()
    S, E = vx.OccupancyLayer(0.05), vx.EsdfLayer(0.05)
    R, Re = ref.layer(OCC, 0.05), ref.layer(A.LAYER_ESDF, 0.05)
    S.write_blocks(keys, vox)
    ref.write_blocks(R, keys, vox)
    assert np.array_equal(vx.update_esdf(E, S, keys, cfg), ref.update_esdf(Re, R, keys, cfg))
    assert layers_identical(*E.export(), *ref.export(Re))
    # a source change: the wall's second layer becomes free (site flips, clears)
    vox2 = vox.copy()
    for x in range(3, 13):
        vox2[x // 8]["log_odds"][(x % 8) + 8 * (2 + 8 * 1)] = -1.5
    S.write_blocks(keys, vox2)
    ref.write_blocks(R, keys, vox2)
    assert np.array_equal(vx.update_esdf(E, S, keys, cfg), ref.update_esdf(Re, R, keys, cfg))
    assert layers_identical(*E.export(), *ref.export(Re))


@pytest.mark.gpu
def test_gpu_occupancy_frame_step_and_replay(vx, ref):
    """The fused frame step and replay(use_occupancy) (pipeline.cpp:73-77, 95-101)
    equal the reference's calls in pipeline order."""
    import torch
    cam, seq = camera_frames("room", 320, 240, 5, 16)
    cfg = vx.make_replay_config(0.04)
    cfg.use_occupancy = 1
    cfg.update_every = 2
    src, E, timings = vx.replay(seq, cam, cfg)
    assert isinstance(src, vx.OccupancyLayer)
    R, Re = ref.layer(OCC, 0.04), ref.layer(A.LAYER_ESDF, 0.04)
    pending = np.zeros((0, 3), np.int32)
    for k, (T, d) in enumerate(seq):
        pending = np.unique(np.concatenate([pending, ref.integrate_camera(R, d, T, cam, cfg.integrator)]), axis=0)
        if ((k + 1) % 2 == 0 or k + 1 == len(seq)) and len(pending):
            ref.update_esdf(Re, R, pending, cfg.esdf)
            pending = np.zeros((0, 3), np.int32)
    assert layers_identical(*src.export(), *ref.export(R))
    assert layers_identical(*E.export(), *ref.export(Re))
    # frame step (one round trip per frame) from an occupancy source
    G, Ge = vx.OccupancyLayer(0.04), vx.EsdfLayer(0.04)
    R, Re = ref.layer(OCC, 0.04), ref.layer(A.LAYER_ESDF, 0.04)
    tout, eout = vx.BlockList(G.ctx), vx.BlockList(G.ctx)
    for T, d in seq:
        dd = torch.from_numpy(d).cuda()
        vx.update_frame_device(G, Ge, dd.data_ptr(), d.shape[1], d.shape[0], T, cam,
                               cfg.integrator, cfg.esdf, tout, eout)
        b = ref.integrate_camera(R, d, T, cam, cfg.integrator)
        assert np.array_equal(tout.numpy(), b)
        assert np.array_equal(eout.numpy(), ref.update_esdf(Re, R, b, cfg.esdf))
    assert layers_identical(*G.export(), *ref.export(R))
    assert layers_identical(*Ge.export(), *ref.export(Re))


@pytest.mark.gpu
def test_gpu_occupancy_snapshot_matches_reference(vx, ref, tmp_path):
    keys, vox = _wall_world()
    S, E = vx.OccupancyLayer(0.05), vx.EsdfLayer(0.05)
    R, Re = ref.layer(OCC, 0.05), ref.layer(A.LAYER_ESDF, 0.05)
    S.write_blocks(keys, vox)
    ref.write_blocks(R, keys, vox)
    cfg = A.default_esdf_config(site_threshold=0.05)
    vx.update_esdf(E, S, keys, cfg)
    ref.update_esdf(Re, R, keys, cfg)
    T = vx.TsdfLayer(0.05)
    ours, theirs = tmp_path / "ours.vxlf", tmp_path / "ref.vxlf"
    vx.save_snapshot(str(ours), 0.05, None, E, occupancy=S)
    ref.save_snapshot(str(theirs), 0.05, None, Re, occupancy=R)
    assert ours.read_bytes() == theirs.read_bytes()
    vs, t, o, e = vx.load_snapshot(str(theirs), with_occupancy=True)
    assert vs == 0.05 and t is None
    assert layers_identical(*o.export(), *ref.export(R))
    assert layers_identical(*e.export(), *ref.export(Re))
    with pytest.raises(vx.IoError, match="occupancy"):
        vx.load_snapshot(str(theirs))  # the two-layer entry point cannot return it
    del T


@pytest.mark.gpu
def test_gpu_occupancy_layer_type_errors(vx):
    cam, seq = camera_frames("sphere_in_box", 160, 120, 1, 8)
    T, d = seq[0]
    E = vx.EsdfLayer(0.05)
    with pytest.raises(vx.InvalidArgumentError):
        vx.integrate_depth(E, d, T, cam, A.default_integrator_config())
    S = vx.OccupancyLayer(0.05)
    with pytest.raises(vx.InvalidArgumentError):
        vx.update_esdf(S, S, np.zeros((1, 3), np.int32), A.default_esdf_config())
