"""GPU parity: ESDF update (mark / clear / lower / full update) and queries.

Bitwise against the oracle restatement of proj/src/esdf/integrator.cpp, plus
the reference's own ESDF known-answer tests (proj/tests/esdf_test.cpp).
"""
import numpy as np
import pytest

from paper_2311_00626_b200 import _abi as A
from tests.helpers import camera_frames, layers_identical

pytestmark = pytest.mark.gpu

VS = 0.05


def ecfg(**kw):
    c = A.default_esdf_config(site_threshold=0.05, max_distance=2.0)
    for k, v in kw.items():
        setattr(c, k, v)
    return c


def make_tsdf(side, dist_fn):
    """esdf_test.cpp:40-59: fully observed side^3 region, distance from callback."""
    nb = side // 8
    keys, vox = [], []
    lin = np.arange(512)
    vx_, vy_, vz_ = lin % 8, (lin // 8) % 8, lin // 64
    for bz in range(nb):
        for by in range(nb):
            for bx in range(nb):
                keys.append((bx, by, bz))
                b = np.zeros(512, A.TSDF_DTYPE)
                b["distance"] = dist_fn(bx * 8 + vx_, by * 8 + vy_, bz * 8 + vz_)
                b["weight"] = 1.0
                vox.append(b)
    return np.array(keys, np.int32), np.stack(vox)


def gpu_tsdf(vx, keys, vox):
    L = vx.TsdfLayer(VS)
    L.write_blocks(keys, vox)
    return L


def test_esdf_distance_kat(vx):
    """esdf_test.cpp:61-78."""
    assert vx.esdf_distance(25, False, 0.05) == pytest.approx(0.25, rel=1e-12)
    assert vx.esdf_distance(25, True, 0.05) == pytest.approx(-0.25, rel=1e-12)


def test_mark_sites_site_kat(vx):
    """esdf_test.cpp:80-98."""
    keys, vox = make_tsdf(8, lambda x, y, z: np.where((x == 3) & (y == 3) & (z == 3), 0.01, 0.15))
    T = gpu_tsdf(vx, keys, vox)
    E = vx.EsdfLayer(VS)
    st = vx.EsdfUpdateState()
    vx.mark_sites(E, T, keys, ecfg(), st)
    blk = E.block((0, 0, 0))
    v = blk[3 + 8 * 3 + 64 * 3]
    assert v["flags"] & A.ESDF_SITE and v["squared_distance"] == 0 and not v["flags"] & A.ESDF_INSIDE
    assert st.indices_to_update.tolist() == [[0, 0, 0]]
    assert len(st.indices_to_clear) == 0


def test_site_flip_queues_clear(vx):
    """esdf_test.cpp:125-148."""
    def wall(x0):
        return lambda x, y, z: np.where(x == x0, 0.0, 0.2)
    k, v = make_tsdf(16, wall(2))
    T = gpu_tsdf(vx, k, v)
    E = vx.EsdfLayer(VS)
    vx.update_esdf(E, T, k, ecfg())
    k2, v2 = make_tsdf(16, wall(12))
    T2 = gpu_tsdf(vx, k2, v2)
    st = vx.EsdfUpdateState()
    vx.mark_sites(E, T2, k2, ecfg(), st)
    assert [0, 0, 0] in st.indices_to_clear.tolist()
    assert [1, 0, 0] in st.indices_to_update.tolist()


def test_clear_invalid_noop_and_reset(vx):
    """esdf_test.cpp:150-191."""
    k, v = make_tsdf(16, lambda x, y, z: np.where(x == 5, 0.0, 0.2))
    T = gpu_tsdf(vx, k, v)
    E = vx.EsdfLayer(VS)
    vx.update_esdf(E, T, k, ecfg())
    before = E.export()
    st = vx.EsdfUpdateState()
    assert len(vx.clear_invalid(E, ecfg(), st)) == 0
    after = E.export()
    assert layers_identical(*before, *after)

    cfg = ecfg(max_distance=0.6)
    k, v = make_tsdf(16, lambda x, y, z: np.where((x == 8) & (y == 8) & (z == 8), 0.0, 0.2))
    T = gpu_tsdf(vx, k, v)
    E = vx.EsdfLayer(VS)
    vx.update_esdf(E, T, k, cfg)
    k2, v2 = make_tsdf(16, lambda x, y, z: np.full_like(x, 0.2, dtype=np.float64))
    T2 = gpu_tsdf(vx, k2, v2)
    st = vx.EsdfUpdateState()
    vx.mark_sites(E, T2, k2, cfg, st)
    vx.clear_invalid(E, cfg, st)
    _, vox = E.export()
    max_sq = int(round((0.6 / VS) ** 2))
    assert (vox["squared_distance"] == max_sq).all()
    assert ((vox["parent_x"] == 0) & (vox["parent_y"] == 0) & (vox["parent_z"] == 0)).all()


def test_single_site_exact_and_bounded_rounds(vx):
    """esdf_test.cpp:232-269."""
    k, v = make_tsdf(16, lambda x, y, z: np.where((x == 0) & (y == 0) & (z == 0), 0.0, 0.2))
    T = gpu_tsdf(vx, k, v)
    E = vx.EsdfLayer(VS)
    st = vx.EsdfUpdateState()
    vx.mark_sites(E, T, k, ecfg(), st)
    vx.clear_invalid(E, ecfg(), st)
    rounds, _ = vx.lower_esdf(E, st, ecfg())
    assert rounds <= 4
    keys, vox = E.export()
    lin = np.arange(512)
    for b, g in enumerate(keys):
        gx, gy, gz = g[0] * 8 + lin % 8, g[1] * 8 + (lin // 8) % 8, g[2] * 8 + lin // 64
        exact = gx * gx + gy * gy + gz * gz
        assert np.array_equal(vox[b]["squared_distance"], exact)
        m = exact > 0
        assert np.array_equal(vox[b]["parent_x"][m], -gx[m])
        assert np.array_equal(vox[b]["parent_y"][m], -gy[m])
        assert np.array_equal(vox[b]["parent_z"][m], -gz[m])
    st2 = vx.EsdfUpdateState()
    st2.indices_to_update = keys
    _, relowered = vx.lower_esdf(E, st2, ecfg())
    assert len(relowered) == 0


def test_update_empty_and_idempotent(vx):
    """esdf_test.cpp:308-344."""
    k, v = make_tsdf(16, lambda x, y, z: np.where(y == 4, 0.02, 0.2))
    T = gpu_tsdf(vx, k, v)
    E = vx.EsdfLayer(VS)
    vx.update_esdf(E, T, k, ecfg())
    before = E.export()
    assert len(vx.update_esdf(E, T, np.zeros((0, 3), np.int32), ecfg())) == 0
    assert layers_identical(*before, *E.export())
    assert len(vx.update_esdf(E, T, k, ecfg())) == 0
    assert layers_identical(*before, *E.export())
    E2 = vx.EsdfLayer(0.10)
    with pytest.raises(vx.InvalidArgumentError):
        vx.update_esdf(E2, T, k, ecfg())


def _oracle_tsdf(port, keys, vox):
    o = port.layer(A.LAYER_TSDF, VS)
    port.write_blocks(o, keys, vox)
    return o


def test_update_esdf_bitwise_vs_oracle_sphere_world(vx, port):
    """Incremental edits of a SphereWorld-style volume (fixtures.hpp:34-98)."""
    rng = np.random.default_rng(5)
    side = 32
    cfg = ecfg(max_distance=0.8)
    spheres = []
    E = vx.EsdfLayer(VS)
    Eo = port.layer(A.LAYER_ESDF, VS)
    T = vx.TsdfLayer(VS)
    To = port.layer(A.LAYER_TSDF, VS)
    prev = None
    for edit in range(6):
        ext = side * VS
        if not spheres or (len(spheres) < 6 and rng.uniform() < 0.6):
            spheres.append((rng.uniform(0.15 * ext, 0.85 * ext, 3), rng.uniform(0.08 * ext, 0.25 * ext)))
        else:
            spheres.pop(int(rng.integers(len(spheres))))

        def sdf(x, y, z):
            c = np.stack([(x + 0.5) * VS, (y + 0.5) * VS, (z + 0.5) * VS], -1)
            d = np.full(x.shape, 1e9)
            for cc, r in spheres:
                d = np.minimum(d, np.linalg.norm(c - cc, axis=-1) - r)
            return np.clip(d, -0.2, 0.2).astype(np.float32)
        keys, vox = make_tsdf(side, sdf)
        upd = keys if prev is None else keys[[vox[i].tobytes() != prev[i].tobytes() for i in range(len(keys))]]
        prev = vox
        T.write_blocks(keys, vox)
        port.write_blocks(To, keys, vox)
        a = vx.update_esdf(E, T, upd, cfg)
        b = port.update_esdf(Eo, To, upd, cfg)
        assert np.array_equal(a, b), edit
        ka, va = E.export()
        kb, vb = Eo.export()
        assert layers_identical(ka, va, kb, vb), edit
        # incremental == batch (esdf_test.cpp:377-398)
        Eb = vx.EsdfLayer(VS)
        vx.update_esdf(Eb, T, keys, cfg)
        assert layers_identical(ka, va, *Eb.export())


def test_pipeline_camera_esdf_bitwise(vx, port):
    """integrate_depth + update_esdf per frame (C1 scene, small frames)."""
    cam, seq = camera_frames("sphere_in_box", 160, 120, 4, 8)
    icfg = A.default_integrator_config(truncation=0.2)
    cfg = ecfg(site_threshold=0.05)
    T = vx.TsdfLayer(VS)
    E = vx.EsdfLayer(VS)
    To = port.layer(A.LAYER_TSDF, VS)
    Eo = port.layer(A.LAYER_ESDF, VS)
    for Tp, d in seq:
        ch = vx.BlockList()
        vx.integrate_depth(T, d, Tp, cam, icfg, out=ch)
        cho = port.integrate_camera(To, d, Tp, cam, icfg)
        assert np.array_equal(ch.numpy(), cho)
        a = vx.update_esdf(E, T, ch, cfg)  # device-resident changed list
        b = port.update_esdf(Eo, To, cho, cfg)
        assert np.array_equal(a, b)
    assert layers_identical(*E.export(), *Eo.export())


def test_c2_room_2cm_esdf_bitwise(vx, port):
    """BASELINE config C2 (first frames): room, 640x480, 2 cm, ESDF every frame."""
    cam, seq = camera_frames("room", 640, 480, 2, 100)
    icfg = A.default_integrator_config(truncation=0.08)
    cfg = A.default_esdf_config(site_threshold=0.02, max_distance=2.0)
    T = vx.TsdfLayer(0.02)
    E = vx.EsdfLayer(0.02)
    To = port.layer(A.LAYER_TSDF, 0.02)
    Eo = port.layer(A.LAYER_ESDF, 0.02)
    for Tp, d in seq:
        a = vx.integrate_depth(T, d, Tp, cam, icfg)
        b = port.integrate_camera(To, d, Tp, cam, icfg)
        assert np.array_equal(a, b)
        ea = vx.update_esdf(E, T, a, cfg)
        eb = port.update_esdf(Eo, To, b, cfg)
        assert np.array_equal(ea, eb)
    assert layers_identical(*E.export(), *Eo.export())


def test_phase_api_vs_oracle(vx, port):
    cam, seq = camera_frames("room", 160, 120, 3, 8)
    icfg = A.default_integrator_config(truncation=0.2)
    cfg = ecfg()
    T = vx.TsdfLayer(VS)
    E = vx.EsdfLayer(VS)
    To = port.layer(A.LAYER_TSDF, VS)
    Eo = port.layer(A.LAYER_ESDF, VS)
    for Tp, d in seq:
        a = vx.integrate_depth(T, d, Tp, cam, icfg)
        port.integrate_camera(To, d, Tp, cam, icfg)
        st, so = vx.EsdfUpdateState(), port.state()
        assert np.array_equal(vx.mark_sites(E, T, a, cfg, st), port.mark_sites(Eo, To, a, cfg, so))
        assert np.array_equal(st.indices_to_update, so.get(0))
        assert np.array_equal(st.indices_to_clear, so.get(1))
        assert np.array_equal(vx.clear_invalid(E, cfg, st), port.clear_invalid(Eo, cfg, so))
        assert np.array_equal(st.cleared_indices, so.get(2))
        ra, ca = vx.lower_esdf(E, st, cfg)
        rb, cb = port.lower_esdf(Eo, so, cfg)
        assert ra == rb
        assert np.array_equal(ca, cb)
        assert layers_identical(*E.export(), *Eo.export())


def test_query_bitwise_vs_oracle(vx, port):
    """integrate_test.cpp:490-534 shape; production evaluation order -> bitwise."""
    cam, seq = camera_frames("sphere_in_box", 128, 96, 3, 6)
    icfg = A.default_integrator_config(truncation=0.4)
    cfg = A.default_esdf_config(site_threshold=0.1)
    T, E = vx.TsdfLayer(0.1), vx.EsdfLayer(0.1)
    To, Eo = port.layer(A.LAYER_TSDF, 0.1), port.layer(A.LAYER_ESDF, 0.1)
    for Tp, d in seq:
        a = vx.integrate_depth(T, d, Tp, cam, icfg)
        vx.update_esdf(E, T, a, cfg)
        b = port.integrate_camera(To, d, Tp, cam, icfg)
        port.update_esdf(Eo, To, b, cfg)
    rng = np.random.default_rng(0x0ddba11)
    span = rng.uniform(-0.5, 3.5, (2000, 3))
    span[:, 2] = 0.3 + 0.6 * span[:, 2]
    span[0] = [np.nan, 0, 0]
    for interp in (True, False):
        qa = vx.query_batch(E, span, True, interp)
        qb = port.query_batch(Eo, span, True, A.QueryConfigC(int(interp), 1))
        assert qa.tobytes() == qb.tobytes()
        assert qa["known"].sum() > 200
