"""GPU parity: the ESDF quiet chain of k_lower_xr (Layer::stamp_quiet).

A block an update left untouched, whose round-1 reset_parented was the
identity (esdf/integrator.cpp:352-363), keeps the same bytes in both ESDF
pools, so the next update's round 1 skips it (no read, no copy) — as long as
nothing else wrote the layer in between.  The result must stay bit-identical
to the oracle's update_impl (esdf/integrator.cpp:365-413) through sequences
that keep the chain (repeated updates on a large, mostly far-field map) and
through every event that must break it: a user write of ESDF blocks, a change
of the limits (max_distance), pool growth, the phased API between updates.
"""
import numpy as np
import pytest

from paper_2311_00626_b200 import _abi as A
from tests.helpers import camera_frames, layers_identical

pytestmark = pytest.mark.gpu

VS = 0.04


def _frames(n):
    cam, seq = camera_frames("room", 320, 240, n, 16)
    return cam, seq


def _pair(vx, port):
    T, E = vx.TsdfLayer(VS), vx.EsdfLayer(VS)
    To, Eo = port.layer(A.LAYER_TSDF, VS), port.layer(A.LAYER_ESDF, VS)
    return T, E, To, Eo


def _step(vx, port, T, E, To, Eo, cam, pose, d, icfg, ecfg):
    a = vx.integrate_depth(T, d, pose, cam, icfg)
    b = port.integrate_camera(To, d, pose, cam, icfg)
    assert np.array_equal(a, b)
    ea = vx.update_esdf(E, T, a, ecfg)
    eb = port.update_esdf(Eo, To, b, ecfg)
    assert np.array_equal(ea, eb)


def test_chain_over_frames_and_repeats(vx, port):
    cam, seq = _frames(6)
    icfg = A.default_integrator_config(truncation=0.16)
    ecfg = A.default_esdf_config(site_threshold=0.04, max_distance=0.3)  # small: many far blocks
    T, E, To, Eo = _pair(vx, port)
    E.reserve(1 << 16)  # no growth: the chain holds from the second update on
    for pose, d in seq:
        _step(vx, port, T, E, To, Eo, cam, pose, d, icfg, ecfg)
        assert layers_identical(*E.export(), *Eo.export())
    # repeated updates of the same list: quiet blocks skipped, nothing changes
    keys = T.export()[0]
    for _ in range(2):
        assert np.array_equal(vx.update_esdf(E, T, keys, ecfg), port.update_esdf(Eo, To, keys, ecfg))
    assert layers_identical(*E.export(), *Eo.export())


def test_chain_breaks_on_user_write_limits_and_phases(vx, port):
    cam, seq = _frames(5)
    icfg = A.default_integrator_config(truncation=0.16)
    ecfg = A.default_esdf_config(site_threshold=0.04, max_distance=0.3)
    T, E, To, Eo = _pair(vx, port)
    E.reserve(1 << 16)
    for pose, d in seq[:2]:
        _step(vx, port, T, E, To, Eo, cam, pose, d, icfg, ecfg)
    # a user write of ESDF blocks: some far-field blocks get a parented voxel
    ke, ve = E.export()
    pick = np.arange(0, len(ke), max(1, len(ke) // 40))
    w = ve[pick].copy()
    obs = (w["flags"] & 1) != 0
    for i in range(len(pick)):
        j = np.flatnonzero(obs[i] & ((w["flags"][i] & 2) == 0))
        if len(j):
            v = j[0]
            w[i]["parent_x"][v] = 1
            w[i]["squared_distance"][v] = 1
    E.write_blocks(ke[pick], w)
    port.write_blocks(Eo, ke[pick], w)
    assert layers_identical(*E.export(), *Eo.export())
    _step(vx, port, T, E, To, Eo, cam, seq[2][0], seq[2][1], icfg, ecfg)
    assert layers_identical(*E.export(), *Eo.export())
    # other limits: the reset of far blocks differs
    ecfg2 = A.default_esdf_config(site_threshold=0.04, max_distance=0.5)
    _step(vx, port, T, E, To, Eo, cam, seq[3][0], seq[3][1], icfg, ecfg2)
    assert layers_identical(*E.export(), *Eo.export())
    # the phased API between two updates (mark_sites / clear_invalid / lower_esdf)
    keys = T.export()[0][:200]
    st = vx.EsdfUpdateState()
    sto = port.state()
    assert np.array_equal(vx.mark_sites(E, T, keys, ecfg2, st), port.mark_sites(Eo, To, keys, ecfg2, sto))
    assert np.array_equal(vx.clear_invalid(E, ecfg2, st), port.clear_invalid(Eo, ecfg2, sto))
    assert layers_identical(*E.export(), *Eo.export())
    _step(vx, port, T, E, To, Eo, cam, seq[4][0], seq[4][1], icfg, ecfg2)
    assert layers_identical(*E.export(), *Eo.export())


def test_chain_breaks_on_pool_growth(vx, port):
    # no reservation: the ESDF pool grows while the map grows (the scratch
    # pool's blocks are not kept across growth)
    cam, seq = camera_frames("room", 320, 240, 6, 16)
    icfg = A.default_integrator_config(truncation=0.16)
    ecfg = A.default_esdf_config(site_threshold=0.04, max_distance=0.3)
    T, E, To, Eo = _pair(vx, port)
    for pose, d in seq:
        _step(vx, port, T, E, To, Eo, cam, pose, d, icfg, ecfg)
    assert layers_identical(*E.export(), *Eo.export())


def test_mark_skip_source_writes_and_switch(vx, port):
    """k_mark skips effective blocks whose TSDF block is unchanged since their
    last marking (Layer::mark_stamp): a host write of TSDF blocks, and a switch
    of the source layer, must make them marked again (mark_impl,
    esdf/integrator.cpp:268-348, marks every effective block)."""
    cam, seq = _frames(5)
    icfg = A.default_integrator_config(truncation=0.16)
    ecfg = A.default_esdf_config(site_threshold=0.04, max_distance=0.3)
    T, E, To, Eo = _pair(vx, port)
    E.reserve(1 << 16)
    for pose, d in seq[:3]:
        _step(vx, port, T, E, To, Eo, cam, pose, d, icfg, ecfg)
    # host write of TSDF blocks (a surface sheet moved): then an update whose
    # list names only some of them — the others are effective as neighbours
    kt, vt = T.export()
    pick = kt[::7]
    w = vt[::7].copy()
    w["distance"] = np.where(w["weight"] > 0, -w["distance"], w["distance"])
    T.write_blocks(pick, w)
    port.write_blocks(To, pick, w)
    listed = pick[::3]
    assert np.array_equal(vx.update_esdf(E, T, listed, ecfg), port.update_esdf(Eo, To, listed, ecfg))
    assert layers_identical(*E.export(), *Eo.export())
    # another source layer, then back (the blocks' flags follow each source)
    T2, To2 = vx.TsdfLayer(VS), port.layer(A.LAYER_TSDF, VS)
    a = vx.integrate_depth(T2, seq[3][1], seq[3][0], cam, icfg)
    b = port.integrate_camera(To2, seq[3][1], seq[3][0], cam, icfg)
    assert np.array_equal(vx.update_esdf(E, T2, a, ecfg), port.update_esdf(Eo, To2, b, ecfg))
    keys = T.export()[0]
    assert np.array_equal(vx.update_esdf(E, T, keys, ecfg), port.update_esdf(Eo, To, keys, ecfg))
    assert layers_identical(*E.export(), *Eo.export())
    # another site threshold
    ecfg2 = A.default_esdf_config(site_threshold=0.06, max_distance=0.3)
    assert np.array_equal(vx.update_esdf(E, T, keys, ecfg2), port.update_esdf(Eo, To, keys, ecfg2))
    assert layers_identical(*E.export(), *Eo.export())
    _step(vx, port, T, E, To, Eo, cam, seq[4][0], seq[4][1], icfg, ecfg2)
    assert layers_identical(*E.export(), *Eo.export())
