"""VXLF snapshots (core/serialization.hpp:29-35, serialization.cpp:20-158).

CPU: the reference's own save/load round trip through the oracle driver (pins
the binding).  GPU: the device layers' snapshot is byte-identical to the
reference's for the same map, files written by the reference load back into
device layers bit-exactly, and every IoError case of load_snapshot maps to
VXM_ERR_IO (IoError) with the reference's message.
"""
import struct

import numpy as np
import pytest

from paper_2311_00626_b200 import _abi as A
from tests.helpers import camera_frames, layers_identical


def _ref_maps(ref, vs=0.05):
    cam, seq = camera_frames("sphere_in_box", 160, 120, 2, 8)
    icfg = A.default_integrator_config(truncation=0.2)
    ecfg = A.default_esdf_config(site_threshold=0.05)
    T, E = ref.layer(A.LAYER_TSDF, vs), ref.layer(A.LAYER_ESDF, vs)
    for pose, d in seq:
        ch = ref.integrate_camera(T, d, pose, cam, icfg)
        ref.update_esdf(E, T, ch, ecfg)
    return T, E


def test_reference_snapshot_round_trip(ref, tmp_path):
    T, E = _ref_maps(ref)
    p = tmp_path / "a.vxlf"
    ref.save_snapshot(str(p), 0.05, T, E)
    raw = p.read_bytes()
    assert raw[:4] == b"VXLF" and struct.unpack("<I", raw[4:8])[0] == 1
    vs, T2, E2 = ref.load_snapshot(str(p))
    assert vs == 0.05
    assert layers_identical(*ref.export(T), *ref.export(T2))
    assert layers_identical(*ref.export(E), *ref.export(E2))


@pytest.mark.gpu
def test_snapshot_bytes_match_reference(vx, ref, tmp_path):
    To, Eo = _ref_maps(ref)
    T, E = vx.TsdfLayer(0.05), vx.EsdfLayer(0.05)
    T.write_blocks(*ref.export(To))
    E.write_blocks(*ref.export(Eo))
    ours, theirs = tmp_path / "ours.vxlf", tmp_path / "ref.vxlf"
    vx.save_snapshot(str(ours), 0.05, T, E)
    ref.save_snapshot(str(theirs), 0.05, To, Eo)
    assert ours.read_bytes() == theirs.read_bytes()
    # TSDF only / ESDF only
    vx.save_snapshot(str(ours), 0.05, tsdf=T)
    ref.save_snapshot(str(theirs), 0.05, To, None)
    assert ours.read_bytes() == theirs.read_bytes()


@pytest.mark.gpu
def test_snapshot_load_reference_file(vx, ref, tmp_path):
    To, Eo = _ref_maps(ref)
    p = tmp_path / "ref.vxlf"
    ref.save_snapshot(str(p), 0.05, To, Eo)
    vs, T, E = vx.load_snapshot(str(p))
    assert vs == 0.05
    assert layers_identical(*T.export(), *ref.export(To))
    assert layers_identical(*E.export(), *ref.export(Eo))
    # the loaded ESDF keeps working: one more frame matches the reference
    cam, seq = camera_frames("sphere_in_box", 160, 120, 1, 8, start=5)
    icfg = A.default_integrator_config(truncation=0.2)
    ecfg = A.default_esdf_config(site_threshold=0.05)
    pose, d = seq[0]
    a = vx.update_esdf(E, T, vx.integrate_depth(T, d, pose, cam, icfg), ecfg)
    b = ref.update_esdf(Eo, To, ref.integrate_camera(To, d, pose, cam, icfg), ecfg)
    assert np.array_equal(a, b)
    assert layers_identical(*E.export(), *ref.export(Eo))


@pytest.mark.gpu
@pytest.mark.parametrize("mutate,msg", [
    (lambda b: b"VXLX" + b[4:], "bad magic"),
    (lambda b: b[:4] + struct.pack("<I", 2) + b[8:], "unsupported version 2"),
    (lambda b: b[:8] + struct.pack("<d", 0.0) + b[16:], "invalid voxel size"),
    (lambda b: b[:-100], "truncated"),
    (lambda b: b[:20] + struct.pack("<I", 65) + b[24:], "layer name too long"),
])
def test_snapshot_load_errors(vx, ref, tmp_path, mutate, msg):
    To, _ = _ref_maps(ref)
    p = tmp_path / "ref.vxlf"
    ref.save_snapshot(str(p), 0.05, To, None)
    bad = tmp_path / "bad.vxlf"
    bad.write_bytes(mutate(p.read_bytes()))
    with pytest.raises(vx.IoError, match=msg):
        vx.load_snapshot(str(bad))
    with pytest.raises(Exception, match=msg):
        ref.load_snapshot(str(bad))


@pytest.mark.gpu
def test_snapshot_missing_file(vx, tmp_path):
    with pytest.raises(vx.IoError, match="cannot open"):
        vx.load_snapshot(str(tmp_path / "missing.vxlf"))
