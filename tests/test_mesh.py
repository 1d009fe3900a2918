"""Color fusion and marching-cubes meshing.

Reference: integrate_color (proj/src/integrate/integrator.cpp:191-273,
color_update updates.hpp:74-92); mesh_block / update_mesh
(src/mesh/marching_cubes.cpp:95-242) with the Lorensen-Cline tables
(marching_cubes_tables.cpp); save_mesh_ply (src/mesh/ply.cpp:33-105); the
color layer of the VXLF snapshot (serialization.cpp:98-104).  Tests mirror
proj/tests/mesh_test.cpp and integrate_test.cpp:365-445.

CPU: the packed triangle table the kernel reads equals the reference's table
and uses exactly the crossed edges (mesh_test.cpp:98-125).  GPU: every
MeshBlock (vertex order, positions, normals, colors, triangles), every color
voxel, the changed / re-meshed lists and the PLY bytes equal the reference's
build bit for bit.
"""
import os
import re

import numpy as np
import pytest

from paper_2311_00626_b200 import _abi as A
from tests.helpers import camera_frames, layers_identical

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CORNERS = [(0, 0, 0), (1, 0, 0), (1, 1, 0), (0, 1, 0), (0, 0, 1), (1, 0, 1), (1, 1, 1), (0, 1, 1)]
EDGES = [(0, 1), (1, 2), (2, 3), (3, 0), (4, 5), (5, 6), (6, 7), (7, 4), (0, 4), (1, 5), (2, 6), (3, 7)]


def _packed_table():
    src = open(os.path.join(ROOT, "paper_2311_00626_b200", "csrc", "mc_table.cuh")).read()
    vals = [int(v, 16) for v in re.findall(r"0x([0-9a-f]{16})ull", src)]
    assert len(vals) == 256
    rows = []
    for v in vals:
        n = 3 * (v >> 60)
        rows.append([(v >> (4 * k)) & 15 for k in range(n)])
    return rows


def _fill_region(n_side, vs, trunc, sdf):
    """mesh_test.cpp:66-86: n^3 blocks, clamped SDF at voxel centres, weight 1."""
    keys, vox = [], []
    lin = np.arange(512)
    for bx in range(n_side):
        for by in range(n_side):
            for bz in range(n_side):
                gx, gy, gz = 8 * bx + (lin & 7), 8 * by + ((lin >> 3) & 7), 8 * bz + (lin >> 6)
                c = ((gx + 0.5) * vs, (gy + 0.5) * vs, (gz + 0.5) * vs)
                v = np.zeros(512, A.TSDF_DTYPE)
                v["distance"] = np.clip(sdf(*c), -trunc, trunc).astype(np.float32)
                v["weight"] = 1.0
                keys.append((bx, by, bz))
                vox.append(v)
    order = np.lexsort(np.array(keys).T[::-1])
    return np.array(keys, np.int32)[order], np.stack(vox)[order]


def _sphere(c, r):
    return lambda x, y, z: np.sqrt((x - c[0]) ** 2 + (y - c[1]) ** 2 + (z - c[2]) ** 2) - r


def _same_block(ours, theirs):
    """ours: MeshBlock; theirs: (vertices, normals, colors, triangles)."""
    v, n, c, t = theirs
    return (ours.vertices.tobytes() == v.tobytes() and ours.normals.tobytes() == n.tobytes()
            and ours.colors.tobytes() == c.tobytes() and ours.triangles.tobytes() == t.tobytes())


def _same_mesh(vx_mesh, ref_mesh):
    ka, kb = vx_mesh.sorted_indices(), ref_mesh.sorted_indices()
    if not np.array_equal(ka, kb):
        return False
    return all(_same_block(vx_mesh.block(g), ref_mesh.block(g)) for g in ka)


# ---- CPU ------------------------------------------------------------------------

def test_packed_triangle_table_matches_reference_and_crossed_edges(ref):
    rows = _packed_table()
    tri = ref.mc_tri_table()
    for c in range(256):
        want = [int(e) for e in tri[c] if e != -1]
        assert rows[c] == want, c
        crossed = 0
        for e, (a, b) in enumerate(EDGES):
            if ((c >> a) & 1) != ((c >> b) & 1):
                crossed |= 1 << e
        used = 0
        for e in rows[c]:
            used |= 1 << e
        assert used == crossed and len(rows[c]) % 3 == 0 and len(rows[c]) <= 15


def test_reference_mesh_watertight_sphere(ref):
    """mesh_test.cpp:213-253 on the reference build (pins the bindings)."""
    keys, vox = _fill_region(1, 0.05, 0.2, _sphere((0.21, 0.19, 0.2), 0.12))
    T = ref.layer(A.LAYER_TSDF, 0.05)
    ref.write_blocks(T, keys, vox)
    M = ref.mesh_layer(0.05)
    v, n, c, t = ref.mesh_block(M, T, (0, 0, 0))
    directed = {}
    for tri in t:
        for k in range(3):
            e = (int(tri[k]), int(tri[(k + 1) % 3]))
            directed[e] = directed.get(e, 0) + 1
    assert all(cnt == 1 and (b, a) in directed for (a, b), cnt in directed.items())
    assert len(v) - len(directed) // 2 + len(t) == 2


# ---- GPU ------------------------------------------------------------------------

@pytest.mark.gpu
@pytest.mark.parametrize("case", ["plane", "sphere8", "sphere1", "positive"])
def test_gpu_mesh_blocks_bitwise(vx, ref, case):
    if case == "plane":      # mesh_test.cpp:144-161
        vs, trunc, n, sdf = 0.05, 0.1, 2, (lambda x, y, z: z - 0.253)
    elif case == "sphere8":  # mesh_test.cpp:163-211
        vs, trunc, n, sdf = 0.02, 0.08, 8, _sphere((0.655, 0.662, 0.649), 0.5)
    elif case == "sphere1":  # mesh_test.cpp:213-253
        vs, trunc, n, sdf = 0.05, 0.2, 1, _sphere((0.21, 0.19, 0.2), 0.12)
    else:                    # mesh_test.cpp:127-137
        vs, trunc, n, sdf = 0.05, 0.2, 1, (lambda x, y, z: 0.1 + 0 * x)
    keys, vox = _fill_region(n, vs, trunc, sdf)
    T, R = vx.TsdfLayer(vs), ref.layer(A.LAYER_TSDF, vs)
    T.write_blocks(keys, vox)
    ref.write_blocks(R, keys, vox)
    M, RM = vx.MeshLayer(vs), ref.mesh_layer(vs)
    a = vx.update_mesh(M, T, keys)
    b = ref.update_mesh(RM, R, keys)
    assert np.array_equal(a, b)
    assert _same_mesh(M, RM)
    blk = vx.mesh_block(vx.MeshLayer(vs), T, (0, 0, 0))
    assert _same_block(blk, ref.mesh_block(ref.mesh_layer(vs), R, (0, 0, 0)))
    if case == "positive":
        assert blk.empty() and len(blk.vertices) == 0
    if case == "plane":
        assert np.all(np.abs(blk.vertices[:, 2].astype(np.float64) - 0.253) <= 1e-6 * trunc)
        assert np.all(blk.normals[:, 2] > 0.99)


@pytest.mark.gpu
def test_gpu_mesh_errors_and_partial_updates(vx, ref):
    T = vx.TsdfLayer(0.05)
    with pytest.raises(vx.InvalidArgumentError, match="not allocated"):
        vx.mesh_block(vx.MeshLayer(0.05), T, (0, 0, 0))  # mesh_test.cpp:139-142
    keys, vox = _fill_region(3, 0.05, 0.15, _sphere((0.6, 0.6, 0.6), 0.3))
    R = ref.layer(A.LAYER_TSDF, 0.05)
    T.write_blocks(keys, vox)
    ref.write_blocks(R, keys, vox)
    M, RM = vx.MeshLayer(0.05), ref.mesh_layer(0.05)
    vx.update_mesh(M, T, keys)
    ref.update_mesh(RM, R, keys)
    assert len(vx.update_mesh(M, T, np.zeros((0, 3), np.int32))) == 0  # mesh_test.cpp:265-267
    before = M.block((2, 2, 2))
    got = vx.update_mesh(M, T, [(1, 1, 1)])  # mesh_test.cpp:269-277
    assert [tuple(g) for g in got] == [(0, 1, 1), (1, 0, 1), (1, 1, 0), (1, 1, 1)]
    assert np.array_equal(got, ref.update_mesh(RM, R, [(1, 1, 1)]))
    assert _same_block(M.block((2, 2, 2)), (before.vertices, before.normals, before.colors,
                                            before.triangles))
    assert _same_mesh(M, RM)


@pytest.mark.gpu
def test_gpu_incremental_mesh_matches_reference_on_frames(vx, ref):
    """update_mesh on the changed lists of real integrations (partial corners,
    unobserved voxels), the replay pipeline's use (pipeline.cpp:79-84)."""
    cam, seq = camera_frames("room", 320, 240, 4, 16)
    cfg = A.default_integrator_config(truncation=0.16)
    T, R = vx.TsdfLayer(0.04), ref.layer(A.LAYER_TSDF, 0.04)
    M, RM = vx.MeshLayer(0.04), ref.mesh_layer(0.04)
    for pose, d in seq:
        a = vx.integrate_depth(T, d, pose, cam, cfg)
        b = ref.integrate_camera(R, d, pose, cam, cfg)
        assert np.array_equal(a, b)
        assert np.array_equal(vx.update_mesh(M, T, a), ref.update_mesh(RM, R, b))
    assert M.num_blocks() > 50
    assert _same_mesh(M, RM)


@pytest.mark.gpu
@pytest.mark.parametrize("scene,w,h,vs,trunc,frames,orbit", [
    ("sphere_in_box", 96, 72, 0.05, 0.2, 3, 8),     # integrate_test.cpp:365-410
    ("room", 640, 480, 0.02, 0.08, 2, 100),
])
def test_gpu_color_fusion_and_colored_mesh(vx, ref, scene, w, h, vs, trunc, frames, orbit):
    cam, seq = camera_frames(scene, w, h, frames, orbit)
    cfg = A.default_integrator_config(truncation=trunc)
    T, R = vx.TsdfLayer(vs), ref.layer(A.LAYER_TSDF, vs)
    Cl, RC = vx.ColorLayer(vs), ref.layer(A.LAYER_COLOR, vs)
    changed = np.zeros((0, 3), np.int32)
    for pose, d in seq:
        rgb = ref.render_color(scene, pose, cam)
        a = vx.integrate_depth(T, d, pose, cam, cfg)
        ref.integrate_camera(R, d, pose, cam, cfg)
        ca = vx.integrate_color(Cl, rgb, d, pose, cam, T, cfg)
        cb = ref.integrate_color(RC, rgb, d, pose, cam, R, cfg)
        assert len(ca) and np.array_equal(ca, cb)
        changed = np.unique(np.concatenate([changed, a]), axis=0)
    assert layers_identical(*Cl.export(), *ref.export(RC))
    # every colored voxel sits in the observed band of the TSDF
    kc, vc = Cl.export()
    kt, vt = T.export()
    idx = {tuple(k): i for i, k in enumerate(kt)}
    for k, blk in zip(kc, vc):
        tv = vt[idx[tuple(k)]]
        m = blk["weight"] > 0
        assert np.all(tv["weight"][m] > 0) and np.all(np.abs(tv["distance"][m]) <= np.float32(trunc))
    M, RM = vx.MeshLayer(vs), ref.mesh_layer(vs)
    assert np.array_equal(vx.update_mesh(M, T, changed, color=Cl),
                          ref.update_mesh(RM, R, changed, color=RC))
    assert _same_mesh(M, RM)
    assert any(len(M.block(g).colors) for g in M.sorted_indices())


@pytest.mark.gpu
def test_gpu_color_errors(vx):
    cam, seq = camera_frames("sphere_in_box", 96, 72, 1, 8)
    pose, d = seq[0]
    T, Cl = vx.TsdfLayer(0.05), vx.ColorLayer(0.05)
    rgb = np.zeros((72, 96, 3), np.uint8)
    with pytest.raises(vx.InvalidArgumentError, match="image size"):
        vx.integrate_color(Cl, rgb[:, :90], d, pose, cam, T)
    with pytest.raises(vx.InvalidArgumentError, match="depth size mismatch"):
        vx.integrate_color(Cl, rgb, d[:, :90], pose, cam, T)
    assert Cl.num_blocks() == 0


@pytest.mark.gpu
def test_gpu_ply_and_color_snapshot_bytes_match_reference(vx, ref, tmp_path):
    """mesh_test.cpp:304-355 (PLY) and the color layer's VXLF record."""
    cam, seq = camera_frames("sphere_in_box", 96, 72, 2, 8)
    cfg = A.default_integrator_config(truncation=0.2)
    T, R = vx.TsdfLayer(0.05), ref.layer(A.LAYER_TSDF, 0.05)
    Cl, RC = vx.ColorLayer(0.05), ref.layer(A.LAYER_COLOR, 0.05)
    for pose, d in seq:
        rgb = ref.render_color("sphere_in_box", pose, cam)
        vx.integrate_depth(T, d, pose, cam, cfg)
        ref.integrate_camera(R, d, pose, cam, cfg)
        vx.integrate_color(Cl, rgb, d, pose, cam, T, cfg)
        ref.integrate_color(RC, rgb, d, pose, cam, R, cfg)
    keys = T.sorted_indices()
    for color in (False, True):
        M, RM = vx.MeshLayer(0.05), ref.mesh_layer(0.05)
        vx.update_mesh(M, T, keys, color=Cl if color else None)
        ref.update_mesh(RM, R, keys, color=RC if color else None)
        ours, theirs = tmp_path / f"o{color}.ply", tmp_path / f"r{color}.ply"
        vx.save_mesh_ply(M, str(ours))
        ref.save_mesh_ply(RM, str(theirs))
        assert ours.read_bytes() == theirs.read_bytes()
        raw = ours.read_bytes()
        assert b"format binary_little_endian 1.0\n" in raw
        assert (b"property uchar red" in raw) == color
    with pytest.raises(vx.IoError):
        vx.save_mesh_ply(M, str(tmp_path / "no" / "such" / "dir.ply"))
    ours, theirs = tmp_path / "o.vxlf", tmp_path / "r.vxlf"
    vx.save_snapshot(str(ours), 0.05, T, None, color=Cl)
    ref.save_snapshot(str(theirs), 0.05, R, None, color=RC)
    assert ours.read_bytes() == theirs.read_bytes()
    vs, t, c, e = vx.load_snapshot(str(theirs), with_color=True)
    assert e is None and layers_identical(*c.export(), *ref.export(RC))
