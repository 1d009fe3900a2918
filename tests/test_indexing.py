"""Index algebra KATs (proj/tests/core_test.cpp:30-71) on the
Python mirror, plus its agreement with the C restatement's voxel centres."""
import numpy as np

import paper_2311_00626_b200 as vx


def test_position_to_indices_floor_semantics():
    vs = 0.05
    for p, g, v in (((0.0, 0.0, 0.0), (0, 0, 0), (0, 0, 0)),
                    ((-0.01, 0.0, 0.0), (-1, 0, 0), (7, 0, 0)),
                    ((0.43, 0.05, -0.40), (1, 0, -1), (0, 1, 0))):
        gb, vb = vx.position_to_indices(np.array(p), vs)
        assert tuple(gb) == g and tuple(vb) == v


def test_voxel_center_inverts_position_to_indices():
    vs = 0.05
    assert tuple(vx.voxel_center([0, 0, 0], [0, 0, 0], vs)) == (0.025, 0.025, 0.025)
    assert tuple(vx.voxel_center([-1, 0, 0], [7, 0, 0], vs)) == (-0.025, 0.025, 0.025)
    rng = np.random.default_rng(7)
    g = rng.integers(-50, 51, (1000, 3))
    v = rng.integers(0, 8, (1000, 3))
    gb, vb = vx.position_to_indices(vx.voxel_center(g, v, vs), vs)
    assert np.array_equal(gb, g) and np.array_equal(vb, v)
    assert np.array_equal(vx.voxel_index_from_linear(vx.linear_voxel_index(v)), v)
    gv = vx.global_voxel_index(g, v)
    assert np.array_equal(vx.block_of_global_voxel(gv), g)
    assert np.array_equal(vx.local_voxel_of_global(gv), v)
    assert np.array_equal(vx.linear_voxel_index(np.array([[1, 2, 3]])), [1 + 8 * (2 + 8 * 3)])
