"""GPU: host key lists through vxm_update_esdf (esdf/integrator.hpp:113-120).

The host list is range-checked, packed and order-checked on the host cores
(BlockList::assign_host; lists of >= 65536 keys in parallel) before any
mutation.  A list in any order, with repeats, must give the same result as
its sorted unique form (update_impl sorts the seeds, esdf/integrator.cpp:
500-505), and a key outside +-2^20 must be rejected before anything changes
(layer.hpp's MapCapacityError / invalid_argument class).
"""
import numpy as np
import pytest

from paper_2311_00626_b200 import _abi as A
from tests.helpers import camera_frames, layers_identical

pytestmark = pytest.mark.gpu


def _map(vx):
    cam, seq = camera_frames("room", 320, 240, 2, 16)
    icfg = A.default_integrator_config(truncation=0.16)
    T = vx.TsdfLayer(0.04)
    upd = None
    for pose, d in seq:
        upd = vx.integrate_depth(T, d, pose, cam, icfg)
    return T, upd


def _big_list(upd, rng):
    # the updated keys plus ~70k keys of no TSDF block, shuffled, with repeats
    extra = rng.integers(-5000, 5000, size=(70000, 3)).astype(np.int32)
    keys = np.concatenate([upd, extra, upd[: len(upd) // 2]])
    return keys[rng.permutation(len(keys))]


def test_large_unsorted_list_matches_sorted(vx):
    rng = np.random.default_rng(7)
    T, upd = _map(vx)
    ecfg = A.default_esdf_config(site_threshold=0.04, max_distance=1.0)
    keys = _big_list(upd, rng)
    assert len(keys) >= 65536
    srt = np.unique(keys, axis=0)  # row-lexicographic == GridIndex order
    E1, E2 = vx.EsdfLayer(0.04), vx.EsdfLayer(0.04)
    c1 = vx.update_esdf(E1, T, keys, ecfg)
    c2 = vx.update_esdf(E2, T, srt, ecfg)
    assert np.array_equal(c1, c2)
    assert layers_identical(*E1.export(), *E2.export())
    # sorted input the second time (the order check's other outcome)
    c1 = vx.update_esdf(E1, T, srt, ecfg)
    c2 = vx.update_esdf(E2, T, keys, ecfg)
    assert np.array_equal(c1, c2)
    assert layers_identical(*E1.export(), *E2.export())


@pytest.mark.parametrize("n_extra", [10, 70000])
def test_out_of_range_key_rejected_before_mutation(vx, n_extra):
    rng = np.random.default_rng(3)
    T, upd = _map(vx)
    ecfg = A.default_esdf_config(site_threshold=0.04, max_distance=1.0)
    E = vx.EsdfLayer(0.04)
    vx.update_esdf(E, T, upd, ecfg)
    before = E.export()
    extra = rng.integers(-100, 100, size=(n_extra, 3)).astype(np.int32)
    bad = np.concatenate([upd, extra])
    bad[len(bad) // 2] = (1 << 20, 0, 0)  # x beyond +2^20 - 1
    with pytest.raises(vx.InvalidArgumentError):
        vx.update_esdf(E, T, bad, ecfg)
    assert layers_identical(*before, *E.export())
    bad[len(bad) // 2] = (0, -(1 << 20) - 1, 0)  # y below -2^20
    with pytest.raises(vx.InvalidArgumentError):
        vx.update_esdf(E, T, bad, ecfg)
    assert layers_identical(*before, *E.export())
