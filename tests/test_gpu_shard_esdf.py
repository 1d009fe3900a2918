"""GPU parity: block-sharded ESDF update (vxm_update_esdf_sharded).

P shards (one context each, on the same B200 here; across GPUs the peer
accesses become NVLink transfers) own the blocks with floor(x / slab) mod P == p.
By default the whole round loop runs in one persistent kernel per shard with
the face exchange over peer memory (k_shard_fused); VXM_SHARD_FUSED=0 selects
the host-driven rounds (event-ordered peer copies), run by the last test in a
subprocess.
Every frame is integrated by every shard (each keeps its own blocks) and by a
single map; the shards' ESDF update must reproduce update_esdf over the single
map bit-for-bit: the union of their changed lists and of their ESDF layers.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_2311_00626_b200 import _abi as A
from paper_2311_00626_b200 import synth
from tests.helpers import camera_frames, layers_identical

pytestmark = pytest.mark.gpu


def _owner(x, P, slab):
    return (np.floor_divide(x, slab) % P).astype(int)


def _union(layers):
    ks, vs = zip(*[L.export() for L in layers])
    k = np.concatenate(ks)
    v = np.concatenate(vs)
    order = np.lexsort((k[:, 2], k[:, 1], k[:, 0]))
    return k[order], v[order]


def _sorted_union(lists):
    k = np.concatenate([np.asarray(x).reshape(-1, 3) for x in lists])
    if len(k) == 0:
        return k
    return k[np.lexsort((k[:, 2], k[:, 1], k[:, 0]))]


def _shards(vx, P, slab, vs):
    ctxs = []
    for p in range(P):
        c = vx.Context(0)
        c.set_shard(p, P, slab)
        ctxs.append(c)
    return ctxs, [vx.TsdfLayer(vs, ctx=c) for c in ctxs], [vx.EsdfLayer(vs, ctx=c) for c in ctxs]


@pytest.mark.parametrize("P,slab", [(2, 3), (3, 2), (2, 1)])
def test_sharded_esdf_frames_equal_single_map(vx, P, slab):
    vs = 0.04
    cam, seq = camera_frames("room", 320, 240, 4, 16)
    icfg = A.default_integrator_config(truncation=0.16)
    ecfg = A.default_esdf_config(site_threshold=0.04, max_distance=1.0)
    T, E = vx.TsdfLayer(vs), vx.EsdfLayer(vs)
    ctxs, Ts, Es = _shards(vx, P, slab, vs)
    for pose, d in seq:
        a = vx.integrate_depth(T, d, pose, cam, icfg)
        parts = [vx.integrate_depth(Ts[p], d, pose, cam, icfg) for p in range(P)]
        for p in range(P):
            assert np.all(_owner(parts[p][:, 0], P, slab) == p) if len(parts[p]) else True
        assert np.array_equal(_sorted_union(parts), a)
        ea = vx.update_esdf(E, T, a, ecfg)
        eb = vx.update_esdf_sharded(Es, Ts, parts, ecfg)
        assert np.array_equal(_sorted_union(eb), ea)
    assert layers_identical(*_union(Es), *E.export())
    assert layers_identical(*_union(Ts), *T.export())


def test_sharded_esdf_dense_volume(vx):
    """C5-style dense volume split across 4 shards (slab 2 blocks)."""
    P, slab, vs = 4, 2, 0.02
    keys, vox = synth.sphere_world(128, vs, 0.08)
    cfg = A.default_esdf_config(site_threshold=0.02, max_distance=2.0)
    T, E = vx.TsdfLayer(vs), vx.EsdfLayer(vs)
    T.write_blocks(keys, vox)
    ea = vx.update_esdf(E, T, keys, cfg)
    ctxs, Ts, Es = _shards(vx, P, slab, vs)
    own = _owner(keys[:, 0], P, slab)
    for p in range(P):
        Ts[p].write_blocks(keys[own == p], vox[own == p])
    eb = vx.update_esdf_sharded(Es, Ts, [keys[own == p] for p in range(P)], cfg)
    assert np.array_equal(_sorted_union(eb), ea)
    assert layers_identical(*_union(Es), *E.export())
    # second update with the same input: nothing changes anywhere
    assert all(len(x) == 0 for x in vx.update_esdf_sharded(Es, Ts, [keys[own == p] for p in range(P)], cfg))


def test_sharded_esdf_rejects_misconfigured_contexts(vx):
    c0, c1 = vx.Context(0), vx.Context(0)
    c0.set_shard(0, 2, 4)
    c1.set_shard(0, 2, 4)  # wrong rank
    Ts = [vx.TsdfLayer(0.05, ctx=c) for c in (c0, c1)]
    Es = [vx.EsdfLayer(0.05, ctx=c) for c in (c0, c1)]
    with pytest.raises(vx.InvalidArgumentError):
        vx.update_esdf_sharded(Es, Ts, [np.zeros((1, 3), np.int32)] * 2, A.default_esdf_config())


def test_sharded_host_driven_rounds_bitwise():
    """The same tests through the host-driven round loop (VXM_SHARD_FUSED=0)."""
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.abspath(__file__), "-q", "-x", "-m", "gpu",
                        "-k", "not host_driven"], env={**os.environ, "VXM_SHARD_FUSED": "0"},
                       capture_output=True, text=True, timeout=900,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
