"""Times one in-process sharded update_esdf (P shards on this GPU) of a
SphereWorld volume: fused persistent kernel vs host-driven rounds
(VXM_SHARD_FUSED), next to the single-map update."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2311_00626_b200 as vx  # noqa: E402
from paper_2311_00626_b200 import _abi as A  # noqa: E402
from paper_2311_00626_b200 import synth  # noqa: E402

side = int(sys.argv[1]) if len(sys.argv) > 1 else 256
P = int(sys.argv[2]) if len(sys.argv) > 2 else 2
slab = 8
keys, va = synth.sphere_world(side, 0.02, 0.08, seed=2311)
_, vb = synth.sphere_world(side, 0.02, 0.08, seed=2312)
cfg = A.default_esdf_config(site_threshold=0.02, max_distance=2.0)
own = (keys[:, 0] // slab) % P
ctxs = []
for p in range(P):
    c = vx.Context(0)
    c.set_shard(p, P, slab)
    ctxs.append(c)
Ts = [[vx.TsdfLayer(0.02, ctx=c) for c in ctxs] for _ in range(2)]
for p in range(P):
    Ts[0][p].write_blocks(keys[own == p], va[own == p])
    Ts[1][p].write_blocks(keys[own == p], vb[own == p])
Es = [vx.EsdfLayer(0.02, ctx=c) for c in ctxs]
upd = [keys[own == p] for p in range(P)]
times = []
for i in range(6):
    t0 = time.perf_counter()
    vx.update_esdf_sharded(Es, Ts[i % 2], upd, cfg)
    times.append(time.perf_counter() - t0)
st = ctxs[0].stats()
mode = "host-driven" if os.environ.get("VXM_SHARD_FUSED") == "0" else "fused"
print(f"{side}^3 P={P} {mode}: {1e3 * np.median(times[2:]):.2f} ms per sharded update "
      f"(rounds/update {st['lower_rounds'] / max(st['esdf_calls'], 1):.1f})")
