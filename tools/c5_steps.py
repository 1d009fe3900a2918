"""Runs N full update_esdf calls of the C5 512^3 volume (for ncu captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
import paper_2311_00626_b200 as vx  # noqa: E402
from paper_2311_00626_b200 import _abi as A  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 3
side = int(sys.argv[2]) if len(sys.argv) > 2 else bench.C5_SIDE
keys, va, vb = bench.c5_volumes(side)
ctx = vx.Context(0)
Ts = [vx.TsdfLayer(0.02, ctx=ctx), vx.TsdfLayer(0.02, ctx=ctx)]
Ts[0].write_blocks(keys, va)
Ts[1].write_blocks(keys, vb)
cfg = A.default_esdf_config(site_threshold=0.02, max_distance=2.0)
upd, out = vx.BlockList(ctx), vx.BlockList(ctx)
upd.assign(keys)
E = vx.EsdfLayer(0.02, ctx=ctx)
for i in range(n):
    vx.update_esdf_device(E, Ts[i % 2], upd, cfg, out)
ctx.synchronize()
print("done", file=sys.stderr)
