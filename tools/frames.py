"""Runs N fused frames of a bench config (for ncu / profiling captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2311_00626_b200 as vx  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 8
sensor, frames, icfg, ecfg = bench.make_inputs(cfg, n)
c = bench.CONFIGS[cfg]
ctx = vx.Context(0)
dev = torch.from_numpy(np.stack([d for _, d in frames])).cuda()
torch.cuda.synchronize()
T = vx.TsdfLayer(c["vs"], ctx=ctx)
E = vx.EsdfLayer(c["vs"], ctx=ctx) if ecfg else None
tch, ech = vx.BlockList(ctx), vx.BlockList(ctx)
for i in range(n):
    vx.update_frame_device(T, E, dev[i].data_ptr(), dev.shape[2], dev.shape[1], frames[i][0], sensor,
                           icfg, ecfg, tch, ech if E is not None else None)
print("launches", ctx.launch_count, file=sys.stderr)
