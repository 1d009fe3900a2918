"""Per-frame timing of the fused device path vs the two-call device path (C2)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2311_00626_b200 as vx  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 12
sensor, frames, icfg, ecfg = bench.make_inputs(cfg, n)
c = bench.CONFIGS[cfg]
ctx = vx.Context(0)
ext = torch.cuda.ExternalStream(ctx.stream)
dev = torch.from_numpy(np.stack([d for _, d in frames])).cuda()
H, W = dev.shape[1], dev.shape[2]
for mode in ("fused", "two-call"):
    T, E = vx.TsdfLayer(c["vs"], ctx=ctx), vx.EsdfLayer(c["vs"], ctx=ctx)
    tch, ech = vx.BlockList(ctx), vx.BlockList(ctx)
    for i in range(n):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(ext)
        if mode == "fused":
            vx.update_frame_device(T, E, dev[i].data_ptr(), W, H, frames[i][0], sensor, icfg, ecfg, tch, ech)
        else:
            vx.integrate_depth_device(T, dev[i].data_ptr(), W, H, frames[i][0], sensor, icfg, tch)
            vx.update_esdf_device(E, T, tch, ecfg, ech)
        e1.record(ext)
        e1.synchronize()
        t1 = time.perf_counter()
        print(f"{mode} frame {i}: host {1e3 * (t1 - t0):.3f} ms, device {e0.elapsed_time(e1):.3f} ms",
              flush=True)
