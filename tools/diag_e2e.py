"""Per-call wall-clock breakdown of the host-API (e2e) path on C2 frames."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2311_00626_b200 as vx  # noqa: E402

sensor, frames, icfg, ecfg = bench.make_inputs("c2", 12)
pinned = [torch.from_numpy(d).pin_memory() for _, d in frames]
T = vx.TsdfLayer(0.02)
E = vx.EsdfLayer(0.02)
for i in range(12):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ch = vx.integrate_depth(T, pinned[i].numpy(), frames[i][0], sensor, icfg)
    t1 = time.perf_counter()
    ech = vx.update_esdf(E, T, ch, ecfg)
    t2 = time.perf_counter()
    print(f"frame {i}: integrate {1e3 * (t1 - t0):.3f} ms  update_esdf {1e3 * (t2 - t1):.3f} ms "
          f"({len(ch)} / {len(ech)} blocks)", flush=True)
