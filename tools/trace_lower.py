"""Per-round phase timing of k_lower on C2 frames (VXM_TRACE_LOWER=1 must be set)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402
import paper_2311_00626_b200 as vx  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 10
sensor, frames, icfg, ecfg = bench.make_inputs(cfg, n)
c = bench.CONFIGS[cfg]
T = vx.TsdfLayer(c["vs"])
E = vx.EsdfLayer(c["vs"])
for i in range(n):
    ch = vx.integrate_depth(T, frames[i][1], frames[i][0], sensor, icfg)
    print(f"--- frame {i}: {len(ch)} changed", file=sys.stderr, flush=True)
    vx.update_esdf(E, T, ch, ecfg)
