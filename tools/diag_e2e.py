"""Per-call wall-clock vs device-time breakdown of the host-API (e2e) path on C2 frames."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2311_00626_b200 as vx  # noqa: E402

N = 24
sensor, frames, icfg, ecfg = bench.make_inputs("c2", N)
if os.environ.get("DIAG_TORCH_PIN") == "1":
    pinned = [torch.from_numpy(d).pin_memory() for _, d in frames]
else:
    pinned_bufs = [vx.pinned_like(np.ascontiguousarray(d, np.float32)) for _, d in frames]
    pinned = [torch.from_numpy(b.array) for b in pinned_bufs]
ctx = vx.default_context()
ext = torch.cuda.ExternalStream(ctx.stream)
T = vx.TsdfLayer(0.02)
E = vx.EsdfLayer(0.02)
rows = []
PROF = os.environ.get("DIAG_PROF") == "1"
KN = bench.TSDF_KERNELS + bench.ESDF_KERNELS
if PROF:
    ctx.set_profiling(True)
for i in range(N):
    if PROF:
        ctx.reset_kernel_times()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ev[0].record(ext)
    ch = vx.integrate_depth(T, pinned[i].numpy(), frames[i][0], sensor, icfg)
    ev[1].record(ext)
    t1 = time.perf_counter()
    ev[2].record(ext)
    ech = vx.update_esdf(E, T, ch, ecfg)
    ev[3].record(ext)
    t2 = time.perf_counter()
    torch.cuda.synchronize()
    rows.append((1e3 * (t1 - t0), ev[0].elapsed_time(ev[1]), 1e3 * (t2 - t1), ev[2].elapsed_time(ev[3])))
    print(f"frame {i}: integrate wall {rows[-1][0]:.3f} dev {rows[-1][1]:.3f} | update_esdf wall "
          f"{rows[-1][2]:.3f} dev {rows[-1][3]:.3f} ({len(ch)} / {len(ech)} blocks)", flush=True)
    if PROF:
        print("   kernels: " + " ".join(f"{k}={ctx.kernel_time(k)[0] * 1e3:.1f}" for k in KN), flush=True)
r = np.array(rows[4:])
print("mean (frames 4..): integrate wall %.3f dev %.3f | esdf wall %.3f dev %.3f" % tuple(r.mean(0)))
