#!/usr/bin/env python
"""Per-frame map update benchmark (BASELINE.json metric).

A step is one frame of the workload: integrate_depth (block allocation + TSDF
integration) followed by update_esdf, for BASELINE config C2 by default
(synthetic room trajectory, 640x480 depth, 2 cm voxels, ESDF every frame).

  value  device-resident frames/s: depth frames already in HBM, the changed
         block list stays on the device between integrate and ESDF.
  e2e    the same frames through the public host API (vxm_integrate_depth_camera
         + vxm_update_esdf: host depth from page-locked memory (vxm_host_alloc)
         copied in, changed lists copied out each step) — the reference-facing
         path.  N>1 runs N replicas (one independent map per GPU, weak scaling).

Timing: W untimed warm-up frames, then K timed frames; before every timed
frame a 256 MB buffer is written to flush L2; CUDA events on the library's
stream bracket each frame; N>1 takes the max over ranks.  `--impl reference`
times the reference's own CPU implementation (oracle/_ref, OpenMP on all host
cores) on the same workload instead.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "TSDF voxel updates/s & frames/s (640x480, 2cm) at 1/2/4/8 GPU; ESDF ms/frame"
UNIT = "frames/s"

CONFIGS = {
    # name: scene, sensor, size, voxel, truncation, max_int, esdf(site, max_dist), orbit
    "c2": dict(scene="room", sensor="camera", w=640, h=480, vs=0.02, trunc=0.08, max_int=5.0,
               esdf=(0.02, 2.0), orbit=100,
               workload="C2: synthetic room trajectory, 640x480 depth, 2 cm voxels, "
                        "TSDF integration + ESDF update every frame"),
    "c1": dict(scene="sphere_in_box", sensor="camera", w=640, h=480, vs=0.05, trunc=0.2,
               max_int=5.0, esdf=None, orbit=100,
               workload="C1: sphere_in_box, 640x480 depth, 5 cm voxels, TSDF integration only"),
    "c5": dict(scene="sphere_world", sensor="none", w=512, h=512, vs=0.02, trunc=0.08, max_int=0.0,
               esdf=(0.02, 2.0), orbit=0,
               workload="C5: ESDF full recompute of a dense 512^3-voxel SphereWorld volume "
                        "(262,144 blocks); each step alternates between two volumes so every "
                        "update resets and re-lowers the whole map"),
    "c4": dict(scene="building", sensor="camera", w=640, h=480, vs=0.01, trunc=0.04, max_int=5.0,
               esdf=(0.01, 2.0), orbit=100, reserve=1 << 19,
               workload="C4 (single GPU): synthetic building walkthrough, 640x480 depth, 1 cm "
                        "voxels, TSDF integration + ESDF update every frame"),
    "c3": dict(scene="lidar_yard", sensor="lidar", w=2048, h=64, vs=0.1, trunc=0.4, max_int=100.0,
               esdf=(0.1, 2.0), orbit=100, reserve=1 << 20,
               workload="C3: 64-beam x 2048-column LiDAR, 10 cm voxels, 100 m range, TSDF + ESDF"),
}


TSDF_KERNELS = ("k_rays", "k_dilate_alloc", "k_integrate", "k_compact")
ESDF_KERNELS = ("k_merge7", "k_effective_alloc", "k_mark", "k_lower", "k_compact_esdf")


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---------------------------------------------------------------------------
def make_inputs(cfgname, n_frames, offset=0, ref=None):
    """Scene, orbit poses and rendered frames of a config.  Our arm renders
    with the product-side generator (libvoxmap_synth.so); the reference arm
    passes `ref` (oracle/_ref) and renders with the reference's own
    render_depth / orbit_pose, so it loads no library of ours (tests pin both
    generators byte-identical: tests/test_abi.py)."""
    from paper_2311_00626_b200 import _abi as A
    c = CONFIGS[cfgname]
    lidar = c["sensor"] == "lidar"
    if ref is None:
        from paper_2311_00626_b200 import synth
        S = synth.Scene(c["scene"])
        pose = lambda k: S.orbit_pose(k, c["orbit"], lidar=lidar)  # noqa: E731
        render = S.render_lidar if lidar else S.render_camera
    else:
        pose = lambda k: ref.orbit_pose(c["scene"], k, c["orbit"], lidar=lidar)  # noqa: E731
        render = ((lambda T, s: ref.render_lidar(c["scene"], T, s)) if lidar
                  else (lambda T, s: ref.render_camera(c["scene"], T, s)))
    if c["sensor"] == "camera":
        sensor = A.default_camera(c["w"], c["h"])
    else:
        sensor = A.default_lidar(c["w"], c["h"])
        sensor.max_range = c["max_int"]
    frames = []
    for k in range(offset, offset + n_frames):
        T = pose(k % c["orbit"])
        frames.append((T, render(T, sensor)))
    icfg = A.default_integrator_config(truncation=c["trunc"], max_integration_distance=c["max_int"])
    ecfg = A.default_esdf_config(site_threshold=c["esdf"][0], max_distance=c["esdf"][1]) if c["esdf"] else None
    return sensor, frames, icfg, ecfg


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""
    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(kernel, config="c2"):
    """Per-launch DRAM bytes of `kernel` from the committed ncu capture summary
    of this config (null when no capture of this config is committed)."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f).get(config, {}).get(kernel)
    except Exception:
        return None


# ---------------------------------------------------------------------------
def run_ours(args, rank, world, device):
    import numpy as np
    import torch

    import paper_2311_00626_b200 as vx
    torch.cuda.set_device(device)
    c = CONFIGS[args.config]
    W, K = args.warmup, args.steps
    sensor, frames, icfg, ecfg = make_inputs(args.config, W + K, offset=rank * 7)
    ctx = vx.Context(device)
    ext = torch.cuda.ExternalStream(ctx.stream, device=device)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=device)
    dev_frames = torch.from_numpy(np.stack([d for _, d in frames])).to(device)
    H, Wd = dev_frames.shape[1], dev_frames.shape[2]

    # ---- value: device-resident path --------------------------------------
    T = vx.TsdfLayer(c["vs"], ctx=ctx)
    E = vx.EsdfLayer(c["vs"], ctx=ctx) if ecfg else None
    if c.get("reserve"):  # pre-size the pools (the map grows every frame)
        T.reserve(c["reserve"])
        if E is not None:
            E.reserve(c["reserve"])
    changed = vx.BlockList(ctx)
    esdf_out = vx.BlockList(ctx)

    def step(Tl, El, i):
        # one replay-pipeline frame on device-resident input (one host round trip)
        vx.update_frame_device(Tl, El, dev_frames[i].data_ptr(), Wd, H, frames[i][0], sensor, icfg,
                               ecfg, changed, esdf_out if El is not None else None)

    for i in range(W):
        step(T, E, i)
    torch.cuda.synchronize(device)
    ctx.reset_stats()
    launches0 = ctx.launch_count
    tot = []
    with ClockSampler(device) as clk:
        for i in range(W, W + K):
            flush.zero_()
            torch.cuda.synchronize(device)
            e0, e1 = (torch.cuda.Event(enable_timing=True) for _ in range(2))
            e0.record(ext)
            step(T, E, i)
            e1.record(ext)
            e1.synchronize()
            tot.append(e0.elapsed_time(e1))
    launches = ctx.launch_count - launches0
    stats = ctx.stats()
    total_s = sum(tot) / 1000.0

    # ---- per-kernel breakdown: the same frames replayed on fresh layers with
    # CUDA events around every kernel (outside the timed region above) -------
    del T, E
    Tp = vx.TsdfLayer(c["vs"], ctx=ctx)
    Ep = vx.EsdfLayer(c["vs"], ctx=ctx) if ecfg else None
    if c.get("reserve"):
        Tp.reserve(c["reserve"])
        if Ep is not None:
            Ep.reserve(c["reserve"])
    for i in range(W):
        step(Tp, Ep, i)
    ctx.set_profiling(True)
    ctx.reset_kernel_times()
    for i in range(W, W + K):
        flush.zero_()
        torch.cuda.synchronize(device)
        step(Tp, Ep, i)
    torch.cuda.synchronize(device)
    kernels = {}
    for name in TSDF_KERNELS + ESDF_KERNELS:
        ms, n = ctx.kernel_time(name)
        if n:
            kernels[name] = {"ms_total": ms, "launches": n, "ms_per_launch": ms / n}
    ctx.set_profiling(False)
    tsdf_ms = sum(kernels[k]["ms_total"] for k in TSDF_KERNELS if k in kernels) / K
    esdf_ms = sum(kernels[k]["ms_total"] for k in ESDF_KERNELS if k in kernels) / K

    # ---- e2e: public host API, host buffers, copies inside the timed region --
    # frames staged in page-locked buffers (vxm_host_alloc, full-rate DMA)
    pinned_bufs = [vx.pinned_like(np.ascontiguousarray(d, np.float32)) for _, d in frames]
    pinned = [torch.from_numpy(b.array) for b in pinned_bufs]
    del Tp, Ep
    T2 = vx.TsdfLayer(c["vs"], ctx=ctx)
    E2 = vx.EsdfLayer(c["vs"], ctx=ctx) if ecfg else None
    if c.get("reserve"):
        T2.reserve(c["reserve"])
        if E2 is not None:
            E2.reserve(c["reserve"])
    for i in range(W):
        ch = vx.integrate_depth(T2, pinned[i].numpy(), frames[i][0], sensor, icfg)
        if E2 is not None:
            vx.update_esdf(E2, T2, ch, ecfg)
    e2e_t, h2d, d2h = [], 0, 0
    for i in range(W, W + K):
        flush.zero_()
        torch.cuda.synchronize(device)
        t0 = time.perf_counter()
        ch = vx.integrate_depth(T2, pinned[i].numpy(), frames[i][0], sensor, icfg)
        h2d += pinned[i].numel() * 4
        d2h += ch.nbytes
        if E2 is not None:
            # the list is byte-identical to the integrate's result, whose device
            # copy update_esdf reuses: no upload (vxm_update_esdf, capi.cu)
            ech = vx.update_esdf(E2, T2, ch, ecfg)
            d2h += ech.nbytes
        e2e_t.append(time.perf_counter() - t0)
    e2e_s = sum(e2e_t)

    # ---- multi-rank: max over ranks ----------------------------------------
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([total_s, e2e_s], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_s, e2e_s = float(t[0]), float(t[1])
    return dict(total_s=total_s, tot=tot, tsdf_ms=tsdf_ms, esdf_ms=esdf_ms, stats=stats,
                kernels=kernels, launches=launches, clocks=clk.summary(), e2e_s=e2e_s,
                h2d=h2d // K, d2h=d2h // K, W=Wd, H=H)


def roofline(res, K, config="c2"):
    peak, peak_src = measured_peaks()
    st, ks = res["stats"], res["kernels"]
    # algorithmic bytes per launch
    bytes_by_kernel = {
        "k_integrate": 8 * st["voxels_read"] + 8 * st["voxels_updated"] + 4 * st["depth_pixels"],
        "k_lower": 12288 * (st["esdf_blocks"] - st.get("quiet_blocks", 0)) + 12288 * st["dirty_blocks_after_round1"]
                   + 3072 * st["pair_exchanges"] + 12288 * st["compared_blocks"],
    }
    cand = [k for k in bytes_by_kernel if k in ks]
    if not cand:
        return None
    dom = max(cand, key=lambda k: ks[k]["ms_total"])
    n = ks[dom]["launches"]
    per_launch = bytes_by_kernel[dom] / n
    achieved = per_launch / (ks[dom]["ms_per_launch"] / 1e3) / 1e9
    out = {"kernel": dom, "bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
           "unit": "GB/s", "frac": round(achieved / peak, 4), "peak_source": peak_src,
           "algorithmic_bytes_per_launch": int(per_launch),
           "share_of_step": round(ks[dom]["ms_total"] / (res["total_s"] * 1e3), 3),
           "traffic": ncu_traffic(dom, config)}
    others = {}
    for k in cand:
        if k != dom:
            b = bytes_by_kernel[k] / ks[k]["launches"]
            a = b / (ks[k]["ms_per_launch"] / 1e3) / 1e9
            others[k] = {"achieved": round(a, 1), "frac": round(a / peak, 4),
                         "algorithmic_bytes_per_launch": int(b), "traffic": ncu_traffic(k, config)}
    out["other_kernels"] = others
    return out


# ---------------------------------------------------------------------------
def cpu_reference_run(cfgname, warmup, steps, budget_s=None):
    """The reference's own CPU path (oracle/_ref, OpenMP) or the C restatement."""
    cores = os.cpu_count() or 1
    os.environ.setdefault("OMP_NUM_THREADS", str(cores))
    from oracle.bindings import PortOracle, RefOracle, have_ref
    from paper_2311_00626_b200 import _abi as A
    c = CONFIGS[cfgname]
    kind = "reference" if have_ref() else "port"
    o = RefOracle() if kind == "reference" else PortOracle()
    sensor, frames, icfg, ecfg = make_inputs(cfgname, warmup + steps,
                                             ref=o if kind == "reference" else None)
    T = o.layer(A.LAYER_TSDF, c["vs"])
    E = o.layer(A.LAYER_ESDF, c["vs"]) if ecfg else None
    integ = o.integrate_camera if c["sensor"] == "camera" else o.integrate_lidar

    def step(i):
        ch = integ(T, frames[i][1], frames[i][0], sensor, icfg)
        if E is not None:
            o.update_esdf(E, T, ch, ecfg)
        return len(ch)

    for i in range(warmup):
        step(i)
    times, t_start = [], time.perf_counter()
    for i in range(warmup, warmup + steps):
        t0 = time.perf_counter()
        step(i)
        times.append(time.perf_counter() - t0)
        if budget_s and time.perf_counter() - t_start > budget_s:
            break
    n = len(times)
    return dict(value=n / sum(times), kind=kind, cores=cores if kind == "reference" else 1,
                frames=n, ms_per_step=1e3 * sum(times) / n,
                sample=f"{c['workload']}; frames {warmup}..{warmup + n - 1} of the orbit after "
                       f"{warmup} untimed warm-up frames; "
                       + ("production integrate_depth + update_esdf (OpenMP)" if kind == "reference"
                          else "oracle/voxmap_oracle.c restatement (serial)"))


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


# ---------------------------------------------------------------------------
C5_SIDE = 512


def c5_volumes(side=C5_SIDE, ref=None):
    if ref is None:
        from paper_2311_00626_b200 import synth
        gen = synth.sphere_world
    else:
        gen = ref.sphere_world
    ka, va = gen(side, 0.02, 0.08, seed=2311)
    kb, vb = gen(side, 0.02, 0.08, seed=2312)
    assert np.array_equal(ka, kb)
    return ka, va, vb


def run_c5(args, rank, world, device):
    import torch

    import paper_2311_00626_b200 as vx
    from paper_2311_00626_b200 import _abi as A
    torch.cuda.set_device(device)
    W, K = args.warmup, args.steps
    keys, va, vb = c5_volumes()
    ctx = vx.Context(device)
    ext = torch.cuda.ExternalStream(ctx.stream, device=device)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=device)
    Ts = [vx.TsdfLayer(0.02, ctx=ctx), vx.TsdfLayer(0.02, ctx=ctx)]
    Ts[0].write_blocks(keys, va)
    Ts[1].write_blocks(keys, vb)
    del va, vb
    ecfg = A.default_esdf_config(site_threshold=0.02, max_distance=2.0)
    upd = vx.BlockList(ctx)
    upd.assign(keys)
    out = vx.BlockList(ctx)
    E = vx.EsdfLayer(0.02, ctx=ctx)
    for i in range(W):
        vx.update_esdf_device(E, Ts[i % 2], upd, ecfg, out)
    torch.cuda.synchronize(device)
    ctx.reset_stats()
    launches0 = ctx.launch_count
    tot = []
    with ClockSampler(device) as clk:
        for i in range(W, W + K):
            flush.zero_()
            torch.cuda.synchronize(device)
            e0, e1 = (torch.cuda.Event(enable_timing=True) for _ in range(2))
            e0.record(ext)
            vx.update_esdf_device(E, Ts[i % 2], upd, ecfg, out)
            e1.record(ext)
            e1.synchronize()
            tot.append(e0.elapsed_time(e1))
    launches = ctx.launch_count - launches0
    stats = ctx.stats()
    total_s = sum(tot) / 1000.0
    # per-kernel breakdown on extra steps (events around each kernel)
    ctx.set_profiling(True)
    ctx.reset_kernel_times()
    for i in range(W + K, W + 2 * K):
        flush.zero_()
        torch.cuda.synchronize(device)
        vx.update_esdf_device(E, Ts[i % 2], upd, ecfg, out)
    torch.cuda.synchronize(device)
    kernels = {}
    for name in ESDF_KERNELS:
        ms, n = ctx.kernel_time(name)
        if n:
            kernels[name] = {"ms_total": ms, "launches": n, "ms_per_launch": ms / n}
    ctx.set_profiling(False)
    # e2e: the public host API (host key list in, host changed list out); the
    # key list is staged in page-locked memory (vxm_host_alloc, as C2's frames),
    # one untimed call warms the host path's staging buffers
    hkeys = vx.pinned_like(np.ascontiguousarray(keys, np.int32))
    vx.update_esdf(E, Ts[(W + 2 * K + 1) % 2], hkeys.array, ecfg)
    e2e_t, h2d, d2h = [], 0, 0
    for i in range(W + 2 * K, W + 3 * K):
        flush.zero_()
        torch.cuda.synchronize(device)
        t0 = time.perf_counter()
        ch = vx.update_esdf(E, Ts[i % 2], hkeys.array, ecfg)
        e2e_t.append(time.perf_counter() - t0)
        h2d += keys.nbytes
        d2h += ch.nbytes
    return dict(total_s=total_s, tot=tot, tsdf_ms=0.0, esdf_ms=total_s * 1e3 / K, stats=stats,
                kernels=kernels, launches=launches, clocks=clk.summary(), e2e_s=sum(e2e_t),
                h2d=h2d // K, d2h=d2h // K, n_blocks=len(keys))


def cpu_reference_c5(steps, side=C5_SIDE):
    """The reference's update_esdf (oracle/_ref, OpenMP) on the same volumes."""
    cores = os.cpu_count() or 1
    os.environ.setdefault("OMP_NUM_THREADS", str(cores))
    from oracle.bindings import PortOracle, RefOracle, have_ref
    from paper_2311_00626_b200 import _abi as A
    kind = "reference" if have_ref() else "port"
    o = RefOracle() if kind == "reference" else PortOracle()
    keys, va, vb = c5_volumes(side, ref=o if kind == "reference" else None)
    Ts = [o.layer(A.LAYER_TSDF, 0.02), o.layer(A.LAYER_TSDF, 0.02)]
    o.write_blocks(Ts[0], keys, va)
    o.write_blocks(Ts[1], keys, vb)
    del va, vb
    ecfg = A.default_esdf_config(site_threshold=0.02, max_distance=2.0)
    E = o.layer(A.LAYER_ESDF, 0.02)
    o.update_esdf(E, Ts[0], keys, ecfg)  # warm-up (allocation)
    times = []
    for i in range(1, 1 + steps):
        t0 = time.perf_counter()
        o.update_esdf(E, Ts[i % 2], keys, ecfg)
        times.append(time.perf_counter() - t0)
    n = len(times)
    return dict(value=n / sum(times), kind=kind, cores=cores if kind == "reference" else 1, frames=n,
                ms_per_step=1e3 * sum(times) / n,
                sample=f"C5 {side}^3 SphereWorld, {n} full update_esdf call(s) alternating two volumes "
                       f"after one untimed allocation call; "
                       + ("production update_esdf (OpenMP)" if kind == "reference"
                          else "oracle/voxmap_oracle.c restatement (serial)"))


# ---------------------------------------------------------------------------
def shard_owner(x, world, slab):
    """owner(g) = floor(g.x / slab) mod world (vxm_context_set_shard)."""
    return (np.asarray(x, np.int64) // slab) % world


def run_sharded(args, rank, world, device):
    """--shard: ONE map block-sharded over the ranks; a step is
    one frame of the whole map: rank 0's depth frame is broadcast over NCCL,
    every rank allocates and integrates only its x-slabs (no exchange), then
    update_esdf runs over the union map with per-round slab-boundary face
    exchange (paper_2311_00626_b200/dist.py: NCCL send/recv + an on-device
    all-reduce of the next dirty count on the library's stream).  C5: each rank
    holds its slabs of the volume and updates them."""
    import torch
    import torch.distributed as dist

    import paper_2311_00626_b200 as vx
    from paper_2311_00626_b200 import _abi as A
    from paper_2311_00626_b200 import dist as vxd
    torch.cuda.set_device(device)
    c = CONFIGS[args.config]
    W, K = args.warmup, args.steps
    ctx = vx.Context(device)
    ctx.set_shard(rank, world, args.slab)
    ext = torch.cuda.ExternalStream(ctx.stream, device=device)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=device)
    cuda = torch.device("cuda", device)
    xfer = {"h2d": 0, "d2h": 0}
    if args.config == "c5":
        keys, va, vb = c5_volumes()
        own = shard_owner(keys[:, 0], world, args.slab) == rank
        Ts = [vx.TsdfLayer(c["vs"], ctx=ctx), vx.TsdfLayer(c["vs"], ctx=ctx)]
        Ts[0].write_blocks(keys[own], va[own])
        Ts[1].write_blocks(keys[own], vb[own])
        del va, vb
        upd = np.ascontiguousarray(keys[own])
        ecfg = A.default_esdf_config(site_threshold=c["esdf"][0], max_distance=c["esdf"][1])
        E = vx.EsdfLayer(c["vs"], ctx=ctx)

        def step(i, host=False):
            ch = vxd.update_esdf_distributed(E, Ts[i % 2], upd, ecfg)
            if host:
                xfer["h2d"] += upd.nbytes
                xfer["d2h"] += ch.nbytes
    else:
        sensor, frames, icfg, ecfg = make_inputs(args.config, W + K)
        H, Wd = frames[0][1].shape
        if rank == 0:
            dev_frames = torch.from_numpy(np.stack([d for _, d in frames])).to(cuda)
            pinned = [vx.pinned_like(np.ascontiguousarray(d, np.float32)) for _, d in frames]
        buf = torch.empty((H, Wd), dtype=torch.float32, device=cuda)
        T = vx.TsdfLayer(c["vs"], ctx=ctx)
        E = vx.EsdfLayer(c["vs"], ctx=ctx)
        if c.get("reserve"):
            T.reserve(max(1, c["reserve"] // world))
            E.reserve(max(1, c["reserve"] // world))
        tl = vx.BlockList(ctx)

        def step(i, host=False):
            with torch.cuda.stream(ext):  # the broadcast is ordered before our kernels
                if rank == 0:
                    if host:  # the frame arrives in host memory on the sensor's rank
                        buf.copy_(torch.from_numpy(pinned[i].array), non_blocking=True)
                        xfer["h2d"] += buf.numel() * 4
                    else:
                        buf.copy_(dev_frames[i])
                if dist.get_backend() == "gloo":
                    hb = buf.cpu()
                    dist.broadcast(hb, src=0)
                    buf.copy_(hb)
                else:
                    dist.broadcast(buf, src=0)
            vx.integrate_depth_device(T, buf.data_ptr(), Wd, H, frames[i][0], sensor, icfg, tl)
            ch = vxd.update_esdf_distributed(E, T, tl, ecfg)
            if host:
                xfer["d2h"] += ch.nbytes

    for i in range(W):
        step(i)
    torch.cuda.synchronize(device)
    ctx.reset_stats()
    launches0 = ctx.launch_count
    tot = []
    with ClockSampler(device) as clk:
        for i in range(W, W + K):
            flush.zero_()
            torch.cuda.synchronize(device)
            dist.barrier()
            e0, e1 = (torch.cuda.Event(enable_timing=True) for _ in range(2))
            e0.record(ext)
            step(i)
            e1.record(ext)
            e1.synchronize()
            tot.append(e0.elapsed_time(e1))
    launches = ctx.launch_count - launches0
    stats = ctx.stats()
    total_s = sum(tot) / 1000.0
    # e2e: host frame on the sensor rank, changed lists back to each host
    e2e_t = []
    for i in range(W, W + K):
        torch.cuda.synchronize(device)
        dist.barrier()
        t0 = time.perf_counter()
        step(i, host=True)
        torch.cuda.synchronize(device)
        e2e_t.append(time.perf_counter() - t0)
    t = torch.tensor([total_s, sum(e2e_t)], dtype=torch.float64, device=cuda)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    blocks = torch.tensor([stats["esdf_blocks"]], dtype=torch.float64, device=cuda)
    dist.all_reduce(blocks, op=dist.ReduceOp.SUM)
    return dict(total_s=float(t[0]), tot=tot, tsdf_ms=0.0, esdf_ms=0.0, stats=stats, kernels={},
                launches=launches, clocks=clk.summary(), e2e_s=float(t[1]),
                h2d=xfer["h2d"] // K, d2h=xfer["d2h"] // K, union_esdf_blocks=float(blocks[0]) / K)


# ---------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--cpu-budget", type=float, default=20.0, help="seconds of CPU baseline work")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--shard", action="store_true",
                    help="one map block-sharded over the ranks (x-slabs, NCCL exchange) instead of "
                         "N independent replicas")
    ap.add_argument("--slab", type=int, default=0, help="shard slab width in blocks (default by config)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    c = CONFIGS[args.config]
    config = {"workload": c["workload"], "scene": c["scene"], "sensor": c["sensor"],
              "image": f"{c['w']}x{c['h']}", "voxel_size_m": c["vs"], "truncation_m": c["trunc"],
              "esdf": {"site_threshold_m": c["esdf"][0], "max_distance_m": c["esdf"][1]} if c["esdf"] else None,
              "l2": "flushed (256 MB write) before every timed step",
              "parallelism": f"replicas{args.gpus}" if args.gpus > 1 else "single"}

    if args.config == "c5":
        config = {"workload": c["workload"], "volume_voxels": f"{C5_SIDE}^3", "voxel_size_m": c["vs"],
                  "truncation_m": c["trunc"],
                  "esdf": {"site_threshold_m": c["esdf"][0], "max_distance_m": c["esdf"][1]},
                  "l2": "flushed (256 MB write) before every timed step; map 1.6 GB ESDF + 2 GB TSDF",
                  "parallelism": f"replicas{args.gpus}" if args.gpus > 1 else "single"}
    if args.impl == "reference":
        if rank != 0:
            return
        r = (cpu_reference_c5(max(1, min(args.steps, 3))) if args.config == "c5"
             else cpu_reference_run(args.config, args.warmup, args.steps))
        line = {"impl": "reference", "metric": METRIC, "value": round(r["value"], 3), "unit": UNIT,
                "n_gpus": args.gpus, "steps": r["frames"], "warmup": args.warmup,
                "ms_per_step": round(r["ms_per_step"], 3), "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64/f32/i32",
                "data": "synthetic (reference scene + orbit, sphere-traced depth)", "config": config,
                "cpu_baseline": {"value": round(r["value"], 3), "unit": UNIT, "cores": r["cores"],
                                 "kind": r["kind"], "sample": r["sample"], "cpu": cpu_model()},
                "e2e": {"value": round(r["value"], 3), "unit": UNIT, "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    sharded = args.shard and world > 1
    if args.shard:
        if args.config == "c1" or c["sensor"] == "lidar":
            raise SystemExit("--shard: configs c2, c4, c5 (camera / volume maps)")
        args.slab = args.slab or (8 if args.config == "c5" else 16)
        # N = 1: the whole map on one GPU is the single-map path itself
        config["parallelism"] = f"shard{world}" if world > 1 else "shard1 (single map)"
        config["shard"] = {"owner": "floor(block.x / slab) mod n_gpus", "slab_blocks": args.slab,
                           "exchange": "slab-boundary x-faces per lowering round, NCCL send/recv "
                                       "on the library stream; depth broadcast from rank 0"}
    if world > 1:
        import torch
        import torch.distributed as dist
        local = local % max(1, torch.cuda.device_count())  # gloo functional runs share one GPU
        torch.cuda.set_device(local)
        # VXM_DIST_BACKEND=gloo: functional runs of several ranks on ONE GPU
        # (NCCL refuses two ranks on one device); never a bench number
        backend = os.environ.get("VXM_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
            config["backend"] = backend
    if sharded:
        res = run_sharded(args, rank, world, local)
    else:
        res = (run_c5 if args.config == "c5" else run_ours)(args, rank, world, local)
    K = args.steps
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    if rank != 0:
        return
    st = res["stats"]
    # replicas: N maps, N x the frames; sharded: one map, the frames once
    value = (1 if sharded else world) * K / res["total_s"]
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world, "steps": K,
        "warmup": args.warmup, "ms_per_step": round(1e3 * res["total_s"] / K, 4),
        "higher_is_better": True, "scaling": "strong" if args.shard else "weak", "vs_baseline": None,
        "dtype": "f64/f32/i32",
        "data": "synthetic (reference scene + orbit trajectory, sphere-traced depth rendered on the host)",
        "config": config,
        "tsdf_voxel_updates_per_s": (round(world * st["voxels_updated"] / res["total_s"], 1)
                                     if args.config != "c5" else None),
        # kernel time per frame (CUDA events around each kernel, separate replay)
        "tsdf_ms_per_frame": round(res["tsdf_ms"], 4),
        "esdf_ms_per_frame": round(res["esdf_ms"], 4),
        "work_per_frame": {k: round(v / K, 1) for k, v in st.items()},
        "kernels_ms_per_frame": {k: round(v["ms_total"] / K, 4) for k, v in res["kernels"].items()},
        "roofline": roofline(res, K, args.config),
        "gpu_launches": res["launches"],
        "clocks": res["clocks"],
        "e2e": {"value": round((1 if sharded else world) * K / res["e2e_s"], 2), "unit": UNIT,
                "h2d_bytes_per_step": res["h2d"], "d2h_bytes_per_step": res["d2h"],
                "path": "vxm_integrate_depth_camera + vxm_update_esdf (host buffers)"},
        "value_path": "vxm_update_frame_camera_device (depth in HBM, one host round trip per frame)",
    }
    if args.config == "c5":
        line["e2e"]["path"] = "vxm_update_esdf (host key list in, host changed list out)"
        line["value_path"] = "vxm_update_esdf_list (updated list and map in HBM)"
        line["unit_note"] = "a step (frame) is one full update_esdf of the 512^3 map"
    if sharded:
        line["value_path"] = ("NCCL broadcast of rank 0's depth frame -> vxm_integrate_depth_*_device "
                              "(own slabs) -> update_esdf over the union map (dist.py: vxm_shard_update_* "
                              "steps, NCCL face exchange per round)") if args.config != "c5" else (
                              "update_esdf over the union map (dist.py: vxm_shard_update_* steps, NCCL "
                              "face exchange per round)")
        line["e2e"]["path"] = "the same with the frame from pinned host memory on rank 0 and the " \
                              "changed lists copied to each rank's host"
        line["union_esdf_blocks_per_step"] = res.get("union_esdf_blocks")
    if not args.no_cpu_baseline and world == 1:
        try:
            r = (cpu_reference_c5(1) if args.config == "c5" else
                 cpu_reference_run(args.config, args.warmup, args.steps, budget_s=args.cpu_budget))
            line["cpu_baseline"] = {"value": round(r["value"], 3), "unit": UNIT, "cores": r["cores"],
                                    "kind": r["kind"], "sample": r["sample"], "cpu": cpu_model()}
        except Exception as e:  # the CPU baseline is reported, not the measurement
            line["cpu_baseline"] = {"error": str(e)}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
