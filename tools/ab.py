"""A/B timing of library variants: python tools/ab.py ROUNDS CONFIGS VARIANT...

Each VARIANT is a directory under tools/ab/ holding a libvoxmap_b200.so built
with `make -C paper_2311_00626_b200 OUT=$PWD/tools/ab/NAME OBJ=$PWD/tools/ab/NAME/obj`
("cur" = the in-tree build), optionally followed by environment settings:
NAME:VAR=VALUE,VAR2=VALUE2.  Runs bench.py for every (round, config, variant),
interleaved, and prints one line per run: variant, config, device frames/s,
e2e frames/s, dominant-kernel ms/frame.
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rounds = int(sys.argv[1])
configs = sys.argv[2].split(",")
variants = sys.argv[3:]
for r in range(rounds):
    for c in configs:
        for v in variants:
            env = dict(os.environ)
            name, _, extra = v.partition(":")
            if name != "cur":
                env["VXM_LIB_PATH"] = os.path.join(ROOT, "tools", "ab", name, "libvoxmap_b200.so")
            for kv in filter(None, extra.split(",")):
                k, _, val = kv.partition("=")
                env[k] = val
            steps = {"c5": "10", "c3": "10", "c4": "10"}.get(c, "20")
            p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--config", c, "--steps", steps,
                                "--warmup", "4", "--no-cpu-baseline"], env=env, capture_output=True, text=True)
            line = [l for l in p.stdout.splitlines() if l.startswith("{")]
            if p.returncode or not line:
                print(v, c, "FAILED", p.returncode, p.stderr[-400:], flush=True)
                continue
            d = json.loads(line[-1])
            k = d.get("kernels_ms_per_frame", {})
            ks = " ".join(f"{n}={t*1000:.1f}" for n, t in k.items())
            print(f"{v:24s} {c} {d['value']:9.2f} e2e {d['e2e']['value']:9.2f} | {ks}", flush=True)
