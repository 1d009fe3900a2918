"""Summarises gpurun_out/*.ncu-rep captures into profiles/ (CSV + traffic JSON).

usage: python tools/summarize_ncu.py <round-tag> cfg:kernel:report.ncu-rep ...
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__warps_active.avg.pct_of_peak_sustained_active",
           "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
           "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
           "smsp__inst_executed.sum"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [dict(zip(hdr, r)) for r in rows[2:]], dict(zip(hdr, units))


def num(s):
    try:
        return float(str(s).replace(",", ""))
    except ValueError:
        return None


def main():
    tag = sys.argv[1]
    summary, traffic = [], {}
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath))
    for spec in sys.argv[2:]:
        cfg, kern, rep = spec.split(":", 2)
        rows, units = raw(rep)
        for r in rows:
            if kern not in r.get("Kernel Name", ""):
                continue
            d = {"config": cfg, "kernel": kern}
            for m in METRICS:
                d[m] = num(r.get(m))
                d[m + ".unit"] = units.get(m)
            summary.append(d)
            rd, wr = d["dram__bytes_read.sum"], d["dram__bytes_write.sum"]
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            if rd is not None and wr is not None:
                br = rd * scale.get(units.get("dram__bytes_read.sum"), 1)
                bw = wr * scale.get(units.get("dram__bytes_write.sum"), 1)
                # keyed by the bench's per-kernel timing names
                traffic.setdefault(cfg, {})[{"k_lower3": "k_lower", "k_lower_xr": "k_lower"}.get(kern, kern)] = int(br + bw)
    out = os.path.join(ROOT, "profiles", f"{tag}_ncu_full_summary.csv")
    with open(out, "w", newline="") as f:
        w = csv.DictWriter(f, fieldnames=list(summary[0].keys()))
        w.writeheader()
        w.writerows(summary)
    traffic["_note"] = ("per-launch dram__bytes_read.sum + dram__bytes_write.sum from one ncu --set "
                        "full capture per config and kernel (cold L2, serialized replay); "
                        f"source profiles/{tag}_ncu_full_summary.csv")
    json.dump(traffic, open(tpath, "w"), indent=1)
    for d in summary:
        print(d["config"], d["kernel"], "dur", d["gpu__time_duration.sum"], d["gpu__time_duration.sum.unit"],
              "dram%", d["gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"],
              "traffic", traffic[d["config"]].get({"k_lower3": "k_lower", "k_lower_xr": "k_lower"}.get(d["kernel"], d["kernel"])))


if __name__ == "__main__":
    main()
