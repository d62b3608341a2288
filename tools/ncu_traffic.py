"""DRAM traffic per kernel class from an ncu metrics CSV
(ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv).

    python tools/ncu_traffic.py gpurun_out/traffic.csv --scale 24 --variant mg --mode det > profiles/ncu_traffic.json

Classes follow the engine's profiling classes (bench.py roofline): a class's
traffic per launch = its kernels' summed dram bytes / their launch count, the
same normalisation as the algorithmic bytes per launch.
"""
import argparse
import csv
import json
import re

CLASSES = {
    "eval_hi_rk": r"k_mg_hi_scan|k_mg_hi_merge|k_mg_hi_finish|k_mg_hi_direct",
    "eval_giant": r"k_giant_gather|k_mg_giant",
    "eval_lo": r"k_lane_direct",
}

ap = argparse.ArgumentParser()
ap.add_argument("csv")
ap.add_argument("--scale", type=int, default=24)
ap.add_argument("--variant", default="mg")
ap.add_argument("--mode", default="det")
a = ap.parse_args()
per = {}
with open(a.csv) as f:
    lines = [l for l in f if l.startswith('"')]
for r in csv.DictReader(lines):
    d = per.setdefault(r["ID"], {"name": r["Kernel Name"]})
    d[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
out = {"scale": a.scale, "variant": a.variant, "mode": a.mode, "source": a.csv, "classes": {}}
for cls, pat in CLASSES.items():
    ks = [d for d in per.values() if re.search(pat, d["name"])]
    if not ks:
        continue
    tot = sum(d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0) for d in ks)
    ns = sum(d.get("gpu__time_duration.sum", 0) for d in ks)
    out["classes"][cls] = {"launches": len(ks), "dram_bytes_per_launch": tot / len(ks), "dram_bytes_total": tot,
                           "ncu_ms_total": ns / 1e6}
print(json.dumps(out, indent=1))
