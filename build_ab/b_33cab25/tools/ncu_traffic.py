"""DRAM traffic and sector efficiency per kernel family over ONE lpa_run,
from an ncu metrics CSV of `tools/prof_run.py --range` (profiler range =
the last run):

    ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,\
l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum \
        --cache-control none --clock-control none --csv --log-file gpurun_out/traffic.csv \
        python tools/prof_run.py --scale 24 --runs 3 --range
    python tools/ncu_traffic.py gpurun_out/traffic.csv --scale 24 > profiles/ncu_traffic.json

Families are the bench.py roofline families (kernel-name patterns below);
bench.py divides dram_bytes_per_run by the family's kernel-launch count per
run from the engine's profiler -- the same count its algorithmic bytes per
launch use.  --cache-control none: L2 is not flushed between kernels, as in
a real run.
"""
import argparse
import csv
import json
import re

FAMILIES = {
    "eval_hi": r"k_mg_hi_|k_bm_hi_",
    "eval_lo": r"k_lane_direct|k_lane_win|k_lo_warp",
    "eval_giant": r"k_giant_gather|k_mg_giant|k_bm_giant",
    "commit": r"k_commit",
    "compact": r"k_scan_dirty|k_filter|k_defer|k_compact",
}

ap = argparse.ArgumentParser()
ap.add_argument("csv")
ap.add_argument("--scale", type=int, default=24)
ap.add_argument("--graph", default="rmat")
ap.add_argument("--variant", default="mg")
ap.add_argument("--mode", default="det")
a = ap.parse_args()
per = {}
with open(a.csv) as f:
    lines = [l for l in f if l.startswith('"')]
for r in csv.DictReader(lines):
    d = per.setdefault(r["ID"], {"name": r["Kernel Name"]})
    try:
        d[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    except ValueError:
        pass
out = {"scale": a.scale, "graph": a.graph, "variant": a.variant, "mode": a.mode, "basis": "one lpa_run",
       "source": a.csv, "kernels_captured": len(per), "families": {}}
for fam, pat in FAMILIES.items():
    ks = [d for d in per.values() if re.search(pat, d["name"])]
    if not ks:
        continue
    tot = sum(d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0) for d in ks)
    ns = sum(d.get("gpu__time_duration.sum", 0) for d in ks)
    sec = sum(d.get("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", 0) for d in ks)
    req = sum(d.get("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", 0) for d in ks)
    names = {}
    for d in ks:
        short = re.sub(r"^void (\(anonymous namespace\)|<unnamed>)::", "", d["name"]).split("(")[0]
        names[short] = names.get(short, 0) + 1
    out["families"][fam] = {"kernel_launches": len(ks), "dram_bytes_per_run": tot, "ncu_ms_per_run": ns / 1e6,
                            "dram_gbs": tot / (ns * 1e-9) / 1e9 if ns else None,
                            "ld_sectors_per_request": sec / req if req else None, "kernels": names}
print(json.dumps(out, indent=1))
