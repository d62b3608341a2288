"""Key metrics of every kernel in an ncu report (one line per launch).

    python tools/ncu_summary2.py REPORT.ncu-rep
"""
import csv
import io
import subprocess
import sys

want = {"Duration": "dur", "DRAM Throughput": "dram%", "Executed Ipc Active": "ipc", "L2 Hit Rate": "l2hit",
        "Achieved Occupancy": "occ", "Registers Per Thread": "regs", "Executed Instructions": "inst",
        "Warp Cycles Per Issued Instruction": "cpi", "Avg. Active Threads Per Warp": "thr/w", "Grid Size": "grid",
        "dram__bytes_read.sum": "rd", "dram__bytes_write.sum": "wr"}
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
ki, ii, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "ID", "Metric Name", "Metric Value", "Metric Unit"))
per = {}
for r in rows[1:]:
    if r[mi] in want:
        d = per.setdefault(r[ii], {"name": r[ki]})
        d[want[r[mi]]] = r[vi] + ("" if r[ui] in ("", "inst", "register/thread") else r[ui][:4])
for i, d in per.items():
    name = d.pop("name").replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
    print(i, name[:70])
    print("    " + "  ".join(f"{k}={v}" for k, v in d.items()))
