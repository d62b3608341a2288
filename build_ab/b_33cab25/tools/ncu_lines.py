"""Per-source-line instruction / stall breakdown of one kernel in an ncu report.

    python tools/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX [top]
"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
skip = sys.argv[4] if len(sys.argv) > 4 else "0"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + kre, "--launch-skip", skip,
                      "--launch-count", "1", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
data, fname, hdr = [], "?", None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < len(hdr) or r[2] != "-":
        continue
    try:
        ie = int(r[7] or 0)
        st = int(r[4] or 0)
    except ValueError:
        continue
    data.append((ie, st, f"{fname}:{r[0]}", r[1][:80]))
tot = sum(d[0] for d in data) or 1
tots = sum(d[1] for d in data) or 1
print(f"total warp-instructions {tot}  stall samples {tots}")
for d in sorted(data, key=lambda x: -(x[0] / tot + x[1] / tots))[:top]:
    print(f"{100*d[0]/tot:5.1f}% inst {100*d[1]/tots:5.1f}% stall  {d[2]:24s} {d[3]}")
