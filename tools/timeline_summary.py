"""Summarise an SLPA_TRACE=3 timeline (tools/prof_run.py under SLPA_TRACE=3,
stdout + stderr in one file): per sweep of the LAST run, the span, the main
stream's busy time, the giant stream's busy time, the time only the giants
run, and the idle time (host round trips between rounds).

    SLPA_TRACE=3 python -u tools/prof_run.py --scale 24 --runs 2 > tl.log 2>&1
    python tools/timeline_summary.py tl.log
"""
import re
import sys


def union(iv):
    iv = sorted(iv)
    out = []
    for a, b in iv:
        if out and a <= out[-1][1]:
            out[-1][1] = max(out[-1][1], b)
        else:
            out.append([a, b])
    return out


def length(iv):
    return sum(b - a for a, b in iv)


def intersect(x, y):
    i = j = 0
    out = []
    while i < len(x) and j < len(y):
        a, b = max(x[i][0], y[j][0]), min(x[i][1], y[j][1])
        if a < b:
            out.append([a, b])
        if x[i][1] < y[j][1]:
            i += 1
        else:
            j += 1
    return out


lines = open(sys.argv[1]).read().split("\n")
runs = [i for i, l in enumerate(lines) if l.startswith("run ")]
start = runs[-2] + 1 if len(runs) > 1 else 0
end = runs[-1] if runs else len(lines)
sweeps, cur = [], None
for l in lines[start:end]:
    m = re.match(r"\[slpa\] tl (\S+)\s+([MG])\s+([\d.]+)\s+([\d.]+)", l)
    if not m:
        if cur:
            sweeps.append(cur)
            cur = None
        continue
    cur = cur or []
    cur.append((m[1], m[2], float(m[3]), float(m[4])))
if cur:
    sweeps.append(cur)
tot = dict(span=0.0, main=0.0, giant=0.0, giant_only=0.0, idle=0.0)
print("sweep   span_us   main_us  giant_us  giant_only_us  idle_us  launches")
for k, sw in enumerate(sweeps):
    M = union([[a, b] for _, s, a, b in sw if s == "M"])
    G = union([[a, b] for _, s, a, b in sw if s == "G"])
    span = max(b for _, _, _, b in sw) - min(a for _, _, a, _ in sw)
    both = length(intersect(M, G))
    busy = length(M) + length(G) - both
    row = dict(span=span, main=length(M), giant=length(G), giant_only=length(G) - both, idle=span - busy)
    for key in tot:
        tot[key] += row[key]
    print(f"{k:5d} {span:9.0f} {row['main']:9.0f} {row['giant']:9.0f} {row['giant_only']:14.0f} {row['idle']:8.0f}  {len(sw)}")
print(f"total {tot['span']:9.0f} {tot['main']:9.0f} {tot['giant']:9.0f} {tot['giant_only']:14.0f} {tot['idle']:8.0f}")
