"""Summarise an SLPA_TRACE=2 profile log (second run only): per class and top launches."""
import re
import sys

lines = open(sys.argv[1]).read().split("\n")
runs = [i for i, l in enumerate(lines) if l.startswith("run ")]
sel = lines[runs[-2] + 1:runs[-1]] if len(runs) > 1 else lines
names = {0: "lo_r0", 1: "mid_r0", 2: "hi_r0", 3: "lo_rk", 4: "mid_rk", 5: "hi_rk", 6: "compact", 7: "commit",
         8: "other", 9: "giant"}
tot, big = {}, []
for l in sel:
    m = re.search(r"launch class (\d+): ([\d.]+) ms, (\d+) evals, (\d+) arcs", l)
    if m:
        c, ms, ev, ar = int(m[1]), float(m[2]), int(m[3]), int(m[4])
        t = tot.setdefault(names.get(c, c), [0, 0.0, 0, 0])
        t[0] += 1; t[1] += ms; t[2] += ev; t[3] += ar
        big.append((ms, names.get(c, c), ev, ar))
for k, v in tot.items():
    print(f"{k:8s} launches {v[0]:4d}  ms {v[1]:8.2f}  evals {v[2]:10d}  arcs {v[3]:11d}")
print("sum ms", round(sum(v[1] for v in tot.values()), 2))
for b in sorted(big, reverse=True)[:int(sys.argv[2]) if len(sys.argv) > 2 else 15]:
    print(b)
