"""Summarise ncu artifacts into profiles/ (run here, no GPU needed).

    python tools/ncu_summary.py launches <launches.csv>       # per-kernel share of device time
    python tools/ncu_summary.py full <report.ncu-rep>         # key metrics per captured launch
"""
import collections
import csv
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ix = {k: i for i, k in enumerate(h)}
    tot = collections.Counter()
    cnt = collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) != len(h) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[ix["Kernel Name"]].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
        v = float(r[ix["Metric Value"]].replace(",", ""))
        unit = r[ix["Metric Unit"]]
        v = v / 1e6 if unit in ("nsecond", "ns") else (v / 1e3 if unit in ("usecond", "us") else v)
        tot[name] += v
        cnt[name] += 1
    s = sum(tot.values())
    print(f"| kernel | launches | total ms | share |\n|---|---|---|---|")
    for k, v in tot.most_common():
        print(f"| `{k}` | {cnt[k]} | {v:.2f} | {100 * v / s:.1f}% |")
    print(f"\ntotal device time {s:.1f} ms over {sum(cnt.values())} launches (cold-cache, serialised)")


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    ix = {k: i for i, k in enumerate(h)}
    want = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
            "Compute (SM) Throughput", "Executed Ipc Active", "Achieved Occupancy", "Theoretical Occupancy",
            "Registers Per Thread", "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp",
            "Executed Instructions"]
    per = collections.OrderedDict()
    for r in rows[1:]:
        key = (r[ix["ID"]], r[ix["Kernel Name"]].split("(")[0].replace("void ", "").replace("<unnamed>::", ""))
        if r[ix["Metric Name"]] in want:
            per.setdefault(key, {})[r[ix["Metric Name"]]] = r[ix["Metric Value"]] + " " + r[ix["Metric Unit"]]
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    rh = rr[0]
    for i, r in enumerate(rr[2:]):
        key = list(per.keys())[i] if i < len(per) else None
        if key is None:
            break
        for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            if m in rh:
                per[key][m] = r[rh.index(m)] + " " + rr[1][rh.index(m)]
    for (kid, name), d in per.items():
        print(f"### launch {kid}: `{name}`\n")
        for k, v in d.items():
            print(f"- {k}: {v}")
        print()


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2])
