"""Summarise ncu outputs for profiles/: launch-list CSV -> per-kernel stats,
and --set full reports -> duration / DRAM traffic / occupancy per kernel."""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, agg = None, defaultdict(list)
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            agg[d["Kernel Name"].split("(")[0]].append(float(d["Metric Value"].replace(",", "")) / 1e3)
    tot = sum(sum(v) for v in agg.values())
    print(f"| kernel | launches | avg us | min us | share of GPU time |\n|---|---|---|---|---|")
    for n, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"| `{n}` | {len(v)} | {sum(v)/len(v):.2f} | {min(v):.2f} | {100*sum(v)/tot:.1f}% |")


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr = r[0]
    want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size", "launch__block_size"]
    idx = [hdr.index(w) for w in want]
    print("| kernel | duration us | DRAM read MB | DRAM write MB | DRAM % peak | regs | warps active % | grid x block |")
    print("|---|---|---|---|---|---|---|---|")
    for row in r[2:]:
        v = [row[i] for i in idx]
        print(f"| `{v[0].split('(')[0]}` | {float(v[1]):.2f} | {float(v[2]):.2f} | {float(v[3]):.2f} | {float(v[4]):.1f} | "
              f"{v[5]} | {float(v[6]):.1f} | {v[7]} x {v[8]} |")


if __name__ == "__main__":
    kind, path = sys.argv[1], sys.argv[2]
    launches(path) if kind == "launches" else full(path)
