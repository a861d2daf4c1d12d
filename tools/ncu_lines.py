"""Summarise an ncu report's warp-stall samples per CUDA source line for one kernel.
usage: python tools/ncu_lines.py report.ncu-rep kernel_regex [top]"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout
agg, src, path, hdr = defaultdict(int), {}, None, None
for rec in csv.reader(io.StringIO(out)):
    if not rec:
        continue
    if rec[0] in ("File Path", "File Name"):
        path, hdr = rec[1].split("/")[-1], None
        continue
    if rec[0] == "Line No":
        hdr = rec
        continue
    if hdr and len(rec) == len(hdr):
        s = rec[hdr.index("Warp Stall Sampling (All Samples)")]
        if s.isdigit() and int(s):
            key = (path, rec[0])
            agg[key] += int(s)
            if rec[1].strip():
                src[key] = rec[1].strip()[:100]
tot = sum(agg.values())
print("total samples", tot)
for key, s in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{s:6d} {100 * s / max(tot, 1):5.1f}% {key[0]}:{key[1]}  {src.get(key, '')}")
