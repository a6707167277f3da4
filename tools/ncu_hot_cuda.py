"""Warp-stall samples per CUDA source line (cuda,sass correlation) of one kernel in an ncu report.
usage: python tools/ncu_hot_cuda.py <report> [N [ncu filter args]]"""
import csv, io, subprocess, sys
from collections import defaultdict

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
EXTRA = sys.argv[3:]  # e.g. -k regex:name --launch-skip 1 -c 1
out = subprocess.run(["ncu", "-i", rep, *EXTRA, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg = defaultdict(int)
src_text = {}
cur_file = None
hdr = None
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] == "File Path":
        cur_file = row[1].split("/")[-1]
        continue
    if row[0] == "Line No":
        hdr = row
        continue
    if hdr is None or len(row) != len(hdr) or not row[0].isdigit():
        continue
    try:
        smp = int(row[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
    except ValueError:
        continue
    key = (cur_file, int(row[0]))
    agg[key] += smp
    src_text[key] = row[1].strip()[:100]
tot = sum(agg.values()) or 1
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:N]:
    print(f"{100 * v / tot:5.1f}% {k[0]}:{k[1]:<5} {src_text[k]}")
