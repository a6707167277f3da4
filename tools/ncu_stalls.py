"""Warp-stall samples per CUDA source line of one kernel launch in an ncu report (source page).
usage: python tools/ncu_stalls.py <report> <kernel-regex> [N] [launch-skip]"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
N = int(sys.argv[3]) if len(sys.argv) > 3 else 30
skip = sys.argv[4] if len(sys.argv) > 4 else "0"
out = subprocess.run(["ncu", "-i", rep, "-k", f"regex:{kre}", "--launch-skip", skip, "-c", "1", "--page", "source",
                      "--csv", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if len(r) > 4 and r[0] == "Line No")
ci = hdr.index("Warp Stall Sampling (All Samples)")
tot, byline = 0, {}
for r in rows:
    if len(r) > ci and r[0].isdigit():
        try:
            v = int(r[ci].replace(",", "") or 0)
        except ValueError:
            continue
        k = r[0] + " " + r[1].strip()[:90]
        byline[k] = byline.get(k, 0) + v
        tot += v
print("stall samples", tot)
for k, v in sorted(byline.items(), key=lambda x: -x[1])[:N]:
    print("%5.1f%% %s" % (100 * v / max(tot, 1), k))
