"""Top SASS lines by warp-stall samples for one kernel of an ncu report.
usage: python tools/ncu_hot.py <report> <kernel-regex> [N]"""
import csv, io, re, subprocess, sys

rep, kre = sys.argv[1], sys.argv[2]
N = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
blocks = re.split(r'^"Kernel Name",', out, flags=re.M)
for b in blocks[1:]:
    name = b.split("\n", 1)[0]
    if not re.search(kre, name):
        continue
    rows = list(csv.reader(io.StringIO(b.split("\n", 1)[1])))
    h = rows[0]
    si, ai = h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
    data = [(int(r[si] or 0), r[ai].strip(), i) for i, r in enumerate(rows[1:]) if len(r) == len(h)]
    tot = sum(d[0] for d in data)
    print(name[:90], "total samples", tot, "instructions", len(data))
    for s, src, i in sorted(data, reverse=True)[:N]:
        print(f"{100*s/tot:5.1f}% [{i:5d}] {src}")
    break
