"""Compare per-kernel totals of ncu launch lists: python tools/ab_compare_ll.py a.csv b.csv ..."""
import csv
import sys
from collections import defaultdict


def load(p):
    rows = list(csv.reader(open(p)))
    hdr, tot = None, defaultdict(float)
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                v = float(d["Metric Value"].replace(",", ""))
                unit = d.get("Metric Unit", "ns")
                tot[d["Kernel Name"].split("(")[0][:40]] += v / (1000.0 if unit in ("nsecond", "ns") else 1.0)
    return tot


tabs = [load(p) for p in sys.argv[1:]]
names = sorted(set().union(*tabs), key=lambda k: -tabs[0].get(k, 0))
print("%-40s" % "kernel", " ".join("%10s" % p.split("/")[-1][:10] for p in sys.argv[1:]))
for k in names:
    print("%-40s" % k, " ".join("%10.1f" % t.get(k, 0) for t in tabs))
print("%-40s" % "TOTAL", " ".join("%10.1f" % sum(t.values()) for t in tabs))
