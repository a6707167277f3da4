"""Summarise gpurun_out ncu artefacts into profiles/ (tracked):

    python tools/summarize_profiles.py <tag> [launches.csv] [report.ncu-rep] [config]

* <tag>_launches.csv / <tag>_launches.md: per-launch device times of one bench step
  (ncu --metrics gpu__time_duration.sum, cold-cache and serialised: compare shares);
* <tag>_ncu_<kernel>.txt: key --set full metrics per profiled launch (incl. dram bytes);
* profiles/traffic.json: dram__bytes_read.sum + dram__bytes_write.sum per kernel (mean per launch).
"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")


def launches(tag, path):
    rows = list(csv.reader(open(path)))
    hdr, out = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                out.append((d["Kernel Name"].split("(")[0].replace("void ", ""), float(d["Metric Value"]) / 1e3,
                            d.get("Grid Size", ""), d.get("Block Size", "")))
    shutil.copy(path, os.path.join(PROF, f"{tag}_launches.csv"))
    tot = sum(v for _, v, _, _ in out)
    agg, cnt = defaultdict(float), defaultdict(int)
    for k, v, _, _ in out:
        agg[k] += v
        cnt[k] += 1
    lines = [f"# {tag}: kernel launches of one bench step (ncu gpu__time_duration.sum, us)", "",
             f"total {tot:.1f} us over {len(out)} launches (cold-cache, serialised)", "",
             "| kernel | launches | total us | share |", "|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1]):
        lines.append(f"| {k} | {cnt[k]} | {v:.1f} | {100 * v / tot:.1f}% |")
    lines += ["", "| # | kernel | us | grid | block |", "|---|---|---|---|---|"]
    for i, (k, v, g, b) in enumerate(out):
        lines.append(f"| {i} | {k} | {v:.1f} | {g} | {b} |")
    open(os.path.join(PROF, f"{tag}_launches.md"), "w").write("\n".join(lines) + "\n")


WANT = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Achieved Occupancy",
        "Theoretical Occupancy", "Registers Per Thread", "Executed Ipc Active", "Issue Slots Busy",
        "Warp Cycles Per Issued Instruction", "Executed Instructions", "Grid Size", "Block Size",
        "L2 Hit Rate", "Branch Efficiency", "Avg. Active Threads Per Warp"]


def report(tag, rep, cfg_name="tum"):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    traffic = defaultdict(list)
    r = list(csv.reader(io.StringIO(raw)))
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    if r:
        h, units = r[0], r[1]
        kn = h.index("Kernel Name")
        try:
            rd, wr = h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
        except ValueError:
            rd = wr = None
        for row in r[2:]:
            if rd is None or len(row) != len(h):
                continue
            name = row[kn].split("(")[0].replace("void ", "").split("<")[0]
            try:
                traffic[name].append(float(row[rd].replace(",", "")) * scale.get(units[rd], 1.0) +
                                     float(row[wr].replace(",", "")) * scale.get(units[wr], 1.0))
            except ValueError:
                pass
    d = list(csv.reader(io.StringIO(det)))
    per = defaultdict(list)
    if d:
        h = d[0]
        ki, ii, mn, mv, mu = (h.index(x) for x in ("Kernel Name", "ID", "Metric Name", "Metric Value",
                                                    "Metric Unit"))
        for row in d[1:]:
            if len(row) > mv and row[mn] in WANT:
                per[(row[ii], row[ki].split("(")[0].replace("void ", ""))].append(f"{row[mn]}: {row[mv]} {row[mu]}")
    by_kernel = defaultdict(list)
    for (i, k), lines in per.items():
        by_kernel[k.split("<")[0]].append((i, lines))
    for k, items in by_kernel.items():
        with open(os.path.join(PROF, f"{tag}_ncu_{k.replace('gsk::', '')}.txt"), "w") as f:
            f.write(f"# {tag} ncu --set full summary: {k} (source {os.path.basename(rep)})\n")
            for i, lines in sorted(items, key=lambda x: int(x[0])):
                f.write(f"\n## launch id {i}\n")
                f.write("\n".join(lines) + "\n")
            t = traffic.get(k.split("<")[0], [])
            if t:
                f.write(f"\ndram bytes (read + write) per launch: {', '.join(f'{x / 1e6:.2f} MB' for x in t)}\n")
    tj = os.path.join(PROF, "traffic.json")
    data = json.load(open(tj)) if os.path.exists(tj) else {}
    cfg = data.setdefault(cfg_name, {})
    for k, v in traffic.items():
        cfg[k.replace("gsk::", "")] = sum(v) / len(v)
    # bench.py times kernel families (one libgs.so scope each per GP level, gs_profile_kernel):
    # traffic per scope = all member launches' bytes in the captured step / the scope's count
    fam = {"k_raster_bwd": (("k_raster_bwd",), "k_raster_bwd"), "k_raster_fwd": (("k_raster_fwd", "k_chunk_index",
           "k_tile_order"), "k_raster_fwd"), "k_tile_sort": (("k_tile_sort_small", "k_tile_sort_big"),
           "k_tile_sort_small"), "k_ssim": (("k_ssim_fwd", "k_ssim_bwd", "k_loss_final"), "k_ssim_fwd")}
    names = {k.replace("gsk::", ""): v for k, v in traffic.items()}
    for f, (members, anchor) in fam.items():
        tot = sum(x for k, v in names.items() if k.startswith(members) for x in v)
        n = sum(len(v) for k, v in names.items() if k.startswith(anchor))
        if n:
            cfg[f] = tot / n
    json.dump(data, open(tj, "w"), indent=1)


if __name__ == "__main__":
    tag = sys.argv[1]
    os.makedirs(PROF, exist_ok=True)
    if len(sys.argv) > 2:
        launches(tag, sys.argv[2])
    if len(sys.argv) > 3:
        report(tag, sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else "tum")
