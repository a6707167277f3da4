"""the Table 3 ablation on a synthetic incremental-mapping run,
with gradient densify / prune (f1) and geometry-based densification (Geo, f2) on, for the
paper's rows: (1) w/o Geo, n = 2; (2) w/ Geo, w/o GP; (3) w/o Geo, w/o GP; (4) w/ Geo, n = 1;
(5) w/ Geo, n = 3; default w/ Geo, n = 2.

Setup (all synthetic, seeded): the target map is the config's scene; `keyframes` views of it are
the keyframe images (renders of the target map by this path).  Mapping starts from the sparse
map the geometry thread would hand over ("the geometry mapping component only
establishes sparse hyper primitives"): a random `sparse` fraction of the target's Gaussians,
perturbed.  Keypoints of a keyframe (monocular) are the pixels of target
Gaussians visible in it; `active_frac` of them are active (observed map points with their true
depth), the rest are inactive -- Geo back-projects those at the inverse-distance depth of their
4 nearest active neighbours (mono, R32), i.e. at inaccurate positions, the case the paper
credits GP with fixing.  Keyframes arrive one at a time; after each arrival (Geo: its temporary
primitives are added) the engine runs `iters` iterations over all keyframes so far, with the
Eq. 5 schedule restarted for the new keyframe (level = gp_level(i, n, iters / (n + 1))), and
densify / prune every `densify_every` iterations.  Reported per row: level-0 PSNR over all
keyframes, model size (Gaussians, MB), render FPS of one level-0 view (graph replay), device ms
of the mapping iterations.  Writes profiles/<tag>_gp_ablation.{json,md}.

    python tools/gp_ablation.py [--config tum] [--keyframes 6] [--iters 150] [--tag r02]
"""
import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

ROWS = [("(1)", False, 2), ("(2)", True, 0), ("(3)", False, 0), ("(4)", True, 1), ("(5)", True, 3),
        ("default", True, 2)]


def keypoints(scene, cam, n_kp, active_frac, seed):
    """Keypoint pixels = projections of target Gaussians in view (test input construction)."""
    import numpy as np
    rng = np.random.default_rng(seed)
    P = scene.means.astype(np.float64)
    pc = P @ cam.R.astype(np.float64).T + cam.t.astype(np.float64)
    z = pc[:, 2]
    ok = z > 0.3
    u = np.where(ok, cam.fx * pc[:, 0] / np.maximum(z, 1e-9) + cam.cx, -1)
    v = np.where(ok, cam.fy * pc[:, 1] / np.maximum(z, 1e-9) + cam.cy, -1)
    ok &= (u >= 0) & (u <= cam.width - 1) & (v >= 0) & (v <= cam.height - 1)
    idx = np.nonzero(ok)[0]
    pick = rng.choice(idx, size=min(n_kp, idx.size), replace=False)
    uv = np.stack([u[pick], v[pick]], 1).astype(np.float32)
    active = (rng.uniform(size=pick.size) < active_frac).astype(np.int32)
    kd = np.where(active == 1, z[pick], 0.0).astype(np.float32)
    return uv, active, kd


def main():
    import numpy as np
    import torch
    from paper_2311_16728_b200.build import build
    from paper_2311_16728_b200.core import DensifyConfig, Renderer, pack_params
    from paper_2311_16728_b200.mapping import MappingEngine, gp_level
    from synth import make_cameras, make_scene, perturb

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="tum")
    ap.add_argument("--keyframes", type=int, default=6)
    ap.add_argument("--iters", type=int, default=150, help="iterations after each keyframe arrival")
    ap.add_argument("--sparse", type=float, default=0.15)
    ap.add_argument("--active-frac", type=float, default=0.3)
    ap.add_argument("--keypoints", type=int, default=3000)
    ap.add_argument("--densify-every", type=int, default=50)
    ap.add_argument("--grad-threshold", type=float, default=2e-5,
                    help="mean ||dL/dmean2d|| (pixels of the level rendered) above which a Gaussian densifies")
    ap.add_argument("--tag", default="r02")
    args = ap.parse_args()
    build()
    target = make_scene(args.config)
    cams = make_cameras(args.config, args.keyframes, seed=77)
    H, W = cams[0].height, cams[0].width
    r = Renderer(target.n, target.sh_degree, len(cams), W, H, 8 << 20)
    gts = r.forward(pack_params(target), cams)[0].clone()
    del r
    rng = np.random.default_rng(3)
    sparse = perturb(target.subset(np.sort(rng.choice(target.n, int(args.sparse * target.n), replace=False))), 7)
    kps = [keypoints(target, c, args.keypoints, args.active_frac, 100 + k) for k, c in enumerate(cams)]
    rows = run_rows(args, ROWS, cams, gts, sparse, kps, {})
    # online mapping is time-bound (faster rendering buys more iterations): the
    # same rows again with each row's iterations scaled so its mapping time matches the row
    # with the same Geo setting and no GP
    ref = {r["geo"]: r["mapping_device_ms"] for r in rows if r["gp_levels_above_0"] == 0}
    scale = {r["row"]: ref[r["geo"]] / r["mapping_device_ms"] for r in rows}
    rows_t = run_rows(args, ROWS, cams, gts, sparse, kps, scale)
    write(args, target, rows, rows_t)


def run_rows(args, row_defs, cams, gts, sparse, kps, scale):
    import numpy as np
    import torch
    from paper_2311_16728_b200.core import DensifyConfig, Renderer
    from paper_2311_16728_b200.mapping import MappingEngine, gp_level
    H, W = cams[0].height, cams[0].width
    rows = []
    for name, geo, n in row_defs:
        iters = max(args.densify_every + 1, int(round(args.iters * scale.get(name, 1.0))))
        dcfg = DensifyConfig(grad_threshold=args.grad_threshold, scene_extent=2.5)
        eng = None
        dev_ms, added = 0.0, 0
        seed = 0
        for k in range(len(cams)):
            # keyframe k arrives: the engine maps keyframes 0..k (parameters, Adam state carry on)
            if eng is None:
                eng = MappingEngine(sparse, cams[:1], gts[:1], n_levels=n, densify_cfg=dcfg)
            else:
                eng.add_keyframe(cams[k], gts[k])
            if geo:
                uv, act, kd = kps[k]
                added += eng.add_keyframe_features(k, uv, act, kd, None, gts[k], mode=0)
            per = max(1, iters // (n + 1))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            for i in range(iters):
                eng.build_pyramids() if i == 0 else None
                eng.iteration(gp_level(i, n, per))
                if (i + 1) % args.densify_every == 0 and i + 1 < iters:
                    e1.record()
                    torch.cuda.synchronize()
                    dev_ms += e0.elapsed_time(e1)
                    seed += 1
                    eng.densify_and_prune(seed)
                    torch.cuda.synchronize()
                    e0.record()
            e1.record()
            torch.cuda.synchronize()
            dev_ms += e0.elapsed_time(e1)
        img = eng.render(0)[0]
        mse = float(((img - gts) ** 2).mean().item())
        psnr = 10.0 * math.log10(1.0 / max(mse, 1e-12))
        # render FPS of one level-0 view (CUDA-graph replay of A1-A6)
        one = Renderer(eng.n, eng.D, 1, W, H, max(eng.renderers[0].ws.capacity, 1 << 16))
        one.forward(eng.params, cams[:1])
        g = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            one.forward(eng.params, cams[:1])
        torch.cuda.current_stream().wait_stream(side)
        with torch.cuda.graph(g):
            one.forward(eng.params, cams[:1])
        for _ in range(3):
            g.replay()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(50):
            g.replay()
        b.record()
        torch.cuda.synchronize()
        fps = 1000.0 / (a.elapsed_time(b) / 50)
        row = {"row": name, "geo": geo, "gp_levels_above_0": n, "iters_per_keyframe": iters,
               "psnr_level0": psnr, "gaussians": eng.n,
               "model_mb": eng.n * eng.params.shape[0] * 4 / 1e6, "render_fps": fps, "mapping_device_ms": dev_ms,
               "geo_added": added}
        rows.append(row)
        print(json.dumps(row), flush=True)
    return rows


def write(args, target, rows, rows_t):
    out = {"config": args.config, "keyframes": args.keyframes, "iters_per_keyframe": args.iters,
           "sparse_start": f"{args.sparse:.0%} of the {target.n} target Gaussians, perturbed",
           "keypoints_per_keyframe": args.keypoints, "active_frac": args.active_frac,
           "densify_every": args.densify_every, "grad_threshold": args.grad_threshold, "geo_mode": "mono (R32)",
           "rows_equal_iterations": rows,
           "rows_equal_time": rows_t}
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    json.dump(out, open(os.path.join(ROOT, "profiles", f"{args.tag}_gp_ablation.json"), "w"), indent=1)
    lines = [f"# {args.tag}: Table 3 ablation, synthetic ({args.config}, {args.keyframes} keyframes, sparse start "
             f"{args.sparse:.0%}, densify/prune every {args.densify_every} iterations, mono Geo)", ""]
    for title, rr in ((f"equal iterations ({args.iters} per keyframe)", rows),
                      ("equal mapping time (iterations scaled to the no-GP row of the same Geo setting)", rows_t)):
        lines += [f"## {title}", "",
                  "| row | Geo | GP (n) | iters/keyframe | PSNR L0 (dB) | Gaussians | MB | render FPS | mapping ms |"
                  " Geo added |", "|---|---|---|---|---|---|---|---|---|---|"]
        for x in rr:
            lines.append(f"| {x['row']} | {'w/' if x['geo'] else 'w/o'} | {x['gp_levels_above_0'] or 'w/o'} | "
                         f"{x['iters_per_keyframe']} | {x['psnr_level0']:.2f} | {x['gaussians']} | {x['model_mb']:.1f} | "
                         f"{x['render_fps']:.0f} | {x['mapping_device_ms']:.0f} | {x['geo_added']} |")
        lines.append("")
    for d in ("profiles", "gpurun_out"):  # gpurun_out: what a GPU-box run brings back
        os.makedirs(os.path.join(ROOT, d), exist_ok=True)
        open(os.path.join(ROOT, d, f"{args.tag}_gp_ablation.md"), "w").write("\n".join(lines) + "\n")
        json.dump(out, open(os.path.join(ROOT, d, f"{args.tag}_gp_ablation.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
