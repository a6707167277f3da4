"""Gaussian-pyramid ablation direction check (Table 3; Eq. 5).

For n in {0, 1, 2, 3} pyramid levels above the full resolution, optimise the same perturbed
synthetic map against the same keyframe with the Eq. 5 schedule (level = gp_level(i, n, T / (n+1)),
SPEC.md:443-451) for T iterations, then report the level-0 PSNR against the target and the device
time of the T iterations.  Writes profiles/<tag>_gp_ablation.{json,md}.

    python tools/gp_ablation.py [--config tum] [--iters 600] [--tag r01]
"""
import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2311_16728_b200.build import build
    from paper_2311_16728_b200.core import Renderer, pack_params
    from paper_2311_16728_b200.mapping import MappingEngine, gp_level
    from synth import make_cameras, make_scene, perturb

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="tum")
    ap.add_argument("--iters", type=int, default=600)
    ap.add_argument("--tag", default="r01")
    args = ap.parse_args()
    build()
    scene = make_scene(args.config)
    cams = make_cameras(args.config, 1)
    p0 = pack_params(scene)
    r = Renderer(scene.n, 3, 1, cams[0].width, cams[0].height, 1 << 22)
    gt = r.forward(p0, cams)[0].clone()
    del r
    start = perturb(scene, 7)
    rows = []
    for n in (0, 1, 2, 3):
        eng = MappingEngine(start, cams, gt, n_levels=n)
        per = max(1, args.iters // (n + 1))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(args.iters):
            eng.iteration(gp_level(i, n, per))
        e1.record()
        torch.cuda.synchronize()
        img = eng.render(0)[0]
        mse = float(((img - gt) ** 2).mean().item())
        psnr = 10.0 * math.log10(1.0 / max(mse, 1e-12))
        loss0 = float(eng.losses[0](img, gt, grad=False)[0][0].item())
        rows.append({"n_levels_above_0": n, "iterations": args.iters, "iters_per_level": per,
                     "device_ms": e0.elapsed_time(e1), "psnr_level0": psnr, "loss_level0": loss0})
        print(json.dumps(rows[-1]), flush=True)
    out = {"config": args.config, "n_gaussians": scene.n, "schedule": "Eq. 5: level = max(0, n - i // per)",
           "target": "render of the unperturbed synthetic map (perturbed start, seed 7)", "runs": rows}
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    json.dump(out, open(os.path.join(ROOT, "profiles", f"{args.tag}_gp_ablation.json"), "w"), indent=1)
    lines = [f"# {args.tag}: Gaussian-pyramid ablation ({args.config}, {scene.n} Gaussians, {args.iters} iterations)",
             "", "| levels above 0 (n) | iters/level | device ms | PSNR L0 (dB) | loss L0 |", "|---|---|---|---|---|"]
    for x in rows:
        lines.append(f"| {x['n_levels_above_0']} | {x['iters_per_level']} | {x['device_ms']:.1f} | "
                     f"{x['psnr_level0']:.2f} | {x['loss_level0']:.5f} |")
    open(os.path.join(ROOT, "profiles", f"{args.tag}_gp_ablation.md"), "w").write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
