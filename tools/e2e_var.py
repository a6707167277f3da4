"""Run-to-run spread of the pipelined end-to-end step (bench.py's e2e leg): R repetitions of K
steps in one process, with and without the nvidia-smi clock sampler running.  Prints JSON."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import ClockSampler  # noqa: E402
from paper_2311_16728_b200.build import build  # noqa: E402
from paper_2311_16728_b200.core import Renderer, pack_params  # noqa: E402
from paper_2311_16728_b200.mapping import MappingEngine  # noqa: E402
from synth import config, make_cameras, make_scene, perturb  # noqa: E402


def main(cname="tum", K=20, R=8):
    build()
    cfg = config(cname)
    scene = make_scene(cfg)
    cams = make_cameras(cfg, cfg["views"])
    rt = Renderer(scene.n, cfg["sh_degree"], len(cams), cams[0].width, cams[0].height, 8 << 20)
    gt = rt.forward(pack_params(scene), cams)[0].clone()
    del rt
    L = cfg["levels"] + 1
    eng = MappingEngine(perturb(scene, 99), cams, gt, n_levels=cfg["levels"])
    g = [gt.cpu().pin_memory() for _ in range(2)]
    o = [torch.empty((L, len(cams))).pin_memory() for _ in range(2)]
    eng.capture_pipelined(g, o)

    def timed(per_step=False):
        for _ in range(3):
            eng.step_pipelined()
        eng.pipeline_join()
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(K + 1)]
        ev[0].record()
        for k in range(K):
            eng.step_pipelined()
            if per_step:
                ev[k + 1].record()
        eng.pipeline_join()
        ev[K].record()
        torch.cuda.synchronize()
        tot = ev[0].elapsed_time(ev[K]) / K
        steps = [round(ev[k].elapsed_time(ev[k + 1]), 3) for k in range(K)] if per_step else None
        return round(tot, 4), steps

    out = {"no_sampler": [timed()[0] for _ in range(R)]}
    with ClockSampler(0):
        out["sampler"] = [timed()[0] for _ in range(R)]
        out["per_step_sampler"] = [timed(True) for _ in range(3)]
    out["per_step"] = [timed(True) for _ in range(3)]
    print(json.dumps(out))


if __name__ == "__main__":
    main(*(sys.argv[1:2] or ["tum"]))
