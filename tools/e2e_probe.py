"""Where does the end-to-end step lose time against the device-resident graph replay?
Times, on one GPU, K steps of: (A) capture()/replay(), (B) capture_pipelined with pinned host
targets, (C) the same with device-resident 'host' buffers (D2D copies), (D) capture() with
pinned host targets (step_host inside the graph, no prefetch).  Prints one JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2311_16728_b200.build import build  # noqa: E402
from paper_2311_16728_b200.core import Renderer, pack_params  # noqa: E402
from paper_2311_16728_b200.mapping import MappingEngine  # noqa: E402
from synth import config, make_cameras, make_scene, perturb  # noqa: E402


def main(cname="tum", K=40):
    build()
    cfg = config(cname)
    scene = make_scene(cfg)
    cams = make_cameras(cfg, cfg["views"])
    rt = Renderer(scene.n, cfg["sh_degree"], len(cams), cams[0].width, cams[0].height, 8 << 20)
    gt = rt.forward(pack_params(scene), cams)[0].clone()
    del rt
    L = cfg["levels"] + 1

    def timed(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(K):
            fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / K

    out = {}
    eng = MappingEngine(perturb(scene, 99), cams, gt, n_levels=cfg["levels"])
    eng.capture()
    out["A_replay_ms"] = timed(eng.replay)
    del eng
    for name, mk in (("B_pipelined_pinned_ms", lambda: gt.cpu().pin_memory()),
                     ("C_pipelined_device_ms", lambda: gt.clone())):
        eng = MappingEngine(perturb(scene, 99), cams, gt, n_levels=cfg["levels"])
        g = [mk() for _ in range(2)]
        o = [torch.empty((L, len(cams))).pin_memory() for _ in range(2)]
        eng.capture_pipelined(g, o)
        out[name] = timed(eng.step_pipelined)
        del eng
    eng = MappingEngine(perturb(scene, 99), cams, gt, n_levels=cfg["levels"])
    gp = gt.cpu().pin_memory()
    op = torch.empty((L, len(cams))).pin_memory()
    eng.capture(gp, op)
    out["D_replay_host_serial_ms"] = timed(eng.replay)
    out["h2d_MB"] = gt.numel() * 4 / 1e6
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main(*(sys.argv[1:2] or ["tum"]))
