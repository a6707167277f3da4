"""One mapping iteration (A1-A11, both binning paths, the chunked and tile raster paths) on a
small input, for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):

    compute-sanitizer --tool racecheck python tools/sanitize_step.py tiny 0
    compute-sanitizer --tool racecheck python tools/sanitize_step.py tum 2 20000
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import oracle.oracle as orc  # noqa: E402  (level cameras: test-input preparation)
from paper_2311_16728_b200 import _lib as L  # noqa: E402
from paper_2311_16728_b200.core import (Adam, PhotometricLoss, Renderer, gaussian_pyramid,  # noqa: E402
                                        pack_params)
from synth import make_cameras, make_scene, noise_image  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "tiny"
    level = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    n = int(sys.argv[3]) if len(sys.argv) > 3 else None
    views = int(sys.argv[4]) if len(sys.argv) > 4 else 1
    scene = make_scene(cfg, n=n)
    cams = [orc.level_camera(c, level) for c in make_cameras(cfg, views)]
    H, W = cams[0].height, cams[0].width
    D = scene.sh_degree
    gt = torch.from_numpy(noise_image(H, W, 1)).float().cuda()[None].expand(views, 3, H, W).contiguous()
    gaussian_pyramid(gt, 2 if min(H, W) > 8 else 0)
    for binning in (0, 1):
        L.gs_set_binning(binning)
        params = pack_params(scene)
        r = Renderer(scene.n, D, views, W, H, 1 << 20)
        rgb, T = r.forward(params, cams)
        loss, dL = PhotometricLoss(views, H, W)(rgb, gt)
        grads = torch.zeros_like(params)
        gn = torch.zeros(scene.n, device="cuda")
        r.backward(params, cams, dL, grads, gn)
        Adam(params, scene.n, D).step(grads)
        r.forward(params, cams)
        r.backward_adam(params, cams, dL, Adam(params, scene.n, D), gn)
        torch.cuda.synchronize()
        st, flags, P = r.ws.status()
        print(f"binning {binning}: status {st} flags {flags} pairs {P} loss {loss.sum().item():.5f}", flush=True)
    L.gs_set_binning(0)


if __name__ == "__main__":
    main()
