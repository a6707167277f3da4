"""Binning at scale (no oracle: 125 M pairs): the bucket path's keys are sorted with (depth, id)
order inside every tile, its ranges tile the pair array, and the radix path (key duplication +
onesweep LSD sort) gives the same keys and values.  python tools/check_binning_scale.py [cfg] [views]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2311_16728_b200 import _lib as L  # noqa: E402
from paper_2311_16728_b200.build import build  # noqa: E402
from paper_2311_16728_b200.core import Renderer, pack_params  # noqa: E402
from synth import make_cameras, make_scene  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "stress"
    views = int(sys.argv[2]) if len(sys.argv) > 2 else 64
    build()
    scene = make_scene(cfg)
    cams = make_cameras(cfg, views)
    params = pack_params(scene)
    out = {}
    for binning in (0, 1):
        L.gs_set_binning(binning)
        r = Renderer(scene.n, scene.sh_degree, views, cams[0].width, cams[0].height, 1 << 20)
        r.forward(params, cams)
        st, flags, P = r.ws.status()
        r = Renderer(scene.n, scene.sh_degree, views, cams[0].width, cams[0].height, int(P * 1.05) + 4096)
        r.forward(params, cams)
        torch.cuda.synchronize()
        st, flags, P = r.ws.status()
        v = r.ws.views()
        k = v["keys"][:P].clone()
        vals = v["vals"][:P].clone()
        ranges = v["ranges"].clone()
        out[binning] = (k, vals, ranges, P, st)
        del r
        torch.cuda.empty_cache()
    L.gs_set_binning(0)
    k0, v0, r0, P0, s0 = out[0]
    k1, v1, r1, P1, s1 = out[1]
    print("status", s0, s1, "pairs", P0, P1)
    ku = k0.view(torch.int64)
    sorted_ok = bool((ku[1:] >= ku[:-1]).all().item()) if P0 > 1 else True
    print("bucket keys non-decreasing:", sorted_ok)
    if not sorted_ok:
        bad = torch.nonzero(ku[1:] < ku[:-1]).flatten()
        print("first unsorted positions", bad[:10].tolist(), "count", bad.numel())
        i = int(bad[0])
        print("keys around", [hex(int(x) & 0xFFFFFFFFFFFFFFFF) for x in ku[max(0, i - 3):i + 4].tolist()])
    eqk = torch.equal(k0, k1)
    eqv = torch.equal(v0, v1)
    print("keys equal:", eqk, "vals equal:", eqv, "ranges equal:", torch.equal(r0, r1))
    if not eqk:
        d = torch.nonzero(k0 != k1).flatten()
        print("key mismatches", d.numel(), "first", d[:10].tolist())
    if eqk and not eqv:
        d = torch.nonzero(v0 != v1).flatten()
        print("val mismatches", d.numel(), "first", d[:10].tolist())


if __name__ == "__main__":
    main()
