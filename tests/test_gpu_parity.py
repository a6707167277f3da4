"""GPU parity of the CUDA path (libgs.so through the C ABI) against the CPU oracle, on the same
seeded synthetic inputs (SURVEY §8(c) parity contract):

1. decision quantities (cull, radius, rect, tiles, depth, mean2d, conic): bit-exact;
2. binning keys, values, ranges: bit-exact;
3. colour and final T: |d| <= 1e-4 on pixels outside the oracle's ambiguity band; flagged
   pixels <= 1e-3 of all and each within 1.1e-2;
4. last contributor equal on non-flagged pixels;
5. gradients: |d| <= 1e-3 max(|g_ref|, 5e-2 RMS_class(g_ref)) outside Gaussians touching
   flagged pixels (the floor covers fp32 accumulation of cancelling per-pixel terms, DESIGN.md
   "Tolerances"); loss rel <= 1e-5;
6. pyramid |d| <= 1e-6; Adam rel <= 1e-6 after one step.
"""
import math

import numpy as np
import pytest
import torch

import oracle.oracle as orc
from paper_2311_16728_b200 import _lib as L
from paper_2311_16728_b200.core import (Adam, AdamConfig, PhotometricLoss, Renderer, gaussian_pyramid, pack_params,
                                        unpack)
from paper_2311_16728_b200.mapping import MappingEngine
from synth import make_cameras, make_scene, noise_image, perturb

scaled_camera = orc.level_camera

pytestmark = pytest.mark.gpu

CLASSES = ["means", "quats", "log_scales", "opacity_logits", "sh"]


@pytest.fixture(scope="module", autouse=True)
def _setup():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2311_16728_b200.build import build
    build()
    L.lib()


def _renderer(scene, cams, cap=None):
    n = scene.means.shape[0]
    D = int(round(math.sqrt(scene.sh.shape[1]))) - 1
    params = pack_params(scene)
    if cap is None:
        _, _, _, tt = orc.bin_pairs(scene, cams)
        cap = int(tt.sum()) + 4096
    r = Renderer(n, D, len(cams), cams[0].width, cams[0].height, cap)
    return r, params, D


def _sample_pixels(V, H, W, k, seed):
    rng = np.random.default_rng(seed)
    idx = rng.choice(V * H * W, size=min(k, V * H * W), replace=False)
    v, rem = np.divmod(idx, H * W)
    y, x = np.divmod(rem, W)
    return np.stack([v, y, x], 1).astype(np.int32)


# ------------------------------------------------------------------------------ recipe pieces
def test_exp_scale_bit_exact():
    """The recipe's e = (float)exp((double)s) on the GPU equals the oracle's, over every 7th
    fp32 bit pattern of log-scales in [-12, 3] (DESIGN.md fp32 recipe)."""
    lo = np.array([-12.0], np.float32).view(np.uint32)[0]
    hi = np.array([3.0], np.float32).view(np.uint32)[0]
    neg = np.arange(np.array([-0.0], np.float32).view(np.uint32)[0], lo, 7, dtype=np.uint32)
    pos = np.arange(0, hi, 7, dtype=np.uint32)
    for chunk in (neg, pos):
        s = chunk.view(np.float32)
        ref = orc.exp_scale_f32(s)
        st = torch.from_numpy(s).cuda()
        out = torch.empty_like(st)
        L.gs_debug_exp_scale(st, out)
        got = out.cpu().numpy()
        bad = np.nonzero(got.view(np.uint32) != ref.view(np.uint32))[0]
        assert bad.size == 0, (bad.size, s[bad[:5]])


@pytest.fixture(params=[0, 1], ids=["buckets", "radix"])
def binning(request):
    L.gs_set_binning(request.param)
    yield request.param
    L.gs_set_binning(0)


@pytest.mark.parametrize("cfg,n,views,level", [("tiny", None, 1, 0), ("tum", 60000, 1, 0), ("tum", 60000, 3, 2),
                                               ("replica", 40000, 2, 1), ("tum", None, 1, 2)])
def test_preprocess_and_binning_bit_exact(cfg, n, views, level, binning):
    """Both binning paths (tile buckets + in-tile sort; global onesweep radix sort) give the
    oracle's keys, values and ranges bit for bit (SURVEY §8(c) contract item 2)."""
    scene = make_scene(cfg, n=n)
    cams = [scaled_camera(c, level) for c in make_cameras(cfg, views)]
    r, params, D = _renderer(scene, cams)
    r.forward(params, cams)
    torch.cuda.synchronize()
    v = r.ws.views()
    N = scene.means.shape[0]
    for k, cam in enumerate(cams):
        o = orc.project(scene, cam, "recipe")
        sl = slice(k * N, (k + 1) * N)
        rad = v["radius"][sl].cpu().numpy()
        np.testing.assert_array_equal(rad, o["radius"])
        vis = o["radius"] > 0
        np.testing.assert_array_equal(v["rect"][sl].cpu().numpy()[vis], o["rect"][vis])
        np.testing.assert_array_equal(v["depth"][sl].cpu().numpy()[vis].view(np.uint32), o["depth_bits"][vis])
        np.testing.assert_array_equal(v["mean2d"][sl].cpu().numpy()[vis].view(np.uint32),
                                      o["mean2d_f"][vis].view(np.uint32))
        np.testing.assert_array_equal(v["conic"][sl].cpu().numpy()[vis].view(np.uint32),
                                      o["conic_f"][vis].view(np.uint32))
    keys, vals, ranges, tt = orc.bin_pairs(scene, cams)
    st, flags, P = r.ws.status()
    assert st == L.GS_OK and flags == 0 and P == keys.size
    np.testing.assert_array_equal(v["tiles_touched"].cpu().numpy(), tt.reshape(-1))
    np.testing.assert_array_equal(v["keys"][:P].cpu().numpy().view(np.uint64), keys)
    np.testing.assert_array_equal(v["vals"][:P].cpu().numpy().view(np.uint32), vals)
    np.testing.assert_array_equal(v["ranges"].cpu().numpy().view(np.uint32), ranges)


@pytest.mark.parametrize("n,bits,kind", [(1, 40, "rand"), (4095, 44, "depth"), (4096, 44, "rand"),
                                         (4097, 48, "depth"), (300_001, 44, "depth"), (1_000_003, 64, "rand"),
                                         (2_000_000, 12, "rand"), (3_000_017, 50, "depth"), (5_000_000, 20, "rand"),
                                         (40_000_003, 50, "depth")])
def test_radix_sort_stable(n, bits, kind):
    rng = np.random.default_rng(n)
    if bits > 32:
        hi = rng.integers(0, 1 << (bits - 32), size=n, dtype=np.uint64)
        if kind == "depth":  # float bits of depths in [0.5, 8): constant top bits (skipped passes)
            lo = np.sort(rng.uniform(0.5, 8.0, size=n).astype(np.float32)).view(np.uint32).astype(np.uint64)
        else:
            lo = rng.integers(0, 1 << 32, size=n, dtype=np.uint64)
        keys = (hi << np.uint64(32)) | lo
    else:
        keys = rng.integers(0, 1 << bits, size=n, dtype=np.uint64)
    if n > 10:
        keys[rng.integers(0, n, size=n // 10)] = keys[0]  # many ties
    vals = np.arange(n, dtype=np.uint32)
    k = torch.from_numpy(keys.view(np.int64)).cuda()
    v = torch.from_numpy(vals.view(np.int32)).cuda()
    k2, v2 = torch.empty_like(k), torch.empty_like(v)
    temp = torch.empty(L.gs_sort_temp_size(n, bits), dtype=torch.uint8, device="cuda")
    L.gs_debug_sort_pairs(k, v, k2, v2, bits, temp)
    order = np.argsort(keys, kind="stable")
    np.testing.assert_array_equal(k.cpu().numpy().view(np.uint64), keys[order])
    np.testing.assert_array_equal(v.cpu().numpy().view(np.uint32), vals[order])


# ------------------------------------------------------------------------------ forward
def _check_colour(got_rgb, got_T, ref, pixels_mask=None):
    flag = ref["flag"].astype(bool)
    d = np.abs(got_rgb - ref["rgb"]).max(axis=-1 if got_rgb.ndim == 2 else 1)
    dT = np.abs(got_T - ref["T"])
    ok = ~flag
    assert flag.mean() <= 1e-3 + 1e-9, flag.mean()
    assert d[ok].max(initial=0) <= 1e-4, d[ok].max()
    assert dT[ok].max(initial=0) <= 1e-4, dT[ok].max()
    assert d[flag].max(initial=0) <= 1.1e-2


@pytest.mark.parametrize("n", [6000, 12000, 20000])
def test_long_tile_bucket_sorts(n):
    """Tile lists longer than one 4096-pair window are sorted window by window with global merge
    stages in between (2, 3 and 5 windows here); they must match the oracle's binning exactly."""
    from tests.helpers import camera, scene_of
    rng = np.random.default_rng(5)
    means = np.stack([rng.uniform(-0.02, 0.02, n), rng.uniform(-0.02, 0.02, n), rng.uniform(1.0, 3.0, n)], 1)
    scene = scene_of(means, log_scales=np.full((n, 3), np.log(0.002)), D=0)
    scene.depth_ties = None
    cams = [camera(width=64, height=48, cx=32, cy=24, fx=60, fy=60)]
    r, params, D = _renderer(scene, cams)
    r.forward(params, cams)
    torch.cuda.synchronize()
    keys, vals, ranges, tt = orc.bin_pairs(scene, cams)
    assert (ranges[:, 1] - ranges[:, 0]).max() > 4096
    v = r.ws.views()
    st, flags, P = r.ws.status()
    assert P == keys.size
    np.testing.assert_array_equal(v["keys"][:P].cpu().numpy().view(np.uint64), keys)
    np.testing.assert_array_equal(v["vals"][:P].cpu().numpy().view(np.uint32), vals)
    np.testing.assert_array_equal(v["ranges"].cpu().numpy().view(np.uint32), ranges)


def test_forward_parity_tiny_full_image():
    scene = make_scene("tiny")
    cams = make_cameras("tiny", 1)
    r, params, _ = _renderer(scene, cams)
    rgb, T = r.forward(params, cams)
    ref = orc.render(scene, cams, "recipe")
    _check_colour(rgb.cpu().numpy(), T.cpu().numpy(), ref)
    # last contributor (Gaussian id) equal on non-flagged pixels
    v = r.ws.views()
    nc = v["n_contrib"].cpu().numpy().reshape(1, cams[0].height, cams[0].width)
    ranges = v["ranges"].cpu().numpy()
    vals = v["vals"].cpu().numpy()
    TX = r.ws.tiles_x
    ys, xs = np.mgrid[0:cams[0].height, 0:cams[0].width]
    tile = (ys // 16) * TX + xs // 16
    last = np.where(nc[0] > 0, vals[np.clip(ranges[tile, 0] + nc[0] - 1, 0, None)], -1)
    ok = ref["flag"][0] == 0
    np.testing.assert_array_equal(last[ok], ref["last"][0][ok])
    assert (ref["ncomp"] > 0).mean() > 0.3
    # composited counts (a diagnostic output, gs_set_render_stats) equal the oracle's
    L.gs_set_render_stats(True)
    try:
        r.forward(params, cams)
        torch.cuda.synchronize()
        nco = r.ws.views()["n_composited"].cpu().numpy().reshape(cams[0].height, cams[0].width)
    finally:
        L.gs_set_render_stats(False)
    np.testing.assert_array_equal(nco[ok], ref["ncomp"][0][ok])


@pytest.mark.parametrize("cfg,views,level", [("tum", 1, 0), ("tum", 1, 2), ("euroc", 4, 1), ("euroc", 2, 0), ("replica", 1, 0)])
def test_forward_parity_full_size_sampled(cfg, views, level):
    scene = make_scene(cfg)
    cams = [scaled_camera(c, level) for c in make_cameras(cfg, views)]
    r, params, _ = _renderer(scene, cams, cap=None)
    rgb, T = r.forward(params, cams)
    H, W = cams[0].height, cams[0].width
    pix = _sample_pixels(views, H, W, 4096, 7)
    ref = orc.render(scene, cams, "recipe", pixels=pix)
    g = rgb.cpu().numpy()[pix[:, 0], :, pix[:, 1], pix[:, 2]]
    gT = T.cpu().numpy()[pix[:, 0], pix[:, 1], pix[:, 2]]
    _check_colour(g, gT, ref)


def test_forward_deterministic_and_empty():
    scene = make_scene("tum", n=50000)
    cams = make_cameras("tum", 1)
    r, params, _ = _renderer(scene, cams)
    a = r.forward(params, cams)[0].clone()
    b = r.forward(params, cams)[0].clone()
    assert torch.equal(a, b)
    # all Gaussians behind the camera: empty image, T = 1
    s2 = scene.copy()
    s2.means[:] = cams[0].centre() - 5 * cams[0].R[2]
    r2, p2, _ = _renderer(s2, cams, cap=4096)
    rgb, T = r2.forward(p2, cams)
    assert rgb.abs().max().item() == 0 and T.min().item() == 1.0


def test_capacity_overflow_flag_and_stale_state():
    scene = make_scene("tiny")
    cams = make_cameras("tiny", 1)
    r, params, D = _renderer(scene, cams, cap=1)  # rounds up to 4096 pairs
    s2 = scene.copy()
    s2.log_scales += 2.5  # huge footprints: far more than 4096 pairs
    p2 = pack_params(s2)
    r.forward(p2, cams)
    st, flags, P = r.ws.status()
    assert st == L.GS_ERR_CAPACITY and flags & 1 and P > 4096
    # backward with other cameras than the last forward -> StaleRenderState
    import dataclasses
    cam2 = [dataclasses.replace(cams[0], t=cams[0].t + np.float32(0.01))]
    grads = torch.zeros_like(p2)
    dL = torch.zeros((1, 3, cams[0].height, cams[0].width), device="cuda")
    with pytest.raises(L.GsError) as e:
        r.backward(p2, cam2, dL, grads)
    assert e.value.status == L.GS_ERR_STALE_STATE


# ------------------------------------------------------------------------------ loss / pyramid / adam
@pytest.mark.parametrize("V,H,W", [(1, 16, 16), (2, 45, 61), (1, 120, 160)])
def test_loss_parity(V, H, W):
    rng = np.random.default_rng(H * W)
    x = rng.uniform(0, 1, size=(V, 3, H, W)).astype(np.float32)
    y = rng.uniform(0, 1, size=(V, 3, H, W)).astype(np.float32)
    y[:, :, : H // 3] = x[:, :, : H // 3]  # some exactly equal pixels (L1 subgradient 0)
    pl = PhotometricLoss(V, H, W, 0.2)
    loss, dL = pl(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda())
    loss, dL = loss.cpu().numpy(), dL.cpu().numpy()
    for v in range(V):
        l_ref, _, d_ref = orc.loss(x[v], y[v], 0.2)
        assert loss[v] == pytest.approx(l_ref, rel=1e-5)
        np.testing.assert_allclose(dL[v], d_ref, rtol=1e-3, atol=1e-3 * np.abs(d_ref).max())


def test_pyramid_parity():
    rng = np.random.default_rng(0)
    img = rng.uniform(size=(2, 3, 37, 50)).astype(np.float32)
    lv = gaussian_pyramid(torch.from_numpy(img).cuda(), 2)
    for k in range(2):
        ref = orc.pyramid(img[k], 2)
        for l in range(3):
            np.testing.assert_allclose(lv[l][k].cpu().numpy(), ref[l], atol=1e-6, rtol=0)
    with pytest.raises(L.GsError):
        gaussian_pyramid(torch.zeros((1, 3, 8, 8), device="cuda"), 3)


@pytest.mark.parametrize("sgd", [False, True])
def test_adam_parity(sgd):
    """One fused step from identical generator inputs (p, g, m, v, t = 3) vs the fp64 oracle:
    p within 2 ulp + 1e-6 |dp|, moments rel 1e-6 (SURVEY §8(c) contract item 6)."""
    rng = np.random.default_rng(3)
    scene = make_scene("tiny", n=777)
    n = scene.means.shape[0]
    params = pack_params(scene)
    K, ld = params.shape
    g_np = rng.normal(size=(K, ld)).astype(np.float32)
    m_np = (0.1 * rng.normal(size=(K, ld))).astype(np.float32)
    v_np = (0.01 * rng.uniform(size=(K, ld)) ** 2).astype(np.float32)
    g_np[:, n:] = m_np[:, n:] = v_np[:, n:] = 0
    cfg = AdamConfig(sgd=sgd, lr_means=1e-2)
    opt = Adam(params, n, 0, cfg)
    opt.m.copy_(torch.from_numpy(m_np))
    opt.v.copy_(torch.from_numpy(v_np))
    opt.t = 2
    p_in = params.cpu().numpy().astype(np.float64)
    g = torch.from_numpy(g_np).cuda()
    opt.step(g, zero_grads=True)
    assert g.abs().max().item() == 0
    lrs = cfg.struct().lr
    rows_lr = [lrs[0]] * 3 + [lrs[1]] * 4 + [lrs[2]] * 3 + [lrs[3]] + [lrs[4]] * 3 + [lrs[5]] * (K - 14)
    got_p, got_m, got_v = params.cpu().numpy(), opt.m.cpu().numpy(), opt.v.cpu().numpy()
    for row, lr in enumerate(rows_lr):
        p_ref, m_ref, v_ref = orc.adam(p_in[row, :n], g_np[row, :n], m_np[row, :n], v_np[row, :n],
                                       lr=np.float32(lr).item(), beta1=np.float32(0.9).item(),
                                       beta2=np.float32(0.999).item(), eps=np.float32(1e-15).item(), step=3,
                                       sgd_mode=sgd)
        dp = np.abs(p_ref - p_in[row, :n])
        ulp = np.spacing(np.abs(p_ref).astype(np.float32)).astype(np.float64)
        # fp32 rounding of m = b1 m + (1 - b1) g is relative to its terms (cancellation), and
        # propagates into the step through lr / bc1 / (sqrt(v_hat) + eps)
        term_m = np.maximum(np.abs(0.9 * m_np[row, :n]), np.abs(0.1 * g_np[row, :n])).astype(np.float32)
        m_tol = 2 * np.spacing(term_m).astype(np.float64)
        if sgd:
            prop = 0.0
        else:
            bc1, bc2 = 1 - 0.9 ** 3, 1 - 0.999 ** 3
            prop = lr / bc1 * m_tol / (np.sqrt(np.maximum(v_ref, 1e-30) / bc2) + 1e-15)
        assert (np.abs(got_p[row, :n] - p_ref) <= 2 * ulp + 1e-6 * dp + prop).all(), row
        if not sgd:
            assert (np.abs(got_m[row, :n] - m_ref) <= m_tol + 1e-6 * np.abs(m_ref)).all(), row
            np.testing.assert_allclose(got_v[row, :n], v_ref, rtol=1e-6, atol=1e-15)


# ------------------------------------------------------------------------------ backward
EPS32 = 2.0 ** -24
MAG_FACTOR = 8.0   # fp32 sums / products, ex2.approx, T recovery


def _check_grads(got, ref, flagged, tag=None):
    """Per element |gpu - oracle| <= 1e-3 |g_ref| + 8 * 2^-24 * mag (SURVEY §8(c) contract item 5,
    with the rounding allowance scaled by the oracle's sum of absolute per-pixel terms carried
    through |chain Jacobian| -- orc_backward's `mag`), excluding Gaussians evaluated at
    band-flagged pixels.  Records the worst ratio |delta| / (2^-24 mag) per class."""
    keep = flagged == 0
    worst, fails = {}, []
    for c in CLASSES:
        a, b, mg = got[c][keep], ref[c][keep], ref["mag"][c][keep]
        tol = 1e-3 * np.abs(b) + MAG_FACTOR * EPS32 * mg
        d = np.abs(a - b)
        bad = d > tol
        excess = np.maximum(d - 1e-3 * np.abs(b), 0)
        worst[c] = float((excess / np.maximum(EPS32 * mg, 1e-38)).max(initial=0))
        if bad.sum():
            fails.append((c, int(bad.sum()), float(d[bad].max()), float(mg[bad][np.argmax(d[bad])])))
    _record(tag, dict(worst_excess_over_eps_mag=worst, excluded=int((~keep).sum()), gaussians=int(keep.size)))
    assert not fails, fails


def _record(tag, d):
    """Parity statistics for DESIGN.md (gpurun_out/parity_stats.jsonl when run on the GPU box)."""
    if tag is None:
        return
    import json
    import os
    out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")
    os.makedirs(out, exist_ok=True)
    with open(os.path.join(out, "parity_stats.jsonl"), "a") as f:
        f.write(json.dumps(dict(test=tag, **d)) + "\n")


def test_backward_parity_tiny():
    scene = make_scene("tiny")
    cams = make_cameras("tiny", 1)
    r, params, D = _renderer(scene, cams)
    r.forward(params, cams)
    H, W = cams[0].height, cams[0].width
    G = np.random.default_rng(1).normal(size=(1, 3, H, W)).astype(np.float32)
    grads = torch.zeros_like(params)
    gn = torch.zeros(scene.means.shape[0], device="cuda")
    r.backward(params, cams, torch.from_numpy(G).cuda(), grads, gn)
    got = unpack(grads, scene.means.shape[0], D)
    ref = orc.backward(scene, cams, G, "recipe", mag=True)
    _check_grads(got, ref, ref["flagged"], "backward_tiny")
    keep = ref["flagged"] == 0
    np.testing.assert_allclose(gn.cpu().numpy()[keep], ref["grad2d_norm"][keep], rtol=1e-3,
                               atol=1e-5 * ref["grad2d_norm"].max())


@pytest.mark.parametrize("cfg,views,level,D", [("tum", 1, 0, 3), ("tum", 1, 2, 3), ("euroc", 3, 1, 3),
                                                ("euroc", 6, 2, 3), ("euroc", 16, 2, 3), ("replica", 1, 0, 3)])
def test_backward_parity_sampled(cfg, views, level, D):
    """dL/dI masked to 4096 sampled pixels on both sides (SURVEY §8(d) 'Parity runs'), up to 16
    views per call (the EuRoC keyframe batch of one GPU)."""
    scene = make_scene(cfg)
    cams = [scaled_camera(c, level) for c in make_cameras(cfg, views)]
    r, params, D = _renderer(scene, cams)
    r.forward(params, cams)
    H, W = cams[0].height, cams[0].width
    pix = _sample_pixels(views, H, W, 4096, 3)
    gp = np.random.default_rng(2).normal(size=(pix.shape[0], 3)).astype(np.float32)
    G = np.zeros((views, 3, H, W), np.float32)
    G[pix[:, 0], :, pix[:, 1], pix[:, 2]] = gp
    grads = torch.zeros_like(params)
    r.backward(params, cams, torch.from_numpy(G).cuda(), grads)
    got = unpack(grads, scene.means.shape[0], D)
    ref = orc.backward(scene, cams, gp, "recipe", pixels=pix, mag=True)
    _check_grads(got, ref, ref["flagged"], f"backward_{cfg}_v{views}_l{level}")


def test_backward_accumulates_and_zero_upstream():
    scene = make_scene("tiny")
    cams = make_cameras("tiny", 1)
    r, params, D = _renderer(scene, cams)
    r.forward(params, cams)
    grads = torch.zeros_like(params)
    r.backward(params, cams, torch.zeros((1, 3, 48, 64), device="cuda"), grads)
    assert grads.abs().max().item() == 0
    G = torch.randn((1, 3, 48, 64), device="cuda")
    r.backward(params, cams, G, grads)
    one = grads.clone()
    r.backward(params, cams, G, grads)
    # the raster backward sums with fp32 atomics in no fixed order: allow reordering noise
    torch.testing.assert_close(grads, 2 * one, rtol=1e-5, atol=1e-5 * one.abs().max().item())


@pytest.mark.parametrize("cfg,n,D", [("tiny", None, 0), ("tum", 60000, 3)])
def test_fused_backward_adam_equals_separate(cfg, n, D):
    """gs_render_backward_adam == gs_render_backward into zeroed grads + gs_adam_step, up to the
    order of the raster backward's fp32 atomics (not deterministic).  That reordering moves a
    gradient by at most dg = 2e-5 max|g| (test_backward_accumulates_and_zero_upstream: 1e-5 per
    run); the per-element bound is Adam's sensitivity to it, from m' = b1 m + (1 - b1) g,
    v' = b2 v + (1 - b2) g^2, p' = p - lr m' / (sqrt(v') rs + eps):
      |dm| <= (1 - b1) dg,  |dv| <= (1 - b2)(2 |g| dg + dg^2),
      |dp| <= lr ((1 - b1) dg / Q + |m'| rs |dv| / (2 sqrt(v') Q^2)),  Q = sqrt(v') rs + eps,
    plus a few ulps of each result (SFU sqrt / division)."""
    scene = make_scene(cfg, n=n)
    cams = make_cameras(cfg, 1)
    H, W = cams[0].height, cams[0].width
    G = torch.from_numpy(np.random.default_rng(4).normal(size=(1, 3, H, W)).astype(np.float32)).cuda()
    out = []
    grads = None
    cfg_adam = AdamConfig(lr_means=1e-3)
    t0 = 4
    for fused in (False, True):
        r, params, D = _renderer(scene, cams)
        opt = Adam(params, scene.n, D, cfg_adam)
        opt.m.normal_(generator=torch.Generator("cuda").manual_seed(1))
        opt.v.uniform_(generator=torch.Generator("cuda").manual_seed(2))
        opt.t = t0
        p0 = params.clone()
        r.forward(params, cams)
        if fused:
            r.backward_adam(params, cams, G, opt)
        else:
            grads = torch.zeros_like(params)
            r.backward(params, cams, G, grads)
            g_sep = grads.clone()
            opt.step(grads, zero_grads=True)
        out.append((params.clone(), opt.m.clone(), opt.v.clone()))
    (p_s, m_s, v_s), (p_f, m_f, v_f) = out
    n_ = scene.n
    g = g_sep[:, :n_].double().abs()
    dg = 2e-5 * g.max().item()
    b1, b2, eps = cfg_adam.beta1, cfg_adam.beta2, cfg_adam.eps
    t = t0 + 1
    hp = cfg_adam.struct()
    row_lr = torch.tensor([hp.lr[0 if k < 3 else 1 if k < 7 else 2 if k < 10 else 3 if k == 10 else 4 if k < 14 else 5]
                           for k in range(p_s.shape[0])], dtype=torch.float64, device=g.device)[:, None]
    lr = row_lr / (1 - b1 ** t)
    rs = 1.0 / math.sqrt(1 - b2 ** t)
    m1, v1 = m_s[:, :n_].double(), v_s[:, :n_].double()
    dm = (1 - b1) * dg
    dv = (1 - b2) * (2 * g * dg + dg * dg)
    sq = v1.sqrt()
    Q = sq * rs + eps
    dp = lr * ((1 - b1) * dg / Q + m1.abs() * rs * dv / (2 * sq.clamp_min(1e-30) * Q * Q))
    ulp = 2.0 ** -22
    upd = (p_s[:, :n_].double() - p0[:, :n_].double()).abs()
    checks = (("m", m_f, m_s, dm + ulp * m1.abs()), ("v", v_f, v_s, dv + ulp * v1.abs()),
              ("p", p_f, p_s, 2 * dp + ulp * (p_s[:, :n_].double().abs() + upd)))
    for name, a, b, tol in checks:
        err = (a[:, :n_].double() - b[:, :n_].double()).abs()
        worst = (err / tol.clamp_min(1e-30)).max().item()
        assert worst <= 1.0, f"{name}: worst |fused - separate| / bound = {worst:.3g}"
    # the fused call changed the parameters: a second backward on that forward state is stale
    with pytest.raises(L.GsError) as e:
        r.backward(params, cams, G, torch.zeros_like(params))
    assert e.value.status == L.GS_ERR_STALE_STATE


def test_adam_step_rows_equals_full_step_on_its_rows():
    """gs_adam_step_rows (row-sharded optimiser) = gs_adam_step restricted to its rows,
    bit for bit, with the moments of those rows only; the other rows are untouched."""
    scene = make_scene("tum", n=5000)
    params = pack_params(scene)
    K, ld = params.shape
    gen = torch.Generator("cuda").manual_seed(3)
    grads = torch.randn(params.shape, device="cuda", generator=gen)
    full = Adam(params.clone(), scene.n, 3, AdamConfig(lr_means=1e-3))
    full.m.normal_(generator=gen)
    full.v.uniform_(generator=gen)
    m0, v0 = full.m.clone(), full.v.clone()
    full.t = 2
    full.step(grads.clone(), zero_grads=True)
    for r0, r1 in ((0, 11), (11, 14), (14, K), (5, 23)):
        p = params.clone()
        g = grads.clone()
        m, v = m0[r0:r1].clone(), v0[r0:r1].clone()
        ps = L.params_struct(p, scene.n, 3)
        L.gs_adam_step_rows(ps, g, m, v, full.hp, 3, r0, r1, True)
        torch.cuda.synchronize()
        assert torch.equal(p[r0:r1, :scene.n], full.params[r0:r1, :scene.n])
        assert torch.equal(m[:, :scene.n], full.m[r0:r1, :scene.n])
        assert torch.equal(v[:, :scene.n], full.v[r0:r1, :scene.n])
        assert torch.equal(p[:r0], params[:r0]) and torch.equal(p[r1:], params[r1:])
        assert (g[r0:r1, :scene.n] == 0).all() and torch.equal(g[r1:], grads[r1:])
    with pytest.raises(L.GsError):
        L.gs_adam_step_rows(L.params_struct(params, scene.n, 3), grads, m0, v0, full.hp, 1, 3, K + 1, False)


def test_graph_replay_matches_eager_steps():
    """A captured step (device-resident step counter) replayed gives the same trajectory as eager
    steps: 1 warm-up + 2 replays == 3 eager steps.  Run with the optimiser in SGD mode, where a
    step is -lr g (Adam's normalisation would turn the atomics' last-bit noise on ~0 gradients
    into +-lr moves), so the two trajectories must agree to fp32 summation-order rounding; the
    Adam counter is checked separately."""
    scene = make_scene("tum", n=40000)
    cams = make_cameras("tum", 1)
    r, params, _ = _renderer(scene, cams)
    gt = r.forward(params, cams)[0].clone()
    start = perturb(scene, 3)
    cfg = AdamConfig(sgd=True)
    a = MappingEngine(start, cams, gt, n_levels=2, adam=cfg)
    b = MappingEngine(start, cams, gt, n_levels=2, adam=cfg)
    for _ in range(3):
        a.build_pyramids()
        a.step()
    b.capture()
    b.replay()
    b.replay()
    torch.cuda.synchronize()
    assert int(b.adam.t_dev.item()) == 9 and a.adam.t == 9
    moved = (a.params - pack_params(start)).abs()
    diff = (b.params - a.params).abs()
    # per element: within 1e-3 of the element's own movement (+ fp32 resolution of the value)
    tol = 1e-3 * moved + 4 * torch.finfo(torch.float32).eps * a.params.abs() + 1e-9
    bad = diff > tol
    assert bad.float().mean().item() <= 1e-5, (int(bad.sum()), float(diff.max()))


def test_step_host_prefetch_matches_plain():
    """step_host with the next targets prefetched on a copy stream (double buffering) runs the
    same steps as plain step_host: per-level losses agree (up to atomic-order rounding), and
    switching the targets between calls takes effect on the right step."""
    scene = make_scene("tiny")
    cams = make_cameras("tiny", 1)
    r, params, _ = _renderer(scene, cams)
    gt_a = r.forward(params, cams)[0].clone()
    gt_b = torch.from_numpy(noise_image(48, 64, 9)[None]).cuda()
    start = perturb(scene, 5)
    seq = [gt_a, gt_b, gt_a, gt_b]
    host = [g.cpu().pin_memory() for g in seq]
    a = MappingEngine(start, cams, gt_a, n_levels=1)
    b = MappingEngine(start, cams, gt_a, n_levels=1)
    la, lb = [], []
    for k in range(4):
        out = torch.empty((2, 1)).pin_memory()
        a.step_host(host[k], out)
        torch.cuda.synchronize()
        la.append(out.clone())
    for k in range(4):
        out = torch.empty((2, 1)).pin_memory()
        b.step_host(host[k], out, host[k + 1] if k < 3 else None)
        torch.cuda.synchronize()
        lb.append(out.clone())
    for x, y in zip(la, lb):
        torch.testing.assert_close(x, y, rtol=1e-4, atol=1e-6)
    assert not torch.allclose(la[0], la[1])  # the targets really changed between steps


def test_step_pipelined_matches_step_host():
    """The two-graph pipelined end-to-end step (capture_pipelined / step_pipelined) runs the same
    steps as eager step_host on the same target sequence: its two warm-up steps (targets 0, 1)
    and then calls k = 0..3 (targets k % 2)."""
    scene = make_scene("tiny")
    cams = make_cameras("tiny", 1)
    r, params, _ = _renderer(scene, cams)
    gt_a = r.forward(params, cams)[0].clone()
    gt_b = torch.from_numpy(noise_image(48, 64, 9)[None]).cuda()
    start = perturb(scene, 5)
    host = [gt_a.cpu().pin_memory(), gt_b.cpu().pin_memory()]
    a = MappingEngine(start, cams, gt_a, n_levels=1)
    la = []
    for k in range(6):
        out = torch.empty((2, 1)).pin_memory()
        a.step_host(host[k % 2], out)
        torch.cuda.synchronize()
        la.append(out.clone())
    c = MappingEngine(start, cams, gt_a, n_levels=1)
    outs = [torch.empty((2, 1)).pin_memory() for _ in range(2)]
    c.capture_pipelined(host, outs)
    lc = []
    for k in range(4):
        o = c.step_pipelined()
        torch.cuda.synchronize()
        assert o.data_ptr() == outs[k % 2].data_ptr()
        lc.append(o.clone())
    for x, y in zip(la[2:], lc):
        torch.testing.assert_close(x, y, rtol=1e-3, atol=1e-6)
    assert not torch.allclose(lc[0], lc[1])  # the targets alternate between calls
    assert int(c.adam.t_dev.item()) == 6 * 2


# ------------------------------------------------------------------------------ mapping loop
def test_mapping_engine_reduces_loss():
    """A few Eq. 5 passes on the tiny config reduce the photometric loss (SPEC.md:460 trend)."""
    scene = make_scene("tiny")
    cams = make_cameras("tiny", 1)
    r, params, _ = _renderer(scene, cams)
    gt = r.forward(params, cams)[0].clone()
    eng = MappingEngine(perturb(scene, 9), cams, gt, n_levels=1, adam=AdamConfig(lr_means=1e-3))
    first = torch.stack(eng.step()).cpu().numpy()
    for _ in range(60):
        last = torch.stack(eng.step()).cpu().numpy()
    eng.check()
    assert last[-1] < 0.7 * first[-1], (first, last)


def test_pipelined_step_raises_on_capacity_overflow():
    """The end-to-end pipelined step reads each level's overflow flag back with its losses
    (gs_status_async) and raises once a step rendered into an overflowing workspace (the level's
    pairs exceed its capacity: nothing was binned)."""
    scene = make_scene("tum", n=20000)   # up to 1200 tiles per Gaussian: huge footprints overflow
    cams = make_cameras("tum", 1)
    r, params, _ = _renderer(scene, cams)
    gt = r.forward(params, cams)[0].clone()
    eng = MappingEngine(perturb(scene, 3), cams, gt, n_levels=1)
    gts = [eng.gt0.cpu().pin_memory() for _ in range(2)]
    outs = [torch.empty((2, 1), dtype=torch.float32).pin_memory() for _ in range(2)]
    eng.capture_pipelined(gts, outs)
    for _ in range(3):
        eng.step_pipelined()
    eng.pipeline_join()
    torch.cuda.synchronize()
    eng.pipeline_check()  # no overflow: nothing raised
    # make every Gaussian huge: far more pairs than the calibrated capacity
    with torch.no_grad():
        eng.params[7:10, :eng.n] += 3.0
    with pytest.raises(RuntimeError, match="capacity"):
        for _ in range(4):
            eng.step_pipelined()
        eng.pipeline_join()
        torch.cuda.synchronize()
        eng.pipeline_check()


def test_workspace_release_forgets_forward_state():
    """gs_workspace_release erases the forward-state token: a backward on the released workspace
    is StaleRenderState (a new workspace at the same address cannot inherit the old token)."""
    scene = make_scene("tiny")
    cams = make_cameras("tiny", 1)
    r, params, D = _renderer(scene, cams)
    r.forward(params, cams)
    L.gs_workspace_release(r.ws.buf)
    grads = torch.zeros_like(params)
    with pytest.raises(L.GsError) as e:
        r.backward(params, cams, torch.zeros((1, 3, 48, 64), device="cuda"), grads)
    assert e.value.status == L.GS_ERR_STALE_STATE
