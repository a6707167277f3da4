"""Pins of the oracle's analytic backward: central finite
differences in fp64 (h = 1e-6) on tiny scenes kept away from every threshold, closed-form
zero cases (zero upstream, opaque occluder, clamped colour) and linearity over views."""
import math

import numpy as np
import pytest

import oracle.oracle as orc
from synth import Scene
from tests.helpers import camera, logit, random_small_scene, scene_of

CLASSES = ["means", "quats", "log_scales", "opacity_logits", "sh"]


def _margin_ok(scene, cams, margin=1e-4):
    """Selection helper (not an expected value): every (pixel, Gaussian) pair is >= margin away
    from the cutoff / alpha-skip thresholds and no pixel reaches the stop rule."""
    for cam in cams:
        pr = orc.project(scene, cam, "fp64")
        ys, xs = np.mgrid[0:cam.height, 0:cam.width]
        T = np.ones_like(xs, dtype=np.float64)
        for i in np.nonzero(pr["radius"] > 0)[0]:
            u, v = pr["mean2d"][i]
            A, B, Cc = pr["conic"][i]
            dx, dy = xs - u, ys - v
            p = -0.5 * (A * dx * dx + Cc * dy * dy) - B * dx * dy
            a = pr["sigma"][i] * np.exp(p)
            live = p >= -4.5
            if (np.abs(p + 4.5) < margin).any() or (np.abs(255 * a[live] - 1) < 255 * margin * 1e-2).any():
                return False
            if (a > 0.99).any():
                return False
            T *= np.where(live & (a >= 1 / 255), 1 - a, 1.0)
        if T.min() < 2e-4:
            return False
    return True


def _pick(n, D, seed0, margin=1e-4, **kw):
    for seed in range(seed0, seed0 + 400):
        s, cam = random_small_scene(n, seed, D=D, **kw)
        s.opacity_logits[:] = np.clip(s.opacity_logits, -3, 0)  # sigma <= 0.5: no stop rule
        if _margin_ok(s, [cam], margin):
            return s, cam
    raise RuntimeError("no FD-safe scene")


def _L(scene, cams, G):
    r = orc.render(scene, cams, "fp64")
    return float((r["rgb"] * G).sum())


def _fd(scene, cams, G, cls, idx, h=1e-6):
    arr = getattr(scene, cls)
    old = arr[idx]
    # perturb in float32 storage: use exactly representable steps around the stored value
    arr[idx] = np.float32(old + h)
    hp = float(np.float64(arr[idx]) - np.float64(old))
    Lp = _L(scene, cams, G)
    arr[idx] = np.float32(old - h)
    hm = float(np.float64(old) - np.float64(arr[idx]))
    Lm = _L(scene, cams, G)
    arr[idx] = old
    return (Lp - Lm) / (hp + hm)


def test_zero_upstream_gives_zero_gradients():
    s, cam = random_small_scene(40, 0, D=2)
    g = orc.backward(s, [cam], np.zeros((1, 3, cam.height, cam.width)), "recipe")
    for k in CLASSES + ["grad2d_norm"]:
        assert (g[k] == 0).all()


@pytest.mark.parametrize("D", [0, 3])
def test_fd_single_gaussian_all_params(D):
    """single-Gaussian scene, every gradient vs central finite differences with
    h ~ 2e-6 (the effective step is taken from the float32-stored perturbed values)."""
    s, cam = _pick(1, D, 100, scale=0.08, spread=0.3)
    rng = np.random.default_rng(5)
    G = rng.normal(size=(1, 3, cam.height, cam.width))
    g = orc.backward(s, [cam], G, "fp64")
    worst = 0.0
    for cls in CLASSES:
        arr = getattr(s, cls)
        for idx in np.ndindex(arr.shape):
            fd = _fd(s, [cam], G, cls, idx, h=2e-6 * max(1.0, abs(float(arr[idx]))))
            an = g[cls][idx]
            scale = max(abs(fd), abs(an), 1e-3 * np.abs(g[cls]).max(), 1e-9)
            worst = max(worst, abs(fd - an) / scale)
    assert worst < 1e-6, worst


def test_directional_fd_50_gaussians():
    """50 random Gaussians, random dL/dI: <g, d> vs (L(t+hd) - L(t-hd)) / 2h."""
    s, cam = _pick(50, 3, 300, scale=0.03, margin=1e-3)
    rng = np.random.default_rng(7)
    G = rng.normal(size=(1, 3, cam.height, cam.width))
    g = orc.backward(s, [cam], G, "fp64")
    for trial in range(3):
        dirs = {c: rng.normal(size=getattr(s, c).shape) for c in CLASSES}
        h = 1e-5
        sp, sm = s.copy(), s.copy()
        for c in CLASSES:
            setattr(sp, c, (getattr(s, c).astype(np.float64) + h * dirs[c]).astype(np.float32))
            setattr(sm, c, (getattr(s, c).astype(np.float64) - h * dirs[c]).astype(np.float32))
        # the effective (float32-rounded) displacement is what the FD measures; second-order
        # terms do not cancel for an asymmetric displacement, hence the 1e-4 tolerance
        dp = {c: getattr(sp, c).astype(np.float64) - getattr(s, c).astype(np.float64) for c in CLASSES}
        dm = {c: getattr(s, c).astype(np.float64) - getattr(sm, c).astype(np.float64) for c in CLASSES}
        L0 = _L(s, [cam], G)
        fd_p, fd_m = _L(sp, [cam], G) - L0, L0 - _L(sm, [cam], G)
        an_p = sum(float((g[c] * dp[c]).sum()) for c in CLASSES)
        an_m = sum(float((g[c] * dm[c]).sum()) for c in CLASSES)
        assert abs(fd_p + fd_m - an_p - an_m) <= 1e-4 * abs(an_p + an_m), (trial, fd_p, an_p, fd_m, an_m)


def test_loss_gradient_end_to_end():
    """Eq. 4 composed with Eq. 3: directional FD of sum_v L_v through render, loss and backward."""
    s, cam = _pick(12, 1, 500, scale=0.05, margin=1e-3)
    gts = [np.random.default_rng(9).uniform(0.1, 0.9, size=(3, cam.height, cam.width))]
    g, _, _ = orc.total_grad(s, [cam], gts, 0.2, "fp64")
    rng = np.random.default_rng(11)
    dirs = {c: rng.normal(size=getattr(s, c).shape) for c in CLASSES}
    h = 1e-5
    sp, sm = s.copy(), s.copy()
    for c in CLASSES:
        setattr(sp, c, (getattr(s, c).astype(np.float64) + h * dirs[c]).astype(np.float32))
        setattr(sm, c, (getattr(s, c).astype(np.float64) - h * dirs[c]).astype(np.float32))
    dd = {c: (getattr(sp, c).astype(np.float64) - getattr(sm, c).astype(np.float64)) for c in CLASSES}
    fd = orc.total_loss(sp, [cam], gts) - orc.total_loss(sm, [cam], gts)
    an = sum(float((g[c] * dd[c]).sum()) for c in CLASSES)
    assert abs(fd - an) <= 1e-3 * abs(an), (fd, an)


def test_grad2d_norm_is_screen_gradient():
    """grad2d_norm = ||dL/dmean2d||: for one Gaussian, shifting cx/cy moves only the mean2d
    (u = fx x/z + cx), so dL/du = dL/dcx by central FD."""
    s, cam = _pick(1, 0, 700, scale=0.08, spread=0.2)
    G = np.random.default_rng(1).normal(size=(1, 3, cam.height, cam.width))
    g = orc.backward(s, [cam], G, "fp64")
    h = 2e-5
    fds = []
    for attr in ("cx", "cy"):
        cp, cm = camera(**_camkw(cam)), camera(**_camkw(cam))
        c0 = np.float32(getattr(cam, attr))
        setattr(cp, attr, float(np.float32(c0 + h)))
        setattr(cm, attr, float(np.float32(c0 - h)))
        fds.append((_L(s, [cp], G) - _L(s, [cm], G)) / (getattr(cp, attr) - getattr(cm, attr)))
    assert g["grad2d_norm"][0] == pytest.approx(math.hypot(*fds), rel=1e-6)


def _camkw(cam):
    return dict(fx=cam.fx, fy=cam.fy, cx=cam.cx, cy=cam.cy, width=cam.width, height=cam.height, R=cam.R,
                t=cam.t, lim=cam.lim_x, znear=cam.znear)


def test_opaque_occluder_blocks_gradient():
    """Gaussians behind a stopped pixel get exactly zero colour and zero gradient (SURVEY
    §8(c) 'occluder cutoff'): two wide alpha~0.98 layers stop every pixel of a small splat behind."""
    n_front = 3
    means = [[0, 0, 2.0 + 0.01 * i] for i in range(n_front)] + [[0, 0, 3.0]]
    ls = [[math.log(0.2), math.log(0.15), math.log(0.1)]] * n_front + [[math.log(0.005)] * 3]
    s = scene_of(means, log_scales=ls, quats=[[0.9, 0.1, -0.3, 0.2]] * 4, opac=[logit(0.985)] * n_front + [0.0], D=1,
                 sh=np.random.default_rng(0).normal(size=(4, 4, 3)).astype(np.float32))
    cam = camera(width=96, height=64, cx=48, cy=32, fx=300, fy=300)
    G = np.random.default_rng(2).normal(size=(1, 3, cam.height, cam.width))
    g = orc.backward(s, [cam], G, "recipe")
    for c in CLASSES:
        assert (g[c][3] == 0).all(), c
        assert np.abs(g[c][:2]).sum() > 0


def test_clamped_channel_has_zero_sh_gradient():
    sh = np.zeros((1, 4, 3), np.float32)
    sh[0, 0] = [-5.0, 1.0, 0.5]  # red clamps to 0
    sh[0, 1:] = 0.1
    s = scene_of([[0.05, -0.02, 1.5]], log_scales=[[math.log(0.05)] * 3], opac=[0.0], sh=sh, D=1)
    cam = camera(width=64, height=48, cx=32, cy=24, fx=60, fy=60)
    G = np.ones((1, 3, cam.height, cam.width))
    g = orc.backward(s, [cam], G, "fp64")
    assert (g["sh"][0, :, 0] == 0).all() and (np.abs(g["sh"][0, :, 1]) > 0).all()


def test_views_sum_linearity():
    """Gradient of a batch = sum of per-view gradients."""
    s, cam = random_small_scene(60, 3, D=1)
    cam2 = camera(**{**_camkw(cam), "t": np.array([0.05, -0.03, 0.1], np.float32)})
    rng = np.random.default_rng(4)
    G = rng.normal(size=(2, 3, cam.height, cam.width))
    both = orc.backward(s, [cam, cam2], G, "recipe")
    a = orc.backward(s, [cam], G[:1], "recipe")
    b = orc.backward(s, [cam2], G[1:], "recipe")
    for c in CLASSES + ["grad2d_norm"]:
        np.testing.assert_allclose(both[c], a[c] + b[c], rtol=1e-12, atol=1e-15)
