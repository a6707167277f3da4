"""Pins of the oracle's clamp branches and of its rounding-allowance output.

* R15: the EWA Jacobian of a mean whose tangent x/z (or y/z) lies
  beyond the clamp +-lim is J evaluated at the clamped tangent, and the derivative of the
  clamped axis with respect to that coordinate is zero -- pinned by an independent numerical
  Jacobian of the pinhole projection at the clamped point (forward) and by fp64 central finite
  differences of the rendered image through the clamped branch (backward).
* R7: alpha = min(0.99, sigma e^power) has zero derivative on the clamped
  branch -- closed form at the Gaussian's centre pixel (colour gradient g 0.99 T Y0, zero
  opacity / position / shape gradient) and finite differences one step either side of the clamp.
* The fp32 scale recipe e = (float)exp((double)s) is the
  correctly rounded fp32 exp -- pinned against 60-digit mpmath, not against another rounding of
  a double exp.
* orc_backward's `mag` (sum of absolute per-pixel terms, each weighted by its pixel's
  transmittance conditioning, through the absolute chain): equals the brute-force sum over
  pixels of |per-pixel gradient| / T_final (= kappa for one layer) where every per-pixel term has
  one sign (opacity, SH DC of a lone Gaussian), bounds |g| everywhere (triangle inequality).
"""
import math

import mpmath
import numpy as np
import pytest

import oracle.oracle as orc
from tests.helpers import camera, logit, scene_of

CLASSES = ["means", "quats", "log_scales", "opacity_logits", "sh"]
Y0 = 0.28209479177387814  # sqrt(1 / (4 pi))


def _L(scene, cams, G):
    return float((orc.render(scene, cams, "fp64")["rgb"] * G).sum())


def _fd(scene, cams, G, cls, idx, h):
    arr = getattr(scene, cls)
    old = arr[idx]
    arr[idx] = np.float32(old + h)
    hp = float(np.float64(arr[idx]) - np.float64(old))
    Lp = _L(scene, cams, G)
    arr[idx] = np.float32(old - h)
    hm = float(np.float64(old) - np.float64(arr[idx]))
    Lm = _L(scene, cams, G)
    arr[idx] = old
    return (Lp - Lm) / (hp + hm)


# ------------------------------------------------------------------ R15: tan clamp
def _proj_jacobian(p, fx, fy, h=1e-6):
    """Numerical Jacobian of (fx x/z, fy y/z) at p (independent of the oracle)."""
    J = np.zeros((2, 3))
    for k in range(3):
        a, b = p.copy(), p.copy()
        a[k] += h
        b[k] -= h
        J[:, k] = (np.array([fx * a[0] / a[2], fy * a[1] / a[2]]) - np.array([fx * b[0] / b[2], fy * b[1] / b[2]])) / (2 * h)
    return J


def _rotation(q):
    w, x, y, z = np.asarray(q, np.float64) / np.linalg.norm(q)
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])


@pytest.mark.parametrize("axis", ["x", "y", "both"])
def test_cov2d_beyond_tan_clamp_is_ewa_at_clamped_point(axis):
    """Sigma2 of a mean beyond the clamp = J(p') W Sigma3 W^T J(p')^T + 0.3 I with p' the point of
    the same depth at the clamped tangent (txc z, tyc z, z), J(p') a numerical Jacobian."""
    rng = np.random.default_rng(3)
    cam = camera(fx=60, fy=60, cx=31.5, cy=23.5, width=64, height=48, lim=1.3 * 32 / 60)
    cam.lim_y = float(np.float32(1.3 * 24 / 60))
    cam.lim_x = float(np.float32(cam.lim_x))
    hits = 0
    for _ in range(30):
        z = rng.uniform(1.0, 3.0)
        tx, ty = rng.uniform(-0.3, 0.3), rng.uniform(-0.3, 0.3)
        if axis in ("x", "both"):
            tx = rng.choice([-1, 1]) * cam.lim_x * rng.uniform(1.05, 1.8)
        if axis in ("y", "both"):
            ty = rng.choice([-1, 1]) * cam.lim_y * rng.uniform(1.05, 1.8)
        P = np.array([tx * z, ty * z, z], np.float32)
        q = rng.normal(size=4).astype(np.float32)
        ls = rng.normal(-2.5, 0.4, size=3).astype(np.float32)
        res = orc.debug_cov(P, q, ls, cam)
        assert res is not None
        _, S2 = res
        pc = P.astype(np.float64)
        txc = np.clip(pc[0] / pc[2], -cam.lim_x, cam.lim_x)
        tyc = np.clip(pc[1] / pc[2], -cam.lim_y, cam.lim_y)
        pclamp = np.array([txc * pc[2], tyc * pc[2], pc[2]])
        J = _proj_jacobian(pclamp, cam.fx, cam.fy)
        Rm = _rotation(q)
        S3 = Rm @ np.diag(np.exp(2 * ls.astype(np.float64))) @ Rm.T
        want = J @ S3 @ J.T + 0.3 * np.eye(2)   # W = I
        np.testing.assert_allclose(S2, [want[0, 0], want[0, 1], want[1, 1]], rtol=2e-6, atol=1e-7 * np.abs(want).max())
        # and NOT the unclamped Jacobian (the branch is really taken)
        Ju = _proj_jacobian(pc, cam.fx, cam.fy)
        wu = Ju @ S3 @ Ju.T + 0.3 * np.eye(2)
        hits += not np.allclose(S2, [wu[0, 0], wu[0, 1], wu[1, 1]], rtol=1e-4)
    assert hits >= 25


def test_recipe_conic_beyond_clamp_agrees_with_fp64():
    rng = np.random.default_rng(8)
    cam = camera(fx=60, fy=60, cx=31.5, cy=23.5, width=64, height=48, lim=float(np.float32(1.3 * 32 / 60)))
    n = 200
    z = rng.uniform(1.0, 3.0, n)
    tx = rng.choice([-1, 1], n) * cam.lim_x * rng.uniform(1.05, 1.5, n)
    ty = rng.uniform(-0.9, 0.9, n) * cam.lim_y * 1.3
    means = np.stack([tx * z, ty * z, z], 1)
    s = scene_of(means, log_scales=np.log(rng.uniform(0.1, 0.3, (n, 3))), quats=rng.normal(size=(n, 4)))
    a, b = orc.project(s, cam, "fp64"), orc.project(s, cam, "recipe")
    vis = (a["radius"] > 0) & (b["radius"] > 0)
    assert vis.sum() > 50
    np.testing.assert_allclose(a["conic"][vis], b["conic"][vis], rtol=1e-4, atol=1e-6 * np.abs(a["conic"][vis]).max())


def _clamped_scene(axis, seed):
    """One Gaussian beyond the tan clamp whose 3-sigma footprint still covers part of the image;
    FD-safe: no pixel within 1e-4 of the cutoff / skip thresholds, sigma <= 0.5 (no stop, no
    alpha clamp)."""
    rng = np.random.default_rng(seed)
    lim = float(np.float32(1.3 * 32 / 60))
    cam = camera(fx=60, fy=60, cx=31.5, cy=23.5, width=64, height=48, lim=lim)
    cam.lim_y = float(np.float32(1.3 * 24 / 60))
    for _ in range(500):
        z = rng.uniform(1.5, 2.5)
        tx = rng.uniform(-0.2, 0.2) if axis == "y" else lim * rng.uniform(1.08, 1.25)
        ty = rng.uniform(-0.2, 0.2) if axis == "x" else cam.lim_y * rng.uniform(1.08, 1.25)
        s = scene_of([[tx * z, ty * z, z]], log_scales=np.log(rng.uniform(0.25, 0.4, (1, 3))),
                     quats=rng.normal(size=(1, 4)), opac=[rng.uniform(-2.5, 0.0)], D=1,
                     sh=rng.normal(0, 0.3, (1, 4, 3)))
        s.sh[:, 0] = rng.uniform(0.5, 1.5, (1, 3))
        pr = orc.project(s, cam, "fp64")
        if pr["radius"][0] <= 0:
            continue
        u, v = pr["mean2d"][0]
        A, B, Cc = pr["conic"][0]
        ys, xs = np.mgrid[0:48, 0:64]
        dx, dy = xs - u, ys - v
        p = -0.5 * (A * dx * dx + Cc * dy * dy) - B * dx * dy
        a = pr["sigma"][0] * np.exp(p)
        live = p >= -4.5
        if live.sum() < 30 or (np.abs(p + 4.5) < 1e-4).any() or (np.abs(255 * a[live] - 1) < 1e-3).any():
            continue
        return s, cam
    raise RuntimeError("no FD-safe clamped scene")


@pytest.mark.parametrize("axis", ["x", "y", "both"])
def test_fd_through_tan_clamp(axis):
    """Central FD (fp64) of every parameter of a Gaussian beyond the clamp: the analytic backward's
    clamped branch (zero d/dx of the clamped tangent, the clamped value's own z-derivative)."""
    s, cam = _clamped_scene(axis, {"x": 1, "y": 2, "both": 3}[axis])
    pr = orc.project(s, cam, "fp64")
    u, v = pr["mean2d"][0]
    assert (axis == "y") or not (0 <= u <= 63)        # mean off-image on a clamped axis
    G = np.random.default_rng(5).normal(size=(1, 3, cam.height, cam.width))
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


# ------------------------------------------------------------------ R7: alpha clamp
def _centre_scene(sigma):
    """Isotropic Gaussian at p_c = (0, 0, 2) -> its mean projects exactly onto pixel (320, 240)
    (P3 of SURVEY §8(c)); power = 0 there, so alpha = min(0.99, sigma)."""
    cam = camera()
    s = scene_of([[0, 0, 2]], log_scales=[[math.log(0.01)] * 3], opac=[logit(sigma)], D=0,
                 sh=[[[0.5, 1.0, 1.5]]])
    G = np.zeros((1, 3, 480, 640))
    G[0, :, 240, 320] = [0.3, -0.7, 1.1]
    return s, cam, G


def test_alpha_clamp_closed_form_at_centre():
    """sigma = 0.997: alpha = 0.99 at the centre pixel (clamped).  With dL/dI only there:
    dL/dSH_dc = g * 0.99 * T(=1) * Y0 per channel, and every opacity / position / shape gradient
    is exactly 0 (no derivative through the clamp)."""
    s, cam, G = _centre_scene(0.997)
    r = orc.render(s, [cam], "fp64")
    c = Y0 * np.array([0.5, 1.0, 1.5]) + 0.5
    np.testing.assert_allclose(r["rgb"][0, :, 240, 320], 0.99 * c, rtol=1e-12)
    assert abs(r["T"][0, 240, 320] - 0.01) < 1e-12
    g = orc.backward(s, [cam], G, "fp64")
    np.testing.assert_allclose(g["sh"][0, 0], np.array([0.3, -0.7, 1.1]) * 0.99 * Y0, rtol=1e-12)
    for cls in ("means", "quats", "log_scales", "opacity_logits"):
        assert (g[cls] == 0).all(), cls


@pytest.mark.parametrize("sigma,clamped", [(0.985, False), (0.9899, False), (0.9901, True), (0.995, True)])
def test_alpha_clamp_fd_either_side(sigma, clamped):
    """One step either side of 0.99: central FD of the logit and the means matches the analytic
    gradient -- non-zero below the clamp, zero above it (the FD step keeps alpha on its side)."""
    s, cam, G = _centre_scene(sigma)
    g = orc.backward(s, [cam], G, "fp64")
    fd = _fd(s, [cam], G, "opacity_logits", (0,), h=1e-6)
    an = g["opacity_logits"][0]
    if clamped:
        assert an == 0.0 and abs(fd) < 1e-9
    else:
        # closed form: dL/dlogit = sigma (1 - sigma) * sum_ch g_ch (c_ch - 0) * T (bg = 0, e^0 = 1)
        c = Y0 * np.array([0.5, 1.0, 1.5]) + 0.5
        want = sigma * (1 - sigma) * float(np.dot([0.3, -0.7, 1.1], c))
        np.testing.assert_allclose(an, want, rtol=1e-6)
        np.testing.assert_allclose(fd, an, rtol=1e-5)
    for k in range(3):  # means: zero at the centre pixel either way (d power/d mean = 0 at dx=dy=0)
        assert abs(g["means"][0, k]) < 1e-12


# ------------------------------------------------------------------ fp32 scale recipe
def _correctly_rounded_exp_f32(s: float) -> np.float32:
    mpmath.mp.dps = 60
    e = mpmath.exp(mpmath.mpf(float(s)))
    c = np.float32(float(e))
    lo, hi = np.nextafter(c, np.float32(-np.inf)), np.nextafter(c, np.float32(np.inf))
    best = min((c, lo, hi), key=lambda f: abs(mpmath.mpf(float(f)) - e))
    return np.float32(best)


def test_exp_scale_recipe_is_correctly_rounded():
    """(float)exp((double)s) is the correctly rounded fp32 exp of s: checked against a 60-digit
    mpmath exp (nearest fp32 chosen by exact distance) on random log-scales of the data's range
    and on every s where the long-double exp lies closest to an fp32 rounding midpoint."""
    rng = np.random.default_rng(0)
    s_rand = rng.uniform(-12, 3, 3000).astype(np.float32)
    dense = np.linspace(-12, 3, 400001).astype(np.float32)
    e_ld = np.exp(dense.astype(np.longdouble))
    f = e_ld.astype(np.float32)
    nxt = np.nextafter(f, np.float32(np.inf)).astype(np.longdouble)
    prv = np.nextafter(f, np.float32(-np.inf)).astype(np.longdouble)
    mid_dist = np.minimum(np.abs(e_ld - (f.astype(np.longdouble) + nxt) / 2),
                          np.abs(e_ld - (f.astype(np.longdouble) + prv) / 2)) / e_ld
    hard = dense[np.argsort(mid_dist)[:300]]   # the cases a double-rounding error would hit first
    s = np.concatenate([s_rand, hard])
    got = orc.exp_scale_f32(s)
    want = np.array([_correctly_rounded_exp_f32(x) for x in s], np.float32)
    assert np.array_equal(got, want), np.nonzero(got != want)[0][:10]


# ------------------------------------------------------------------ rounding allowance (mag)
def test_mag_equals_bruteforce_for_single_signed_terms_and_bounds_everything():
    rng = np.random.default_rng(4)
    s = scene_of([[0.02, -0.01, 2.0]], log_scales=[[math.log(0.006), math.log(0.009), math.log(0.004)]],
                 quats=[[0.9, 0.2, -0.3, 0.1]], opac=[logit(0.6)], D=0, sh=[[[0.8, 0.4, 1.2]]])
    cam = camera()
    pr = orc.project(s, cam, "fp64")
    u, v = pr["mean2d"][0]
    r = pr["radius"][0]
    pix = np.array([[0, y, x] for y in range(int(v) - r, int(v) + r + 1) for x in range(int(u) - r, int(u) + r + 1)],
                   np.int32)
    G = rng.uniform(0.1, 1.0, size=(pix.shape[0], 3))   # one sign: every per-pixel term of one sign
    g = orc.backward(s, [cam], G, "fp64", pixels=pix, mag=True)
    # one layer per pixel: the transmittance conditioning kappa = 1 + alpha/(1 - alpha) = 1/T_final
    Tf = orc.render(s, [cam], "fp64", pixels=pix)["T"]
    per = {c: np.zeros_like(g[c]) for c in CLASSES}
    for q in range(pix.shape[0]):
        gq = orc.backward(s, [cam], G[q:q + 1], "fp64", pixels=pix[q:q + 1])
        for c in CLASSES:
            per[c] += np.abs(gq[c]) / Tf[q]
    assert per["opacity_logits"][0] > 0
    np.testing.assert_allclose(g["mag"]["opacity_logits"], per["opacity_logits"], rtol=1e-12)
    np.testing.assert_allclose(g["mag"]["sh"], per["sh"], rtol=1e-12)
    for c in CLASSES:   # sum_p |g_p| <= mag, |g| <= mag
        assert (per[c] <= g["mag"][c] * (1 + 1e-12) + 1e-300).all(), c
        assert (np.abs(g[c]) <= g["mag"][c] * (1 + 1e-12) + 1e-300).all(), c
    # mixed-sign upstream: cancellation makes |g| < mag
    G2 = rng.normal(size=G.shape)
    g2 = orc.backward(s, [cam], G2, "fp64", pixels=pix, mag=True)
    assert g2["mag"]["sh"][0, 0, 0] > 2 * abs(g2["sh"][0, 0, 0])
