"""Pins of the oracle's SH colour and per-pixel compositing of Eq. 3
 against closed forms and invariants."""
import math

import numpy as np
import pytest

import oracle.oracle as orc
from synth import make_cameras, make_scene
from tests.helpers import camera, golden, logit, scene_of


def test_sh_orthonormal_on_sphere():
    """Real SH basis to degree 3 is orthonormal: int Y_l Y_m dOmega = delta_lm (textbook
    normalisation of the constants SURVEY R6 names).  Gauss-Legendre x uniform-phi quadrature
    is exact for these polynomials."""
    xg, wg = np.polynomial.legendre.leggauss(12)
    nphi = 24
    phi = 2 * math.pi * np.arange(nphi) / nphi
    ct, ph = np.meshgrid(xg, phi, indexing="ij")
    st = np.sqrt(1 - ct ** 2)
    dirs = np.stack([st * np.cos(ph), st * np.sin(ph), ct], -1).reshape(-1, 3)
    w = (wg[:, None] * np.full(nphi, 2 * math.pi / nphi)[None, :]).reshape(-1)
    Y, _ = orc.sh_basis(3, dirs)
    G = (Y * w[:, None]).T @ Y
    np.testing.assert_allclose(G, np.eye(16), atol=1e-12)


def test_sh_spec_examples():
    g = golden()["sh"]
    Y, _ = orc.sh_basis(3, np.array([[0, 0, 1.0], [0, 0, -1.0], [0.6, 0, 0.8]]))
    assert Y[0, 0] == pytest.approx(g["Y00"], abs=1e-8)
    assert Y[2, 0] == pytest.approx(g["Y00"], abs=1e-8)  # band 0 isotropic
    # band-1 z coefficient: c(+z) - c(-z) = 2 * 0.48860251 * c1
    assert Y[0, 2] - Y[1, 2] == pytest.approx(2 * g["band1_z_difference_factor"], abs=1e-8)


def test_sh_gradient_matches_fd():
    rng = np.random.default_rng(3)
    d = rng.normal(size=(20, 3))
    _, dY = orc.sh_basis(3, d)
    h = 1e-6
    for k in range(3):
        e = np.zeros(3)
        e[k] = h
        fd = (orc.sh_basis(3, d + e)[0] - orc.sh_basis(3, d - e)[0]) / (2 * h)
        np.testing.assert_allclose(dY[:, :, k], fd, atol=1e-7)


@pytest.mark.parametrize("mode", ["fp64", "recipe"])
def test_sh_degree0_colour(mode):
    """D = 0: c = 0.28209479 c0 + 0.5 for every direction, clamped at 0."""
    c0 = np.array([[0.3, -0.2, -3.0]], np.float32)
    s = scene_of([[0.2, 0.1, 2], [-0.5, 0.3, 3]], sh=np.stack([c0, c0]), D=0)
    out = orc.project(s, camera(), mode)
    want = np.maximum(0.0, 0.28209479177 * c0[0].astype(np.float64) + 0.5)
    np.testing.assert_allclose(out["rgb"], np.stack([want, want]), atol=1e-9)


# ----------------------------------------------------------------------------- compositing
def _px(cam, pts):
    return np.array([[0, y, x] for (x, y) in pts], np.int32)


@pytest.mark.parametrize("mode", ["fp64", "recipe"])
def test_empty_scene(mode):
    cam = camera(width=32, height=24, cx=16, cy=12)
    s = scene_of(np.zeros((0, 3)))
    r = orc.render(s, [cam], mode)
    assert (r["rgb"] == 0).all() and (r["T"] == 1).all() and (r["ncomp"] == 0).all()


@pytest.mark.parametrize("mode", ["fp64", "recipe"])
def test_p4_single_splat_alpha(mode):
    """alpha at pixels of the P3 Gaussian with sigma = 0.5; Mahalanobis^2 > 9 cut (R9)."""
    g = golden()["P4_alpha"]
    cam = camera()
    sh = np.zeros((1, 1, 3), np.float32)
    sh[0, 0] = [1.0, 0.5, -0.5]
    s = scene_of([[0, 0, 2]], log_scales=[[math.log(0.01)] * 3], opac=[0.0], sh=sh)
    c = orc.project(s, cam, mode)["rgb"][0]
    r = orc.render(s, [cam], mode, pixels=_px(cam, [p["xy"] for p in g["pixels"]]))
    for k, p in enumerate(g["pixels"]):
        if p["inside"]:
            alpha = 1 - r["T"][k]
            assert alpha == pytest.approx(p["alpha"], rel=2e-5 if p["alpha"] < 0.01 else 2e-6)
            np.testing.assert_allclose(r["rgb"][k], alpha * c, rtol=1e-9)
            assert r["ncomp"][k] == 1 and r["last"][k] == 0
        else:
            assert r["T"][k] == 1.0 and r["ncomp"][k] == 0 and (r["rgb"][k] == 0).all()


def _stack_scene(alphas, colours_dc, depth0=2.0):
    """Gaussians centred on pixel (320, 240), peak alpha = sigma (power 0), front to back."""
    n = len(alphas)
    sh = np.zeros((n, 1, 3), np.float32)
    for i, c in enumerate(colours_dc):
        sh[i, 0] = c
    return scene_of([[0, 0, depth0 + 0.1 * i] for i in range(n)], log_scales=[[math.log(0.01)] * 3] * n,
                    opac=[logit(a) for a in alphas], sh=sh)


@pytest.mark.parametrize("mode", ["fp64", "recipe"])
def test_two_layers_white_over_black(mode):
    white = 0.5 / 0.28209479177387814  # c = 1
    s = _stack_scene([0.5, 0.5], [[white] * 3, [-10.0] * 3])  # back colour clamps to 0
    r = orc.render(s, [camera()], mode, pixels=_px(None, [(320, 240)]))
    np.testing.assert_allclose(r["rgb"][0], [golden()["compositing"]["two_layers_white_over_black_center"]] * 3,
                               atol=1e-6)
    assert r["T"][0] == pytest.approx(0.25, abs=1e-6)


@pytest.mark.parametrize("mode", ["fp64", "recipe"])
def test_k_layers_closed_form(mode):
    a, K = 0.3, 6
    s = _stack_scene([a] * K, [[1.0, 0.2, -0.4]] * K)
    c = orc.project(s, camera(), mode)["rgb"][0]
    r = orc.render(s, [camera()], mode, pixels=_px(None, [(320, 240)]))
    np.testing.assert_allclose(r["rgb"][0], c * (1 - (1 - a) ** K), rtol=2e-6)
    assert r["T"][0] == pytest.approx((1 - a) ** K, rel=2e-6)
    assert r["ncomp"][0] == K and r["last"][0] == K - 1


@pytest.mark.parametrize("mode", ["fp64", "recipe"])
def test_stop_rule(mode):
    """alpha = 0.98 layers: T 1 -> 0.02 -> 4e-4; the third would give 8e-6 < 1e-4 -> stop."""
    s = _stack_scene([0.98] * 5, [[1.0] * 3] * 5)
    r = orc.render(s, [camera()], mode, pixels=_px(None, [(320, 240)]))
    assert r["ncomp"][0] == golden()["compositing"]["alpha_098_layers_composited"]
    assert r["T"][0] == pytest.approx(4e-4, rel=1e-5)


@pytest.mark.parametrize("mode", ["fp64", "recipe"])
def test_conservation_equal_colours(mode):
    """With every colour equal to c and bg = 0: C = c (1 - T_final) at every pixel, stop or not
    (telescoping sum of Eq. 3)."""
    s = make_scene("tiny")
    s.sh[:] = 0.0
    s.sh[:, 0, :] = 1.0
    cam = make_cameras("tiny", 1)[0]
    c = 0.28209479177387814 + 0.5
    r = orc.render(s, [cam], mode)
    np.testing.assert_allclose(r["rgb"][0], np.repeat(c * (1 - r["T"][0])[None], 3, 0), atol=1e-12)
    assert (r["T"] >= 0).all() and (r["T"] <= 1).all()
    assert (r["ncomp"] > 0).mean() > 0.3


def test_monotone_occlusion():
    """Raising the opacity of front Gaussians never increases any pixel's contribution from the
    Gaussians behind them."""
    s = make_scene("tiny")
    cam = make_cameras("tiny", 1)[0]
    front = s.means[:, 2] < 1.8
    s.sh[front] = -10.0  # front layer black -> image = contribution of the rest
    r0 = orc.render(s, [cam], "fp64")["rgb"]
    s2 = s.copy()
    s2.opacity_logits[front] += 1.5
    r1 = orc.render(s2, [cam], "fp64")["rgb"]
    assert (r1 <= r0 + 1e-12).all() and (r1 < r0 - 1e-6).any()


def test_render_deterministic_and_modes_agree():
    s = make_scene("tiny")
    cam = make_cameras("tiny", 1)[0]
    a = orc.render(s, [cam], "recipe")
    b = orc.render(s, [cam], "recipe")
    assert (a["rgb"] == b["rgb"]).all() and (a["last"] == b["last"]).all()
    c = orc.render(s, [cam], "fp64")
    ok = a["flag"] == 0
    assert ok.mean() > 0.99
    d = np.abs(a["rgb"] - c["rgb"]).max(axis=1)
    assert np.quantile(d[ok], 0.999) < 1e-4
