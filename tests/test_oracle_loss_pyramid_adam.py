"""Pins of the oracle's Eq. 4 loss, Gaussian pyramid
 and optimiser step against closed
forms, special cases and finite differences; plus the end-to-end convergence pin."""
import math

import numpy as np
import pytest

import oracle.oracle as orc
from tests.helpers import camera, golden, logit, scene_of

C1 = 0.01 ** 2
C2 = 0.03 ** 2


def _rand_pair(H, W, seed):
    rng = np.random.default_rng(seed)
    return rng.uniform(0, 1, size=(3, H, W)), rng.uniform(0, 1, size=(3, H, W))


def test_ssim_identical_and_loss_zero():
    x, _ = _rand_pair(20, 24, 0)
    L, S, d = orc.loss(x, x, 0.2)
    assert S == pytest.approx(1.0, abs=1e-12) and L == pytest.approx(0.0, abs=1e-12)
    assert np.abs(d).max() < 1e-12


def test_ssim_constant_images():
    a = np.full((3, 30, 30), 0.5)
    assert orc.loss(a, a, 0.2)[1] == pytest.approx(1.0, abs=1e-12)
    # constant 0 vs 1: interior pixels (window inside the image) give C1/(1+C1)
    _, _, _, m = orc.loss(np.zeros((3, 30, 30)), np.ones((3, 30, 30)), 0.2, ssim_map=True)
    np.testing.assert_allclose(m[:, 5:-5, 5:-5], C1 / (1 + C1), rtol=1e-12)


def test_ssim_zero_padded_border_closed_form():
    """Corner pixel of constant images a, b with zero padding: only the in-image quarter of the
    11x11, sigma = 1.5 window is summed, mass S = (sum_{i>=5} g_i)^2."""
    g = np.exp(-((np.arange(11) - 5) ** 2) / (2 * 1.5 ** 2))
    g /= g.sum()
    S = g[5:].sum() ** 2
    a, b = 0.3, 0.8
    mx, my = a * S, b * S
    vx, vy, cxy = a * a * S - mx * mx, b * b * S - my * my, a * b * S - mx * my
    want = (2 * mx * my + C1) * (2 * cxy + C2) / ((mx * mx + my * my + C1) * (vx + vy + C2))
    _, _, _, m = orc.loss(np.full((3, 30, 30), a), np.full((3, 30, 30), b), 0.2, ssim_map=True)
    np.testing.assert_allclose(m[:, 0, 0], want, rtol=1e-12)
    np.testing.assert_allclose(m[:, -1, -1], want, rtol=1e-12)


def test_lambda_zero_is_l1():
    x, y = _rand_pair(16, 16, 1)
    L, _, d = orc.loss(x, y, 0.0)
    assert L == pytest.approx(np.abs(x - y).mean(), rel=1e-12)
    np.testing.assert_allclose(d, np.sign(x - y) / x.size, rtol=1e-12)


def test_loss_gradient_fd():
    """random 32x32 pair, lambda = 0.2, gradient vs central FD (fp64, h = 1e-6)."""
    x, y = _rand_pair(32, 32, 2)
    _, _, d = orc.loss(x, y, 0.2)
    rng = np.random.default_rng(3)
    h = 1e-6
    for _ in range(40):
        idx = tuple(rng.integers(0, s) for s in x.shape)
        xp, xm = x.copy(), x.copy()
        xp[idx] += h
        xm[idx] -= h
        fd = (orc.loss(xp, y, 0.2, grad=False)[0] - orc.loss(xm, y, 0.2, grad=False)[0]) / (2 * h)
        assert fd == pytest.approx(d[idx], rel=1e-5, abs=1e-12)
    with pytest.raises(ValueError):
        orc.loss(x, y[:, :31], 0.2)


# ------------------------------------------------------------------------------- pyramid
def test_pyramid_level0_identity_and_constant():
    x = np.random.default_rng(0).uniform(size=(3, 33, 47))
    lv = orc.pyramid(x, 2)
    assert (lv[0] == x).all()
    assert [l.shape for l in lv] == [(3, 33, 47), (3, 17, 24), (3, 9, 12)]
    c = orc.pyramid(np.full((3, 20, 20), 0.37), 3)
    for l in c:
        np.testing.assert_allclose(l, 0.37, rtol=1e-15)


def test_pyramid_variance_decreases():
    x = np.random.default_rng(1).normal(size=(1, 64, 64))
    v = [l.var() for l in orc.pyramid(x, 2)]
    assert v[0] > v[1] > v[2]


def test_pyramid_nyquist_checkerboard_exact_constant():
    """[1,4,6,4,1] annihilates the Nyquist frequency; a reflect-101 border keeps the alternation,
    so every output pixel (borders included) equals the mean 0.5 exactly."""
    yy, xx = np.mgrid[0:24, 0:31]
    x = (0.5 + 0.5 * (-1.0) ** (xx + yy))[None]
    np.testing.assert_array_equal(orc.pyramid(x, 1)[1], 0.5)


def test_pyramid_ramp():
    """A linear ramp stays linear (slope x2 after decimation); the border value under
    reflect-101 is (2 + 4*1 + 6*0 + 4*1 + 2)/16 = 0.75."""
    x = np.tile(np.arange(40, dtype=np.float64), (1, 10, 1))
    l1 = orc.pyramid(x, 1)[1]
    assert l1[0, 3, 0] == golden()["pyramid"]["ramp_border_value"]
    np.testing.assert_allclose(np.diff(l1[0, 3, 1:-1]), 2.0, rtol=1e-14)


def test_pyramid_too_many_levels():
    with pytest.raises(ValueError):
        orc.pyramid(np.zeros((3, 8, 8)), 3)


# ------------------------------------------------------------------------------- adam
def test_adam_first_step_closed_form():
    p, m, v = orc.adam([1.0], [3e-7], [0.0], [0.0], lr=1e-3, eps=1e-15, step=1)
    assert p[0] - 1.0 == pytest.approx(golden()["adam"]["delta"], rel=1e-9)
    assert m[0] == pytest.approx(3e-8) and v[0] == pytest.approx(0.001 * 9e-14)
    p, _, _ = orc.adam([2.0], [0.0], [0.0], [0.0], lr=1e-3, step=1)
    assert p[0] == 2.0


def test_adam_constant_gradient_gives_sign_steps():
    """Bias correction: with a constant gradient every step is -lr*sign(g) (m_hat = g, v_hat = g^2)."""
    p, m, v = np.array([0.5, -0.2]), np.zeros(2), np.zeros(2)
    g = np.array([0.3, -2.0])
    for step in range(1, 6):
        p_new, m, v = orc.adam(p, g, m, v, lr=1e-2, eps=1e-15, step=step)
        np.testing.assert_allclose(p_new - p, -1e-2 * np.sign(g), rtol=1e-9)
        p = p_new


def test_sgd_mode():
    p, _, _ = orc.adam([1.0, 2.0], [0.5, -1.0], [0, 0], [0, 0], lr=0.1, sgd_mode=True)
    np.testing.assert_allclose(p, [0.95, 2.1])


# ------------------------------------------------------------------------------- convergence
def test_single_gaussian_fit_converges():
    """single-Gaussian scene vs single-splat target, 200 iterations of render ->
    Eq. 4 -> backward -> Adam: loss falls by >= 10x."""
    cam = camera(width=48, height=40, cx=24, cy=20, fx=60, fy=60)
    sh_t = np.zeros((1, 1, 3), np.float32)
    sh_t[0, 0] = [1.0, -0.5, 0.3]
    target = scene_of([[0.02, -0.01, 1.0]], log_scales=[[math.log(0.05), math.log(0.08), math.log(0.06)]],
                      quats=[[0.9, 0.2, 0.1, -0.1]], opac=[logit(0.8)], sh=sh_t)
    gt = orc.render(target, [cam], "fp64")["rgb"]
    s = target.copy()
    s.means += np.array([[0.03, 0.02, 0.05]], np.float32)
    s.log_scales += 0.3
    s.opacity_logits -= 1.0
    s.sh[0, 0] = [0.0, 0.0, 0.0]
    lrs = dict(means=2e-3, quats=1e-2, log_scales=2e-2, opacity_logits=5e-2, sh=5e-2)
    state = {k: (np.zeros_like(getattr(s, k), np.float64), np.zeros_like(getattr(s, k), np.float64)) for k in lrs}
    losses = []
    for it in range(1, 201):
        g, r, _ = orc.total_grad(s, [cam], gt, 0.2, "fp64")
        losses.append(sum(orc.loss(r["rgb"][v], gt[v], 0.2, grad=False)[0] for v in range(1)))
        for k, lr in lrs.items():
            m, v = state[k]
            p, m, v = orc.adam(getattr(s, k), g[k], m, v, lr=lr, step=it)
            state[k] = (m, v)
            setattr(s, k, p.astype(np.float32).reshape(getattr(s, k).shape))
    assert losses[-1] <= losses[0] / 10, (losses[0], losses[-1])
