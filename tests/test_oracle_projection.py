"""Pins of the oracle's projection (SURVEY §8(c) pins 'projection', 'cov3D',
'P3', culling) against closed forms and independent library routines (scipy rotations,
numerical Jacobians) -- never against a retyped copy of the oracle's own formulas."""
import math

import numpy as np
import pytest
from scipy.spatial.transform import Rotation

import oracle.oracle as orc
from synth import make_cameras, make_scene
from tests.helpers import camera, golden, scene_of

MODES = ["fp64", "recipe"]


@pytest.mark.parametrize("mode", MODES)
def test_projection_spec_examples(mode):
    g = golden()["projection"]
    K = g["intrinsics"]
    cam = camera(fx=K["fx"], fy=K["fy"], cx=K["cx"], cy=K["cy"], width=100, height=100)
    for case in g["cases"]:
        s = scene_of([case["p_cam"]])
        out = orc.project(s, cam, mode)
        assert out["radius"][0] > 0
        np.testing.assert_allclose(out["mean2d"][0], case["uv"], atol=1e-5)
        assert out["depth"][0] == pytest.approx(case["p_cam"][2], abs=1e-6)


@pytest.mark.parametrize("mode", MODES)
def test_p3_isotropic_footprint_and_binning(mode):
    g = golden()["P3_footprint"]
    c = g["camera"]
    cam = camera(fx=c["fx"], fy=c["fy"], cx=c["cx"], cy=c["cy"], width=c["width"], height=c["height"])
    for q in ([1, 0, 0, 0], [0.3, -0.5, 0.7, 0.2]):  # isotropic: any rotation
        s = scene_of([g["p_cam"]], log_scales=[[math.log(g["scale"])] * 3], quats=[q])
        out = orc.project(s, cam, mode)
        assert out["radius"][0] == g["radius"]
        # Sigma2 + floor on the diagonal: conic = 1/7.190625, off-diagonal 0
        np.testing.assert_allclose(out["conic"][0], [1 / g["sigma2_diag"], 0, 1 / g["sigma2_diag"]],
                                   rtol=2e-6, atol=1e-9 if mode == "fp64" else 2e-7)
        x0, y0, x1, y1 = out["rect"][0]
        tiles = sorted(ty * 40 + tx for ty in range(y0, y1) for tx in range(x0, x1))
        assert tiles == g["tiles"]
    if mode == "recipe":
        keys, vals, ranges, tt = orc.bin_pairs(s, [cam])
        assert [int(k) >> 32 for k in keys] == g["tiles"]
        assert hex(int(keys[0])) == hex(int(g["key_579"], 16))
        assert (vals == 0).all() and tt[0, 0] == 4
        assert tuple(ranges[579]) == (0, 1) and tuple(ranges[620]) == (3, 4) and ranges[:579].sum() == 0


def test_cov3d_identity_and_rotation():
    cam = camera(fx=100, fy=100, cx=50, cy=50, width=100, height=100)
    S3, _ = orc.debug_cov([0, 0, 2], [1, 0, 0, 0], [0, 0, 0], cam)
    np.testing.assert_allclose(S3, np.eye(3), atol=1e-12)
    # 90 deg z-rotation of diag(4,1,1) (log_scale = (ln 2, 0, 0)) -> diag(1,4,1)
    q = [math.cos(math.pi / 4), 0, 0, math.sin(math.pi / 4)]
    S3, S2 = orc.debug_cov([0, 0, 2], q, [math.log(2), 0, 0], cam)
    np.testing.assert_allclose(S3, np.diag([1, 4, 1]), atol=1e-6)
    # on-axis: Sigma2 = (f/z)^2 diag(1, 4) + 0.3
    np.testing.assert_allclose(S2, [2500 * 1 + 0.3, 0, 2500 * 4 + 0.3], rtol=1e-6, atol=1e-4)


def test_cov3d_eigenvalues_random():
    # eigenvalues of Sigma3 equal exp(2 log_scale) up to permutation
    rng = np.random.default_rng(0)
    cam = camera()
    for _ in range(50):
        q = rng.normal(size=4) * rng.uniform(0.3, 3)
        ls = rng.normal(-3, 1, size=3)
        S3, _ = orc.debug_cov([0, 0, 2], q, ls, cam)
        ev = np.sort(np.linalg.eigvalsh(S3))
        want = np.sort(np.exp(2 * ls.astype(np.float32).astype(np.float64)))
        np.testing.assert_allclose(ev, want, rtol=1e-6, atol=1e-12)


def _proj_fd_jacobian(pc, fx, fy):
    """Numerical Jacobian of pi(p) = (fx x/z, fy y/z) by central differences."""
    J = np.zeros((2, 3))
    h = 1e-6
    for k in range(3):
        dp = np.zeros(3)
        dp[k] = h
        a, b = pc + dp, pc - dp
        J[:, k] = (np.array([fx * a[0] / a[2], fy * a[1] / a[2]]) -
                   np.array([fx * b[0] / b[2], fy * b[1] / b[2]])) / (2 * h)
    return J


def test_cov2d_matches_independent_ewa():
    """Sigma2 = J W Sigma3 W^T J^T + 0.3 I with Sigma3 from scipy's quaternion->matrix and J a
    numerical Jacobian of the pinhole projection."""
    rng = np.random.default_rng(1)
    cams = make_cameras("tum", 3, seed=11)
    for cam in cams:
        cam = type(cam)(**{**cam.__dict__, "lim_x": float("inf"), "lim_y": float("inf")})
        W = cam.R.astype(np.float64)
        for _ in range(20):
            P = cam.centre() + W[2] * rng.uniform(1, 4) + W[0] * rng.uniform(-1, 1) + W[1] * rng.uniform(-1, 1)
            q = rng.normal(size=4)
            ls = rng.normal(-3.5, 0.5, size=3)
            res = orc.debug_cov(P.astype(np.float32), q, ls, cam)
            assert res is not None
            _, S2 = res
            Pf = P.astype(np.float32).astype(np.float64)
            pc = W @ Pf + cam.t.astype(np.float64)
            Rm = Rotation.from_quat(np.asarray([q[1], q[2], q[3], q[0]], np.float32).astype(np.float64)).as_matrix()
            S3 = Rm @ np.diag(np.exp(2 * ls.astype(np.float32).astype(np.float64))) @ Rm.T
            J = _proj_fd_jacobian(pc, cam.fx, cam.fy)
            want = J @ W @ S3 @ W.T @ J.T + 0.3 * np.eye(2)
            np.testing.assert_allclose(S2, [want[0, 0], want[0, 1], want[1, 1]], rtol=2e-6,
                                       atol=1e-6 * np.abs(want).max())


@pytest.mark.parametrize("mode", MODES)
def test_culling(mode):
    cam = camera()
    s = scene_of([[0, 0, -1], [0, 0, 0.1], [1e4, 0, 2], [0, 0, 2], [0, 0, 2]],
                 quats=[[1, 0, 0, 0]] * 4 + [[0, 0, 0, 0]])
    out = orc.project(s, cam, mode)
    # behind camera, inside the near plane, 10^6 px off image, valid, zero quaternion
    assert list(out["radius"] > 0) == [False, False, False, True, False]


def test_recipe_agrees_with_fp64_on_room_scene():
    s = make_scene("tum", n=20000)
    cam = make_cameras("tum", 1)[0]
    a, b = orc.project(s, cam, "fp64"), orc.project(s, cam, "recipe")
    vis = (a["radius"] > 0) & (b["radius"] > 0)
    assert vis.mean() > 0.1
    assert ((a["radius"] > 0) != (b["radius"] > 0)).sum() <= 2
    np.testing.assert_allclose(a["mean2d"][vis], b["mean2d"][vis], atol=2e-3)
    np.testing.assert_allclose(a["depth"][vis], b["depth"][vis], rtol=1e-6)
    np.testing.assert_allclose(a["conic"][vis], b["conic"][vis], rtol=1e-3,
                               atol=1e-4 * np.abs(a["conic"][vis]).max())
    assert (np.abs(a["radius"][vis] - b["radius"][vis]) <= 1).all()


def test_rect_is_conservative_for_cutoff():
    """Every pixel inside a Gaussian's 3-sigma ellipse (Mahalanobis^2 < 9) lies in a
    tile of its rect: brute force over all pixels of a small image."""
    s = make_scene("tiny")
    cam = make_cameras("tiny", 1)[0]
    out = orc.project(s, cam, "recipe")
    ys, xs = np.mgrid[0:cam.height, 0:cam.width]
    for i in np.nonzero(out["radius"] > 0)[0]:
        u, v = out["mean2d"][i]
        A, B, Cc = out["conic"][i]
        dx, dy = xs - u, ys - v
        inside = (A * dx * dx + 2 * B * dx * dy + Cc * dy * dy) < 9 - 1e-6
        x0, y0, x1, y1 = out["rect"][i]
        tx, ty = xs // 16, ys // 16
        in_rect = (tx >= x0) & (tx < x1) & (ty >= y0) & (ty < y1)
        assert not (inside & ~in_rect).any(), i


@pytest.mark.parametrize("cfg,n", [("tiny", None), ("tum", 20000)])
def test_ellipse_tile_binning_is_exact_and_conservative(cfg, n):
    """Exact ellipse-tile binning: a (Gaussian, tile) pair is binned iff the 3-sigma
    ellipse can reach one of the tile's pixel centres (Mahalanobis^2 <= 9 + 0.1 %), checked by brute
    force over all pixel centres in fp64 -- every pixel inside the ellipse keeps its tile, tiles the
    ellipse cannot reach are dropped -- and far fewer pairs than the square rect."""
    s = make_scene(cfg, n=n)
    cam = make_cameras(cfg, 1)[0]
    out = orc.project(s, cam, "recipe")
    keys, vals, ranges, tt = orc.bin_pairs(s, [cam])
    TX = (cam.width + 15) // 16
    binned = set(zip(vals.tolist(), (keys >> np.uint64(32)).astype(np.int64).tolist()))
    rect_pairs = 0
    rng = np.random.default_rng(0)
    vis = np.nonzero(out["radius"] > 0)[0]
    for i in (vis if cfg == "tiny" else rng.choice(vis, 400, replace=False)):
        u, v = out["mean2d"][i]
        A, B, Cc = out["conic"][i]
        x0, y0, x1, y1 = out["rect"][i]
        rect_pairs += (x1 - x0) * (y1 - y0)
        got = 0
        for ty in range(y0, y1):
            for tx in range(x0, x1):
                ys, xs = np.mgrid[ty * 16:ty * 16 + 16, tx * 16:tx * 16 + 16]
                dx, dy = xs - u, ys - v
                q = (A * dx * dx + 2 * B * dx * dy + Cc * dy * dy).min()  # over pixel centres
                # over the continuous box of pixel centres (fine grid, 1/8 px)
                ys, xs = np.mgrid[ty * 16:ty * 16 + 15.001:0.125, tx * 16:tx * 16 + 15.001:0.125]
                dx, dy = xs - u, ys - v
                qb = (A * dx * dx + 2 * B * dx * dy + Cc * dy * dy).min()
                hit = (int(i), ty * TX + tx) in binned
                got += hit
                if q < 9.0 - 1e-6:
                    assert hit, (i, tx, ty, q)   # a tile holding a reachable pixel is never dropped
                if qb > 9.02:
                    assert not hit, (i, tx, ty, qb)  # a tile the ellipse cannot reach is (0.1 % margin)
        assert got == tt[0, i]
    if cfg == "tiny":
        assert tt.sum() == keys.size and keys.size < rect_pairs


def test_exp_scale_recipe_is_correctly_rounded():
    # (float)exp((double)s) equals the correctly rounded fp32 exp (checked in long double via mpmath-free
    # error bound): compare against float64 exp rounded to float32 on a dense sample.
    s = np.linspace(-12, 3, 200001).astype(np.float32)
    np.testing.assert_array_equal(orc.exp_scale_f32(s), np.exp(s.astype(np.float64)).astype(np.float32))
