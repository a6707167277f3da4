"""Pins of the oracle's geometry-based densification (SPEC.md:473-481,
PAPER.md:231-233): SPEC's worked examples, the back-projection against an independent numpy
projection, the K = 4 inverse-distance depth against a brute-force numpy neighbour search, the
create_map_points initialisation in closed form, and the edge cases."""
import math

import numpy as np

import oracle.oracle as orc
from tests.helpers import camera

C0 = 0.28209479177387814


def _cam():
    R = np.array([[0.0, -1.0, 0.0], [1.0, 0.0, 0.0], [0.0, 0.0, 1.0]], np.float32)  # exact rotation
    return camera(width=160, height=120, cx=80.0, cy=60.0, fx=100.0, fy=100.0, R=R,
                  t=np.array([0.1, -0.2, 0.3], np.float32))


def _image(seed=0):
    return np.random.default_rng(seed).uniform(0.05, 0.95, (3, 120, 160)).astype(np.float32)


def _project(cam, P):
    pc = np.asarray(cam.R, np.float64) @ P + np.asarray(cam.t, np.float64)
    return cam.fx * pc[0] / pc[2] + cam.cx, cam.fy * pc[1] / pc[2] + cam.cy, pc[2]


def test_all_active_gives_nothing():
    cam = _cam()
    uv = np.random.default_rng(1).uniform(0, 100, (20, 2))
    out = orc.geometry_densify(cam, uv, np.ones(20), np.ones(20), np.ones((120, 160)), _image(), mode=1)
    assert out["count"] == 0


def test_rgbd_backprojection_and_init():
    cam = _cam()
    rng = np.random.default_rng(2)
    uv = np.stack([rng.integers(0, 160, 50), rng.integers(0, 120, 50)], 1).astype(np.float32)
    active = (rng.uniform(size=50) < 0.3).astype(np.int32)
    depth = rng.uniform(0.5, 4.0, (120, 160)).astype(np.float32)
    depth[uv[5, 1].astype(int), uv[5, 0].astype(int)] = 0.0  # invalid depth: skipped
    active[5] = 0
    img = _image(3)
    out = orc.geometry_densify(cam, uv, active, np.zeros(50), depth, img, mode=1, D=3)
    expect = [k for k in range(50) if not active[k] and k != 5]
    assert list(out["src"]) == expect
    for rec, k in zip(out["rec"], out["src"]):
        u, v = uv[k]
        d = float(depth[int(v), int(u)])
        pu, pv, pz = _project(cam, rec[:3])
        assert abs(pu - u) < 1e-9 and abs(pv - v) < 1e-9 and abs(pz - d) < 1e-9
        assert list(rec[3:7]) == [1.0, 0.0, 0.0, 0.0]
        np.testing.assert_allclose(rec[7:10], math.log(d / cam.fx), rtol=1e-12)
        assert abs(rec[10] - math.log(0.1 / 0.9)) < 1e-12
        np.testing.assert_allclose(C0 * rec[11:14] + 0.5, img[:, int(v), int(u)], atol=1e-12)
        assert (rec[14:] == 0).all()


def test_mono_equidistant_depths_average():
    cam = _cam()
    uv = np.array([[50, 50], [40, 50], [60, 50]], np.float32)
    out = orc.geometry_densify(cam, uv, [0, 1, 1], [0.0, 1.0, 3.0], None, _image(), mode=0)
    assert out["count"] == 1 and out["src"][0] == 0
    assert abs(_project(cam, out["rec"][0, :3])[2] - 2.0) < 1e-9


def test_mono_radius_and_coincident():
    cam = _cam()
    uv = np.array([[10, 10], [110, 10], [10, 110.5], [20, 20], [20, 20]], np.float32)
    # keypoint 0: active 1 at exactly 100 px (included), active 2 at 100.5 px (excluded)
    out = orc.geometry_densify(cam, uv, [0, 1, 1, 0, 1], [0, 2.5, 7.0, 0, 1.5], None, _image(), mode=0)
    assert list(out["src"]) == [0, 3]
    z = [_project(cam, r[:3])[2] for r in out["rec"]]
    w0, w4 = 1 / 100.0, 1 / math.hypot(10, 10)  # keypoint 0 sees actives 1 (100 px) and 4
    assert abs(z[0] - (w0 * 2.5 + w4 * 1.5) / (w0 + w4)) < 1e-9
    assert abs(z[1] - 1.5) < 1e-12  # coincident active neighbour: its depth exactly
    # nobody within 100 px -> skipped
    out = orc.geometry_densify(cam, np.array([[0, 0], [150, 110]], np.float32), [0, 1], [0, 1.0], None,
                               _image(), mode=0)
    assert out["count"] == 0


def test_mono_k4_nearest_brute_force():
    cam = _cam()
    rng = np.random.default_rng(7)
    n = 400
    uv = rng.uniform(0, [159, 119], (n, 2)).astype(np.float32)  # rounded pixel inside the image
    active = (rng.uniform(size=n) < 0.3).astype(np.int32)
    kd = rng.uniform(0.5, 5.0, n).astype(np.float32)
    out = orc.geometry_densify(cam, uv, active, kd, None, _image(), mode=0)
    act = np.nonzero(active)[0]
    got = dict(zip(out["src"], out["rec"]))
    for k in np.nonzero(active == 0)[0]:
        d = np.hypot(*(uv[act] - uv[k]).astype(np.float64).T)
        keep = d <= 100.0
        if not keep.any():
            assert k not in got
            continue
        idx = act[keep][np.argsort(d[keep], kind="stable")[:4]]
        dd = np.hypot(*(uv[idx] - uv[k]).astype(np.float64).T)
        expect = (kd[idx] / dd).sum() / (1 / dd).sum()
        assert abs(_project(cam, got[k][:3])[2] - expect) < 1e-6 * expect
