"""Small scene builders shared by the tests (inputs only; no method arithmetic)."""
from __future__ import annotations

import json
import math
import os

import numpy as np

from synth import Camera, Scene

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def golden(name="spec_examples.json"):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def camera(fx=525.0, fy=525.0, cx=320.0, cy=240.0, width=640, height=480, R=None, t=None,
           lim=float("inf"), znear=0.2):
    R = np.eye(3, dtype=np.float32) if R is None else np.asarray(R, np.float32)
    t = np.zeros(3, np.float32) if t is None else np.asarray(t, np.float32)
    return Camera(R, t, fx, fy, cx, cy, width, height, znear, lim, lim)


def scene_of(means, log_scales=None, quats=None, opac=None, sh=None, D=0):
    means = np.atleast_2d(np.asarray(means, np.float32))
    n = means.shape[0]
    log_scales = np.full((n, 3), math.log(0.01), np.float32) if log_scales is None else \
        np.atleast_2d(np.asarray(log_scales, np.float32))
    quats = np.tile(np.array([1, 0, 0, 0], np.float32), (n, 1)) if quats is None else \
        np.atleast_2d(np.asarray(quats, np.float32))
    opac = np.zeros(n, np.float32) if opac is None else np.atleast_1d(np.asarray(opac, np.float32))
    if sh is None:
        sh = np.zeros((n, (D + 1) ** 2, 3), np.float32)
        sh[:, 0, :] = 1.0
    return Scene(means, quats, log_scales, opac, np.asarray(sh, np.float32))


def logit(p):
    return math.log(p / (1 - p))


def random_small_scene(n, seed, D=0, depth=2.0, spread=0.5, scale=0.04, width=64, height=48, f=60.0):
    """n Gaussians in a cube in front of an identity camera (tiny-config shaped)."""
    rng = np.random.default_rng(seed)
    means = rng.uniform(-spread, spread, size=(n, 3)) + np.array([0, 0, depth])
    ls = math.log(scale) + rng.normal(0, 0.3, size=(n, 3))
    q = rng.normal(size=(n, 4))
    q *= rng.uniform(0.5, 2.0, size=(n, 1)) / np.linalg.norm(q, axis=1, keepdims=True)
    op = rng.uniform(-2, 3, size=n)
    sh = np.zeros((n, (D + 1) ** 2, 3))
    sh[:, 0] = rng.uniform(-1.5, 1.5, size=(n, 3))
    if D > 0:
        sh[:, 1:] = rng.normal(0, 0.3, size=(n, (D + 1) ** 2 - 1, 3))
    s = Scene(means.astype(np.float32), q.astype(np.float32), ls.astype(np.float32), op.astype(np.float32),
              sh.astype(np.float32))
    cam = camera(fx=f, fy=f, cx=(width - 1) / 2, cy=(height - 1) / 2, width=width, height=height,
                 lim=1.3 * (width / 2) / f)
    return s, cam
