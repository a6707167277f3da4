"""Per-level inputs the mapping engine derives itself (no arithmetic of the method's stages):
the camera of a Gaussian-pyramid level and the random samples densification draws.

Kept inside the package so that the product path never imports the test-input generators
(synth/) or anything the oracle side uses."""
from __future__ import annotations

import dataclasses
import math

import numpy as np


def level_size(height: int, width: int, level: int) -> tuple[int, int]:
    """Image size at GP level l: each level halves with ceil (R18)."""
    for _ in range(level):
        height, width = -(-height // 2), -(-width // 2)
    return height, width


def level_camera(cam, level: int):
    """The keyframe camera at GP level l (R12/R19: the level is rendered at its
    own intrinsics): fx, fy, cx, cy times 2^-l rounded to fp32 (exact: a power-of-two scale),
    ceil-halved size, and the EWA tan clamp of R15 recomputed for the level's size,
    lim = fp32(1.3 (W/2) / fx) (+inf stays +inf).  `cam` is any dataclass with the gs_camera
    fields; a copy is returned (level 0: `cam` itself)."""
    if level == 0:
        return cam
    scale = math.ldexp(1.0, -level)
    H, W = level_size(cam.height, cam.width, level)
    f32 = lambda x: float(np.float32(x))  # noqa: E731
    fx, fy = f32(cam.fx * scale), f32(cam.fy * scale)
    lim_x = cam.lim_x if math.isinf(cam.lim_x) else f32(1.3 * (0.5 * W) / fx)
    lim_y = cam.lim_y if math.isinf(cam.lim_y) else f32(1.3 * (0.5 * H) / fy)
    return dataclasses.replace(cam, fx=fx, fy=fy, cx=f32(cam.cx * scale), cy=f32(cam.cy * scale),
                               width=W, height=H, lim_x=lim_x, lim_y=lim_y)


def densify_samples(n: int, seed: int) -> np.ndarray:
    """The randomness of densification (a clone is shifted by a sample of its own
    Gaussian, a split draws two): standard-normal z [n][2][3] float32 from a seeded PCG64
    stream, passed to gs_densify_apply as an input (R29)."""
    rng = np.random.default_rng(np.random.PCG64(seed))
    return rng.normal(size=(n, 2, 3)).astype(np.float32)
