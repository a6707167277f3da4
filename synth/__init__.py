"""Seeded synthetic inputs shared by the CUDA path, the oracle, the tests and the bench.

This package only *constructs inputs* (Gaussian parameter arrays, camera poses and
intrinsics, ground-truth-like images).  It contains none of the method's arithmetic
(no projection, no SH evaluation, no compositing, no loss): see DESIGN.md "Input recipe".
"""
from .scenes import (  # noqa: F401
    CONFIGS, Camera, Scene, make_scene, make_cameras, noise_image, perturb,
    level_shape, config, densify_samples, make_keypoints, edge_scene,
)
