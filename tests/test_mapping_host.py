"""Host-side logic of the mapping driver (no GPU): the Gaussian-pyramid schedule of Eq. 5
(SPEC.md:443-451), level geometry (R12/R19), parameter packing (include/gs.h layout) and the
bench's launch accounting."""
import math

import numpy as np
import pytest

from paper_2311_16728_b200.core import level_shapes, pack_params, param_rows, unpack
from paper_2311_16728_b200.mapping import gp_level
from paper_2311_16728_b200.levels import level_camera, level_size
from synth import make_cameras, make_scene


def test_gp_level_schedule():
    # level(0) = n; non-increasing; terminal 0; n = 0 -> always 0
    assert gp_level(0, 2, 100) == 2
    seq = [gp_level(i, 2, 100) for i in range(500)]
    assert all(a >= b for a, b in zip(seq, seq[1:]))
    assert seq[-1] == 0 and seq[199] == 1 and seq[200] == 0
    assert all(gp_level(i, 0, 10) == 0 for i in range(50))
    with pytest.raises(ValueError):
        gp_level(-1, 2, 10)


def test_level_shapes_and_cameras():
    assert level_shapes(480, 640, 2) == [(480, 640), (240, 320), (120, 160)]
    assert level_shapes(33, 47, 2) == [(33, 47), (17, 24), (9, 12)]
    assert level_size(33, 47, 2) == (9, 12) and level_size(680, 1200, 2) == (170, 300)
    cam = make_cameras("tum", 1)[0]
    c2 = level_camera(cam, 2)
    # closed form (R12): f/4 and c/4 are exact in fp32; lim = 1.3 (W/2)/fx at the level size
    assert (c2.width, c2.height) == (160, 120)
    assert c2.fx == cam.fx / 4 and c2.cx == cam.cx / 4 and c2.cy == cam.cy / 4
    assert c2.lim_x == float(np.float32(1.3 * 80 / (cam.fx / 4)))
    assert level_camera(cam, 0) is cam


def test_product_level_camera_equals_oracle_reading():
    """The engine's own level cameras (paper_2311_16728_b200.levels) and the oracle side's
    (oracle.level_camera, what the parity tests feed both sides) are written separately; they
    must agree field for field on every config and level."""
    import oracle.oracle as orc
    for cfg in ("tiny", "tum", "replica", "euroc"):
        for cam in make_cameras(cfg, 3):
            for lv in range(4):
                assert level_camera(cam, lv) == orc.level_camera(cam, lv), (cfg, lv)


def test_pack_unpack_roundtrip():
    s = make_scene("tum", n=1000)
    t = pack_params(s, device="cpu")
    assert tuple(t.shape) == (param_rows(3), 1024)
    back = unpack(t, 1000, 3)
    for k in ("means", "quats", "log_scales", "opacity_logits", "sh"):
        assert np.array_equal(back[k], getattr(s, k))
    assert (t[:, 1000:] == 0).all()


def test_launch_accounting_matches_design():
    import bench
    # bucket binning: preprocess, tile scan (+ raster schedule when views x tiles <= 8192),
    # scatter, short + long tile sorts (with the record gather), raster, 2 loss, 3 fused bwd
    assert bench.launches_per_iteration(43, True, view_tiles=1200) == 11
    assert bench.launches_per_iteration(43, True, chunked=True, view_tiles=80) == 11
    assert bench.launches_per_iteration(43, False, view_tiles=1200) == 12
    assert bench.launches_per_iteration(43, True, view_tiles=20000) == 12  # separate schedule kernel
    # radix binning, 43 key bits -> 6 digit passes, + separate gather and schedule
    assert bench.launches_per_iteration(43, True, binning=1) == 2 + (4 + 6 + 1) + 1 + 1 + 2 + 3
