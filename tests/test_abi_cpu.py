"""CPU-side checks of the C ABI (no GPU): libgs.so builds for sm_100a, loads, exports every
function include/gs.h declares, and rejects bad arguments synchronously without touching the
device (include/gs.h error conventions)."""
import ctypes as C
import math
import os
import re

import pytest

from paper_2311_16728_b200 import _lib as L
from paper_2311_16728_b200.build import build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "gs.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gs_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    build()
    return L.lib()


def test_exports_every_declared_symbol(lib):
    names = declared_functions()
    assert len(names) >= 16
    assert set(names) == set(L.EXPORTS)
    for n in names:
        assert hasattr(lib, n), n


def test_built_for_sm100a():
    path = build()
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {path} 2>&1").read()
    assert "sm_100a" in out


def test_layout_helpers(lib):
    assert lib.gs_param_rows(0) == 14 and lib.gs_param_rows(3) == 59
    assert lib.gs_param_ld(1) == 64 and lib.gs_param_ld(64) == 64 and lib.gs_param_ld(65) == 128
    b1 = L.gs_workspace_size(1000, 1, 64, 48, 10000)
    b2 = L.gs_workspace_size(1000, 1, 64, 48, 100000)
    assert 0 < b1 < b2
    assert "capacity" in L.status_str(L.GS_ERR_CAPACITY)


def test_synchronous_argument_errors(lib):
    """Validation happens on the host before anything is enqueued (no device needed)."""
    ps = L.GsParams(None, 10, 64, 0)
    cams = L.camera_struct([type("c", (), dict(R=[1, 0, 0, 0, 1, 0, 0, 0, 1], t=[0, 0, 0], fx=1.0, fy=1.0, cx=0.0,
                                                 cy=0.0, width=8, height=8, znear=0.2, lim_x=math.inf,
                                                 lim_y=math.inf))()])
    assert lib.gs_preprocess(C.byref(ps), cams, 1, None, 0, None) == L.GS_ERR_INVALID_ARG
    ps = L.GsParams(C.c_void_p(16), 10, 10, 0)  # ld not a multiple of 4
    assert lib.gs_preprocess(C.byref(ps), cams, 1, C.c_void_p(16), 0, None) == L.GS_ERR_SHAPE
    ps = L.GsParams(C.c_void_p(16), 10, 64, 4)  # SH degree 4
    assert lib.gs_preprocess(C.byref(ps), cams, 1, C.c_void_p(16), 0, None) == L.GS_ERR_INVALID_ARG
    ps = L.GsParams(C.c_void_p(16), 10, 64, 0)
    assert lib.gs_preprocess(C.byref(ps), cams, 65, C.c_void_p(16), 1 << 20, None) == L.GS_ERR_NOT_SUPPORTED
    # workspace too small -> shape error
    assert lib.gs_preprocess(C.byref(ps), cams, 1, C.c_void_p(16), 16, None) == L.GS_ERR_SHAPE
    # backward before any forward on this workspace -> StaleRenderState
    need = L.gs_workspace_size(10, 1, 8, 8, 4096)
    bg = (C.c_float * 3)(0, 0, 0)
    assert lib.gs_render_backward(C.byref(ps), cams, 1, C.c_void_p(1 << 20), C.c_size_t(need), bg, C.c_void_p(16),
                                  C.c_void_p(16), None, None) == L.GS_ERR_STALE_STATE
    assert lib.gs_render_forward(C.byref(ps), cams, 1, C.c_void_p(1 << 20), C.c_size_t(need), bg, C.c_void_p(16),
                                 None, None) == L.GS_ERR_STALE_STATE
    # pyramid: TooManyLevels
    assert lib.gs_pyramid(C.c_void_p(16), 1, 3, 8, 8, 3, C.c_void_p(16), None) == L.GS_ERR_SHAPE
    assert lib.gs_pyramid(C.c_void_p(16), 1, 3, 8, 8, 0, None, None) == L.GS_OK
    # loss: lambda outside [0, 1]
    assert lib.gs_photometric_loss(C.c_void_p(16), C.c_void_p(16), 1, 8, 8, C.c_float(1.5), C.c_void_p(16),
                                   None, C.c_void_p(16), C.c_size_t(1 << 20), None) == L.GS_ERR_INVALID_ARG
    # adam: step must be >= 1, range inside [0, n]
    hp = L.GsAdamHparams()
    assert lib.gs_adam_step(C.byref(ps), C.c_void_p(16), C.c_void_p(16), C.c_void_p(16), C.byref(hp), C.c_int64(0),
                            C.c_int64(0), C.c_int64(10), 0, None) == L.GS_ERR_INVALID_ARG
    assert lib.gs_adam_step(C.byref(ps), C.c_void_p(16), C.c_void_p(16), C.c_void_p(16), C.byref(hp), C.c_int64(1),
                            C.c_int64(0), C.c_int64(11), 0, None) == L.GS_ERR_INVALID_ARG


def test_binding_fails_loudly_without_library(tmp_path):
    old = L._lib
    try:
        L._lib = None
        with pytest.raises(RuntimeError, match="no CPU fallback"):
            L.lib(str(tmp_path / "missing.so"))
    finally:
        L._lib = old
