"""ctypes wrapper of the CPU oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this module.  It imports nothing from
the CUDA package (paper_2311_16728_b200) and the CUDA package never imports it.

Argument marshalling only; every number is computed in oracle.c (see its header for the
paper passages each function follows).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "oracle.c")
LIB = os.path.join(HERE, "liboracle.so")
FP64, RECIPE = 0, 1
_MODES = {"fp64": FP64, "recipe": RECIPE, FP64: FP64, RECIPE: RECIPE}
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so (IEEE fp32 recipe needs -ffp-contract=off and no fast-math)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        cmd = ["gcc", "-O2", "-std=gnu11", "-fopenmp", "-ffp-contract=off", "-fno-fast-math",
               "-fPIC", "-shared", "-o", LIB + ".tmp", SRC, "-lm"]
        subprocess.run(cmd, check=True)
        os.replace(LIB + ".tmp", LIB)
    return LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            _lib = C.CDLL(LIB)
            _lib.orc_bin.restype = C.c_int64
            _lib.orc_get_threads.restype = C.c_int
    return _lib


def set_threads(n: int) -> None:
    lib().orc_set_threads(int(n))


def threads() -> int:
    return int(lib().orc_get_threads())


class OrcCamera(C.Structure):
    _fields_ = [("R", C.c_float * 9), ("t", C.c_float * 3), ("fx", C.c_float), ("fy", C.c_float),
                ("cx", C.c_float), ("cy", C.c_float), ("width", C.c_int32), ("height", C.c_int32),
                ("znear", C.c_float), ("lim_x", C.c_float), ("lim_y", C.c_float)]


def _cams(cams):
    if not isinstance(cams, (list, tuple)):
        cams = [cams]
    arr = (OrcCamera * len(cams))()
    for k, c in enumerate(cams):
        arr[k].R[:] = [float(v) for v in np.asarray(c.R, np.float32).reshape(9)]
        arr[k].t[:] = [float(v) for v in np.asarray(c.t, np.float32).reshape(3)]
        arr[k].fx, arr[k].fy, arr[k].cx, arr[k].cy = c.fx, c.fy, c.cx, c.cy
        arr[k].width, arr[k].height = int(c.width), int(c.height)
        arr[k].znear, arr[k].lim_x, arr[k].lim_y = c.znear, c.lim_x, c.lim_y
    return arr, len(cams)


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _scene_args(scene):
    arrs = [np.ascontiguousarray(scene.means, np.float32), np.ascontiguousarray(scene.quats, np.float32),
            np.ascontiguousarray(scene.log_scales, np.float32),
            np.ascontiguousarray(scene.opacity_logits, np.float32), np.ascontiguousarray(scene.sh, np.float32)]
    D = int(round(np.sqrt(scene.sh.shape[1]))) - 1
    return arrs, [C.c_int64(scene.means.shape[0]), C.c_int(D)] + [_p(a) for a in arrs]


def level_camera(cam, level: int):
    """The camera of Gaussian-pyramid level l, as the oracle reads the paper: Eq. 5 renders
    I_r^l at the level's own resolution (R19), a pinhole camera scaled by
    2^-l (pixel centres at integers, R12: u_l = fx/2^l x/z + cx/2^l), size ceil-halved per level
    (SPEC.md:402), tan clamp of R15 (1.3 (W/2)/fx) recomputed at the level's size.  Values are
    fp32 like gs_camera."""
    import dataclasses
    import math
    if level == 0:
        return cam
    H, W = cam.height, cam.width
    for _ in range(level):
        H, W = (H + 1) // 2, (W + 1) // 2
    s = 0.5 ** level
    fx, fy = np.float32(cam.fx * s).item(), np.float32(cam.fy * s).item()
    lim_x = cam.lim_x if math.isinf(cam.lim_x) else np.float32(1.3 * (0.5 * W) / fx).item()
    lim_y = cam.lim_y if math.isinf(cam.lim_y) else np.float32(1.3 * (0.5 * H) / fy).item()
    return dataclasses.replace(cam, fx=fx, fy=fy, cx=np.float32(cam.cx * s).item(),
                               cy=np.float32(cam.cy * s).item(), width=W, height=H, lim_x=lim_x, lim_y=lim_y)


def project(scene, cam, mode="recipe") -> dict:
    arrs, sargs = _scene_args(scene)
    n = scene.means.shape[0]
    out = dict(radius=np.zeros(n, np.int32), rect=np.zeros((n, 4), np.int32), depth=np.zeros(n),
               mean2d=np.zeros((n, 2)), conic=np.zeros((n, 3)), rgb=np.zeros((n, 3)), sigma=np.zeros(n),
               depth_bits=np.zeros(n, np.uint32), mean2d_f=np.zeros((n, 2), np.float32),
               conic_f=np.zeros((n, 3), np.float32))
    ca, _ = _cams(cam)
    lib().orc_project(C.c_int(_MODES[mode]), *sargs, ca,
                      *[_p(out[k]) for k in ("radius", "rect", "depth", "mean2d", "conic", "rgb", "sigma",
                                             "depth_bits", "mean2d_f", "conic_f")])
    return out


def bin_pairs(scene, cams):
    """Reference tile binning: sorted keys (u64), values (u32), ranges [V*tiles][2], tiles_touched [V][n]."""
    arrs, sargs = _scene_args(scene)
    ca, V = _cams(cams)
    n = scene.means.shape[0]
    tt = np.zeros((V, n), np.int32)
    P = lib().orc_bin(*sargs, C.c_int(V), ca, None, None, None, _p(tt))
    tiles = ((cams[0].width + 15) // 16) * ((cams[0].height + 15) // 16) if isinstance(cams, (list, tuple)) \
        else ((cams.width + 15) // 16) * ((cams.height + 15) // 16)
    keys = np.zeros(max(P, 1), np.uint64)
    vals = np.zeros(max(P, 1), np.uint32)
    ranges = np.zeros((V * tiles, 2), np.uint32)
    lib().orc_bin(*sargs, C.c_int(V), ca, _p(keys), _p(vals), _p(ranges), _p(tt))
    return keys[:P], vals[:P], ranges, tt


def all_pixels(V, H, W) -> np.ndarray:
    v, y, x = np.meshgrid(np.arange(V), np.arange(H), np.arange(W), indexing="ij")
    return np.ascontiguousarray(np.stack([v.ravel(), y.ravel(), x.ravel()], 1).astype(np.int32))


def render(scene, cams, mode="recipe", bg=(0.0, 0.0, 0.0), pixels=None) -> dict:
    """Per-pixel brute-force Eq. 3.  pixels: int32 [npix, 3] (view, y, x) or None = every pixel,
    in which case outputs are reshaped to rgb [V,3,H,W], T/ncomp/last/flag [V,H,W]."""
    arrs, sargs = _scene_args(scene)
    ca, V = _cams(cams)
    cam0 = cams[0] if isinstance(cams, (list, tuple)) else cams
    full = pixels is None
    pix = all_pixels(V, cam0.height, cam0.width) if full else np.ascontiguousarray(pixels, np.int32)
    npix = pix.shape[0]
    rgb = np.zeros((npix, 3))
    T = np.zeros(npix)
    nc = np.zeros(npix, np.int32)
    last = np.zeros(npix, np.int64)
    flag = np.zeros(npix, np.int32)
    bga = np.asarray(bg, np.float64)
    lib().orc_render(C.c_int(_MODES[mode]), *sargs, C.c_int(V), ca, _p(bga), C.c_int64(npix), _p(pix),
                     _p(rgb), _p(T), _p(nc), _p(last), _p(flag))
    out = dict(rgb=rgb, T=T, ncomp=nc, last=last, flag=flag, pixels=pix)
    if full:
        H, W = cam0.height, cam0.width
        out.update(rgb=rgb.reshape(V, H, W, 3).transpose(0, 3, 1, 2).copy(), T=T.reshape(V, H, W),
                   ncomp=nc.reshape(V, H, W), last=last.reshape(V, H, W), flag=flag.reshape(V, H, W))
    return out


def backward(scene, cams, dL_drgb, mode="recipe", bg=(0.0, 0.0, 0.0), pixels=None, mag=False) -> dict:
    """Gradients of sum_v <dL/dI_v, I_v>.  dL_drgb: [V,3,H,W] (pixels None) or [npix,3].
    mag=True adds out["mag"][class] (same shapes): each element's sum of absolute per-pixel
    terms carried through |chain Jacobian| (oracle.c orc_backward), the rounding allowance's scale."""
    arrs, sargs = _scene_args(scene)
    ca, V = _cams(cams)
    cam0 = cams[0] if isinstance(cams, (list, tuple)) else cams
    if pixels is None:
        pix = all_pixels(V, cam0.height, cam0.width)
        g = np.ascontiguousarray(np.asarray(dL_drgb, np.float64).transpose(0, 2, 3, 1).reshape(-1, 3))
    else:
        pix = np.ascontiguousarray(pixels, np.int32)
        g = np.ascontiguousarray(np.asarray(dL_drgb, np.float64).reshape(-1, 3))
    n = scene.means.shape[0]
    K = scene.sh.shape[1]
    out = dict(means=np.zeros((n, 3)), quats=np.zeros((n, 4)), log_scales=np.zeros((n, 3)),
               opacity_logits=np.zeros(n), sh=np.zeros((n, K, 3)), grad2d_norm=np.zeros(n),
               flagged=np.zeros(n, np.int32))
    bga = np.asarray(bg, np.float64)
    P = 11 + 3 * K
    mg = np.zeros((n, P)) if mag else None
    lib().orc_backward(C.c_int(_MODES[mode]), *sargs, C.c_int(V), ca, _p(bga), C.c_int64(pix.shape[0]), _p(pix),
                       _p(g), *[_p(out[k]) for k in ("means", "quats", "log_scales", "opacity_logits", "sh",
                                                      "grad2d_norm", "flagged")], _p(mg) if mag else None)
    if mag:
        out["mag"] = dict(means=mg[:, 0:3].copy(), quats=mg[:, 3:7].copy(), log_scales=mg[:, 7:10].copy(),
                          opacity_logits=mg[:, 10].copy(), sh=mg[:, 11:].reshape(n, K, 3).copy())
    return out


def loss(render_img, gt, lam=0.2, grad=True, ssim_map=False):
    """Eq. 4 for one view; images [3,H,W].  Returns (loss, mean_ssim, dL/drender or None)
    (+ the per-pixel SSIM map if ssim_map)."""
    r = np.ascontiguousarray(render_img, np.float64)
    g = np.ascontiguousarray(gt, np.float64)
    if r.shape != g.shape or r.ndim != 3 or r.shape[0] != 3:
        raise ValueError("DimensionMismatch")
    H, W = r.shape[1:]
    out_l, out_s = C.c_double(), C.c_double()
    d = np.zeros_like(r) if grad else None
    smap = np.zeros_like(r) if ssim_map else None
    lib().orc_loss(_p(r), _p(g), C.c_int(H), C.c_int(W), C.c_double(lam), C.byref(out_l), C.byref(out_s), _p(d),
                   _p(smap))
    if ssim_map:
        return out_l.value, out_s.value, d, smap
    return out_l.value, out_s.value, d


def pyramid(img, n_levels: int) -> list:
    """Levels 0..n of the Gaussian pyramid of a [C,H,W] image (level 0 = input)."""
    x = np.ascontiguousarray(img, np.float64)
    Cc, H, W = x.shape
    if n_levels < 0 or (n_levels > 0 and min(H, W) <= 2 ** n_levels):
        raise ValueError("TooManyLevels")
    levels = [x]
    for _ in range(n_levels):
        Cc, H, W = levels[-1].shape
        out = np.zeros((Cc, (H + 1) // 2, (W + 1) // 2))
        lib().orc_pyramid_level(_p(levels[-1]), C.c_int(Cc), C.c_int(H), C.c_int(W), _p(out))
        levels.append(out)
    return levels


def adam(p, g, m, v, lr, beta1=0.9, beta2=0.999, eps=1e-15, step=1, sgd_mode=False):
    """In-place optimiser step on fp64 copies; returns (p, m, v)."""
    p = np.ascontiguousarray(p, np.float64).copy()
    g = np.ascontiguousarray(g, np.float64)
    m = np.ascontiguousarray(m, np.float64).copy()
    v = np.ascontiguousarray(v, np.float64).copy()
    lib().orc_adam(C.c_int64(p.size), _p(p), _p(g), _p(m), _p(v), C.c_double(lr), C.c_double(beta1),
                   C.c_double(beta2), C.c_double(eps), C.c_int64(step), C.c_int(int(sgd_mode)))
    return p, m, v


def debug_cov(mean, quat, log_scale, cam):
    """(Sigma3 [3,3], Sigma2 (a, b, c) incl. floor) from the fp64 projection, or None if culled."""
    S3 = np.zeros(9)
    S2 = np.zeros(3)
    ca, _ = _cams(cam)
    ok = lib().orc_debug_cov(_p(np.asarray(mean, np.float32)), _p(np.asarray(quat, np.float32)),
                             _p(np.asarray(log_scale, np.float32)), ca, _p(S3), _p(S2))
    return (S3.reshape(3, 3), S2) if ok else None


def sh_basis(D, dirs):
    d = np.ascontiguousarray(dirs, np.float64).reshape(-1, 3)
    Y = np.zeros((d.shape[0], 16))
    dY = np.zeros((d.shape[0], 16, 3))
    lib().orc_sh_basis(C.c_int(D), C.c_int64(d.shape[0]), _p(d), _p(Y), _p(dY))
    return Y, dY


def scene_records(scene) -> np.ndarray:
    """Per-Gaussian parameter records [n][K] (P xyz | q wxyz | log s | logit | SH coefficient-major,
    the row order of the parameter layout) from a synth.Scene."""
    n = scene.means.shape[0]
    return np.ascontiguousarray(np.concatenate([scene.means, scene.quats, scene.log_scales,
                                                scene.opacity_logits[:, None], scene.sh.reshape(n, -1)], 1),
                                np.float32)


def densify(rec, m, v, grad_accum, vis_count, max_radius, z, grad_thr, percent_dense, extent, op_thr,
            max_screen) -> dict:
    """SPEC.md:463-471 densify_and_prune on per-Gaussian records [n][K] (see oracle.c)."""
    rec = np.ascontiguousarray(rec, np.float32)
    n, K = rec.shape
    m = np.ascontiguousarray(m, np.float32)
    v = np.ascontiguousarray(v, np.float32)
    ga = np.ascontiguousarray(grad_accum, np.float32)
    vc = np.ascontiguousarray(vis_count, np.float32)
    mr = np.ascontiguousarray(max_radius, np.int32)
    z = np.ascontiguousarray(z, np.float32).reshape(n, 2, 3)
    cls = np.zeros(n, np.int8)
    counts = np.zeros(4, np.int64)
    args = (C.c_int64(n), C.c_int(K), _p(rec), _p(m), _p(v), _p(ga), _p(vc), _p(mr), _p(z), C.c_float(grad_thr),
            C.c_float(percent_dense), C.c_float(extent), C.c_float(op_thr), C.c_int32(max_screen), _p(cls),
            _p(counts))
    lib().orc_densify(*args, None, None, None)
    nn = int(counts[3])
    out, om, ov = (np.zeros((max(nn, 1), K)) for _ in range(3))
    lib().orc_densify(*args, _p(out), _p(om), _p(ov))
    return dict(cls=cls, n_clone=int(counts[0]), n_split=int(counts[1]), n_prune=int(counts[2]), n_new=nn,
                rec=out[:nn], m=om[:nn], v=ov[:nn])


def geometry_densify(cam, uv, active, kp_depth, depth_map, image, mode, D=3, rho=100.0) -> dict:
    """SPEC.md:473-481 geometry_densify (see oracle.c): new temporary primitives for the inactive
    keypoints; rec [count][K] per-Gaussian records (fp64), src = keypoint index of each."""
    ca, _ = _cams(cam)
    uv = np.ascontiguousarray(uv, np.float32).reshape(-1, 2)
    nk = uv.shape[0]
    act = np.ascontiguousarray(active, np.int32)
    kd = np.ascontiguousarray(kp_depth, np.float32)
    dm = None if depth_map is None else np.ascontiguousarray(depth_map, np.float32)
    img = np.ascontiguousarray(image, np.float32)
    K = 11 + 3 * (D + 1) ** 2
    lib().orc_geometry_densify.restype = C.c_int64
    args = (ca, C.c_int64(nk), _p(uv), _p(act), _p(kd), _p(dm), _p(img), C.c_int(mode), C.c_int(D), C.c_float(rho))
    cnt = lib().orc_geometry_densify(*args, None, None)
    rec = np.zeros((max(cnt, 1), K))
    src = np.zeros(max(cnt, 1), np.int32)
    lib().orc_geometry_densify(*args, _p(rec), _p(src))
    return dict(count=int(cnt), rec=rec[:cnt], src=src[:cnt])


def exp_scale_f32(s):
    s = np.ascontiguousarray(s, np.float32)
    out = np.zeros_like(s)
    lib().orc_exp_scale_f32(C.c_int64(s.size), _p(s), _p(out))
    return out


def total_loss(scene, cams, gts, lam=0.2, mode="fp64", bg=(0.0, 0.0, 0.0)):
    """sum_v L(render_v, gt_v): the iteration objective."""
    r = render(scene, cams, mode=mode, bg=bg)
    return sum(loss(r["rgb"][v], gts[v], lam, grad=False)[0] for v in range(r["rgb"].shape[0]))


def total_grad(scene, cams, gts, lam=0.2, mode="fp64", bg=(0.0, 0.0, 0.0)):
    """Analytic gradient of total_loss: loss gradient per view fed to the backward."""
    r = render(scene, cams, mode=mode, bg=bg)
    dL = np.stack([loss(r["rgb"][v], gts[v], lam)[2] for v in range(r["rgb"].shape[0])])
    return backward(scene, cams, dL, mode=mode, bg=bg), r, dL
