"""Thin ctypes binding of libgs.so (include/gs.h): argument marshalling only.

Every function here has the name of the C entry point it calls and takes torch tensors
(device memory owned by torch) plus host structs; it passes raw pointers and the current
CUDA stream, checks the returned gs_status and raises on error.  There is no fallback: if
libgs.so is missing or a call fails, an exception is raised.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import threading

import torch

PKG = os.path.dirname(os.path.abspath(__file__))
# GS_LIB_PATH: an alternative build of the same sources (tools/build_variant.py A/B experiments)
LIB_PATH = os.environ.get("GS_LIB_PATH") or os.path.join(PKG, "libgs.so")

GS_OK, GS_ERR_INVALID_ARG, GS_ERR_SHAPE, GS_ERR_CAPACITY, GS_ERR_STALE_STATE, GS_ERR_CUDA, \
    GS_ERR_NOT_SUPPORTED = range(7)
GS_MAX_VIEWS = 64
GS_TILE = 16

# every symbol declared in include/gs.h
EXPORTS = ["gs_param_rows", "gs_param_ld", "gs_workspace_size", "gs_preprocess", "gs_render_forward",
           "gs_loss_workspace_size", "gs_photometric_loss", "gs_render_backward", "gs_render_backward_adam",
           "gs_pyramid", "gs_adam_step", "gs_adam_step_rows", "gs_adam_step_rows_dev", "gs_densify_temp_size", "gs_densify_stats",
           "gs_densify_plan", "gs_densify_apply", "gs_densify_tags", "gs_geometry_densify",
           "gs_query_status", "gs_status_async", "gs_workspace_release", "gs_status_str",
           "gs_comm_shard", "gs_peer_barrier", "gs_reduce_adam_bcast", "gs_spatial_order_temp_size", "gs_spatial_order",
           "gs_permute_columns", "gs_sort_temp_size", "gs_debug_sort_pairs",
           "gs_debug_workspace_view", "gs_set_binning", "gs_set_render_stats", "gs_profile_kernel", "gs_profile_read", "gs_debug_exp_scale"]


class GsError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        super().__init__(f"{where}: gs_status {status} ({status_str(status)})")


class GsCamera(C.Structure):
    _fields_ = [("R", C.c_float * 9), ("t", C.c_float * 3), ("fx", C.c_float), ("fy", C.c_float),
                ("cx", C.c_float), ("cy", C.c_float), ("width", C.c_int32), ("height", C.c_int32),
                ("znear", C.c_float), ("lim_x", C.c_float), ("lim_y", C.c_float)]


class GsParams(C.Structure):
    _fields_ = [("data", C.c_void_p), ("n", C.c_int64), ("ld", C.c_int64), ("sh_degree", C.c_int32)]


class GsAdamHparams(C.Structure):
    _fields_ = [("lr", C.c_float * 6), ("beta1", C.c_float), ("beta2", C.c_float), ("eps", C.c_float),
                ("sgd_mode", C.c_int32)]


class GsDensifyCfg(C.Structure):
    _fields_ = [("grad_threshold", C.c_float), ("percent_dense", C.c_float), ("scene_extent", C.c_float),
                ("opacity_threshold", C.c_float), ("max_screen_px", C.c_int32)]


class GsWsView(C.Structure):
    _fields_ = [("rec0", C.c_void_p), ("rec1", C.c_void_p), ("rec2", C.c_void_p), ("depth", C.c_void_p),
                ("radius", C.c_void_p), ("rect", C.c_void_p), ("tiles_touched", C.c_void_p),
                ("offsets", C.c_void_p), ("keys", C.c_void_p), ("vals", C.c_void_p), ("ranges", C.c_void_p),
                ("n_contrib", C.c_void_p), ("n_composited", C.c_void_p), ("capacity", C.c_int64)]


_lib = None
_lock = threading.Lock()


def lib(path: str | None = None):
    """Load libgs.so (built in-tree by paper_2311_16728_b200.build).  Raises if absent."""
    global _lib
    with _lock:
        if _lib is None:
            p = path or LIB_PATH
            if not os.path.exists(p):
                raise RuntimeError(f"libgs.so not found at {p}: run `python -m paper_2311_16728_b200.build` "
                                   "(there is no CPU fallback)")
            L = C.CDLL(p)
            L.gs_param_rows.restype = C.c_int32
            L.gs_param_rows.argtypes = [C.c_int32]
            L.gs_param_ld.restype = C.c_int64
            L.gs_param_ld.argtypes = [C.c_int64]
            L.gs_status_str.restype = C.c_char_p
            L.gs_status_str.argtypes = [C.c_int]
            for name in EXPORTS:
                if name not in ("gs_param_rows", "gs_param_ld", "gs_status_str"):
                    getattr(L, name).restype = C.c_int
            _lib = L
    return _lib


def status_str(s: int) -> str:
    try:
        return lib().gs_status_str(int(s)).decode()
    except Exception:  # noqa: BLE001
        return "?"


def _check(s: int, where: str):
    if s != GS_OK:
        raise GsError(s, where)


def _stream(stream=None):
    st = torch.cuda.current_stream() if stream is None else stream
    return C.c_void_p(st.cuda_stream)


def _ptr(t: torch.Tensor | None):
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("device tensor required")
    if not t.is_contiguous():
        raise ValueError("contiguous tensor required")
    return C.c_void_p(t.data_ptr())


def camera_struct(cams) -> C.Array:
    """Host array of gs_camera from objects with R, t, fx, fy, cx, cy, width, height, znear, lim_x, lim_y."""
    if not isinstance(cams, (list, tuple)):
        cams = [cams]
    arr = (GsCamera * len(cams))()
    for k, c in enumerate(cams):
        R = [float(x) for x in (c.R.reshape(-1) if hasattr(c.R, "reshape") else c.R)]
        t = [float(x) for x in (c.t.reshape(-1) if hasattr(c.t, "reshape") else c.t)]
        arr[k].R[:] = R
        arr[k].t[:] = t
        arr[k].fx, arr[k].fy, arr[k].cx, arr[k].cy = c.fx, c.fy, c.cx, c.cy
        arr[k].width, arr[k].height = int(c.width), int(c.height)
        arr[k].znear = c.znear
        arr[k].lim_x = c.lim_x if math.isfinite(c.lim_x) else float("inf")
        arr[k].lim_y = c.lim_y if math.isfinite(c.lim_y) else float("inf")
    return arr


def param_rows(sh_degree: int) -> int:
    return int(lib().gs_param_rows(sh_degree))


def param_ld(n: int) -> int:
    return int(lib().gs_param_ld(n))


def params_struct(data: torch.Tensor, n: int, sh_degree: int) -> GsParams:
    """data: float32 CUDA tensor [K, ld]."""
    K = param_rows(sh_degree)
    if data.dtype != torch.float32 or data.dim() != 2 or data.shape[0] != K:
        raise ValueError(f"params must be float32 [{K}, ld]")
    return GsParams(data.data_ptr(), n, data.shape[1], sh_degree)


def gs_workspace_size(n, n_views, width, height, pair_capacity) -> int:
    b = C.c_size_t()
    _check(lib().gs_workspace_size(C.c_int64(n), C.c_int32(n_views), C.c_int32(width), C.c_int32(height),
                                   C.c_int64(pair_capacity), C.byref(b)), "gs_workspace_size")
    return b.value


def gs_preprocess(params: GsParams, cams, ws: torch.Tensor, stream=None):
    ca = camera_struct(cams)
    _check(lib().gs_preprocess(C.byref(params), ca, C.c_int32(len(ca)), _ptr(ws), C.c_size_t(ws.numel()),
                               _stream(stream)), "gs_preprocess")


def gs_render_forward(params: GsParams, cams, ws: torch.Tensor, bg, out_rgb: torch.Tensor,
                      out_T: torch.Tensor | None = None, stream=None):
    ca = camera_struct(cams)
    bga = (C.c_float * 3)(*[float(x) for x in bg])
    _check(lib().gs_render_forward(C.byref(params), ca, C.c_int32(len(ca)), _ptr(ws), C.c_size_t(ws.numel()), bga,
                                   _ptr(out_rgb), _ptr(out_T), _stream(stream)), "gs_render_forward")


def gs_loss_workspace_size(V, H, W) -> int:
    b = C.c_size_t()
    _check(lib().gs_loss_workspace_size(C.c_int32(V), C.c_int32(H), C.c_int32(W), C.byref(b)),
           "gs_loss_workspace_size")
    return b.value


def gs_photometric_loss(render: torch.Tensor, gt: torch.Tensor, lam: float, loss: torch.Tensor,
                        dL: torch.Tensor | None, ws: torch.Tensor, stream=None):
    if render.shape != gt.shape or render.dim() != 4 or render.shape[1] != 3:
        raise GsError(GS_ERR_SHAPE, "gs_photometric_loss (DimensionMismatch)")
    V, _, H, W = render.shape
    _check(lib().gs_photometric_loss(_ptr(render), _ptr(gt), C.c_int32(V), C.c_int32(H), C.c_int32(W),
                                     C.c_float(lam), _ptr(loss), _ptr(dL), _ptr(ws), C.c_size_t(ws.numel()),
                                     _stream(stream)), "gs_photometric_loss")


def gs_render_backward(params: GsParams, cams, ws: torch.Tensor, bg, dL_drgb: torch.Tensor, grads: torch.Tensor,
                       grad2d_norm: torch.Tensor | None = None, stream=None):
    ca = camera_struct(cams)
    bga = (C.c_float * 3)(*[float(x) for x in bg])
    _check(lib().gs_render_backward(C.byref(params), ca, C.c_int32(len(ca)), _ptr(ws), C.c_size_t(ws.numel()), bga,
                                    _ptr(dL_drgb), _ptr(grads), _ptr(grad2d_norm), _stream(stream)),
           "gs_render_backward")


def gs_render_backward_adam(params: GsParams, cams, ws: torch.Tensor, bg, dL_drgb: torch.Tensor, m, v,
                            hp: GsAdamHparams, step: int, grad2d_norm: torch.Tensor | None = None, stream=None,
                            step_dev: torch.Tensor | None = None):
    """step > 0: host step number; step == 0: device int64 counter step_dev (graph replay)."""
    ca = camera_struct(cams)
    bga = (C.c_float * 3)(*[float(x) for x in bg])
    _check(lib().gs_render_backward_adam(C.byref(params), ca, C.c_int32(len(ca)), _ptr(ws), C.c_size_t(ws.numel()),
                                         bga, _ptr(dL_drgb), _ptr(m), _ptr(v), C.byref(hp), C.c_int64(step),
                                         _ptr(step_dev), _ptr(grad2d_norm), _stream(stream)),
           "gs_render_backward_adam")


def gs_pyramid(img: torch.Tensor, n_levels: int, out: torch.Tensor, stream=None):
    """img [N, C, H, W]; out: flat float32 buffer for levels 1..n."""
    N, Cc, H, W = img.shape
    _check(lib().gs_pyramid(_ptr(img), C.c_int32(N), C.c_int32(Cc), C.c_int32(H), C.c_int32(W),
                            C.c_int32(n_levels), _ptr(out), _stream(stream)), "gs_pyramid")


def gs_adam_step(params: GsParams, grads, m, v, hp: GsAdamHparams, step: int, g_begin: int, g_end: int,
                 zero_grads: bool, stream=None):
    _check(lib().gs_adam_step(C.byref(params), _ptr(grads), _ptr(m), _ptr(v), C.byref(hp), C.c_int64(step),
                              C.c_int64(g_begin), C.c_int64(g_end), C.c_int32(int(zero_grads)), _stream(stream)),
           "gs_adam_step")


def gs_adam_step_rows(params: GsParams, grads, m_rows, v_rows, hp: GsAdamHparams, step: int, row_begin: int,
                      row_end: int, zero_grads: bool, stream=None):
    _check(lib().gs_adam_step_rows(C.byref(params), _ptr(grads), _ptr(m_rows), _ptr(v_rows), C.byref(hp),
                                   C.c_int64(step), C.c_int32(row_begin), C.c_int32(row_end),
                                   C.c_int32(int(zero_grads)), _stream(stream)), "gs_adam_step_rows")


def gs_adam_step_rows_dev(params: GsParams, grads, m_rows, v_rows, hp: GsAdamHparams, step_dev, row_begin: int,
                          row_end: int, zero_grads: bool, stream=None):
    _check(lib().gs_adam_step_rows_dev(C.byref(params), _ptr(grads), _ptr(m_rows), _ptr(v_rows), C.byref(hp),
                                       _ptr(step_dev), C.c_int32(row_begin), C.c_int32(row_end),
                                       C.c_int32(int(zero_grads)), _stream(stream)), "gs_adam_step_rows_dev")


def gs_comm_shard(n: int, sh_degree: int, rank: int, world: int) -> tuple[int, int]:
    e0, e1 = C.c_int64(), C.c_int64()
    _check(lib().gs_comm_shard(C.c_int64(n), C.c_int32(sh_degree), C.c_int32(rank), C.c_int32(world),
                               C.byref(e0), C.byref(e1)), "gs_comm_shard")
    return e0.value, e1.value


def _ptr_array(ptrs) -> C.Array:
    return (C.c_void_p * len(ptrs))(*[C.c_void_p(int(p)) for p in ptrs])


def gs_peer_barrier(flag_ptrs, rank: int, world: int, epoch: torch.Tensor, step_dev: torch.Tensor | None,
                    stream=None):
    """flag_ptrs: `world` device addresses (ints) of each rank's uint32[world] flags."""
    _check(lib().gs_peer_barrier(_ptr_array(flag_ptrs), C.c_int32(rank), C.c_int32(world), _ptr(epoch),
                                 _ptr(step_dev), _stream(stream)), "gs_peer_barrier")


def gs_reduce_adam_bcast(params: GsParams, param_ptrs, grad_ptrs, param_mc: int, grad_mc: int, m_shard, v_shard,
                         hp: GsAdamHparams, step: int, step_dev: torch.Tensor | None, rank: int, world: int,
                         stream=None):
    """param_ptrs / grad_ptrs: `world` device addresses (ints); param_mc / grad_mc: multicast
    addresses or 0."""
    _check(lib().gs_reduce_adam_bcast(C.byref(params), _ptr_array(param_ptrs), _ptr_array(grad_ptrs),
                                      C.c_void_p(param_mc or None), C.c_void_p(grad_mc or None), _ptr(m_shard),
                                      _ptr(v_shard), C.byref(hp), C.c_int64(step), _ptr(step_dev), C.c_int32(rank),
                                      C.c_int32(world), _stream(stream)), "gs_reduce_adam_bcast")


def gs_densify_temp_size(n: int) -> int:
    b = C.c_size_t()
    _check(lib().gs_densify_temp_size(C.c_int64(n), C.byref(b)), "gs_densify_temp_size")
    return b.value


def gs_densify_stats(params: GsParams, cams, ws: torch.Tensor, vis_count: torch.Tensor, max_radius: torch.Tensor,
                     stream=None):
    ca = camera_struct(cams)
    _check(lib().gs_densify_stats(C.byref(params), ca, C.c_int32(len(ca)), _ptr(ws), C.c_size_t(ws.numel()),
                                  _ptr(vis_count), _ptr(max_radius), _stream(stream)), "gs_densify_stats")


def gs_densify_plan(params: GsParams, grad_accum, vis_count, max_radius, cfg: GsDensifyCfg, temp: torch.Tensor,
                    stream=None) -> tuple:
    """-> (n_clone, n_split, n_prune, n_new); synchronises the stream."""
    counts = (C.c_int64 * 4)()
    _check(lib().gs_densify_plan(C.byref(params), _ptr(grad_accum), _ptr(vis_count), _ptr(max_radius), C.byref(cfg),
                                 _ptr(temp), C.c_size_t(temp.numel()), counts, _stream(stream)), "gs_densify_plan")
    return tuple(int(x) for x in counts)


def gs_densify_apply(params: GsParams, m, v, z: torch.Tensor, temp: torch.Tensor, out: GsParams, out_m, out_v,
                     stream=None):
    _check(lib().gs_densify_apply(C.byref(params), _ptr(m), _ptr(v), _ptr(z), _ptr(temp), C.c_size_t(temp.numel()),
                                  C.byref(out), _ptr(out_m), _ptr(out_v), _stream(stream)), "gs_densify_apply")


def gs_densify_tags(n: int, temp: torch.Tensor, tags_in: torch.Tensor, tags_out: torch.Tensor, stream=None):
    _check(lib().gs_densify_tags(C.c_int64(n), _ptr(temp), C.c_size_t(temp.numel()), _ptr(tags_in), _ptr(tags_out),
                                 _stream(stream)), "gs_densify_tags")


def gs_geometry_densify(cam, uv: torch.Tensor, active: torch.Tensor, kp_depth, depth_map, image: torch.Tensor,
                        mode: int, rho: float, out: GsParams, src: torch.Tensor, count: torch.Tensor, stream=None):
    ca = camera_struct([cam])
    _check(lib().gs_geometry_densify(ca, _ptr(uv), _ptr(active), _ptr(kp_depth), _ptr(depth_map), _ptr(image),
                                     C.c_int32(uv.shape[0]), C.c_int32(mode), C.c_float(rho), C.byref(out),
                                     _ptr(src), _ptr(count), _stream(stream)), "gs_geometry_densify")


def gs_query_status(ws: torch.Tensor, stream=None):
    """Synchronises the stream; returns (status, flags, pairs)."""
    f = C.c_int32()
    p = C.c_int64()
    s = lib().gs_query_status(_ptr(ws), C.c_size_t(ws.numel()), _stream(stream), C.byref(f), C.byref(p))
    return s, f.value, p.value


def gs_status_async(ws: torch.Tensor, dst: torch.Tensor, stream=None):
    """Enqueue {flags, pairs} of the workspace into dst (int32[2], device or pinned host)."""
    if dst.dtype != torch.int32 or dst.numel() < 2 or not dst.is_contiguous():
        raise ValueError("dst must be a contiguous int32 tensor of >= 2 elements")
    if not dst.is_cuda and not dst.is_pinned():
        raise ValueError("dst must be device or pinned host memory")
    _check(lib().gs_status_async(_ptr(ws), C.c_size_t(ws.numel()), C.c_void_p(dst.data_ptr()), _stream(stream)),
           "gs_status_async")


def gs_workspace_release(ws: torch.Tensor):
    _check(lib().gs_workspace_release(C.c_void_p(ws.data_ptr())), "gs_workspace_release")


def gs_spatial_order_temp_size(n) -> int:
    b = C.c_size_t()
    _check(lib().gs_spatial_order_temp_size(C.c_int64(n), C.byref(b)), "gs_spatial_order_temp_size")
    return b.value


def gs_spatial_order(params: GsParams, perm: torch.Tensor, temp: torch.Tensor, stream=None):
    _check(lib().gs_spatial_order(C.byref(params), _ptr(perm), _ptr(temp), C.c_size_t(temp.numel()),
                                  _stream(stream)), "gs_spatial_order")


def gs_permute_columns(src: torch.Tensor, dst: torch.Tensor, ld: int, rows: int, n: int, perm: torch.Tensor,
                       stream=None):
    _check(lib().gs_permute_columns(_ptr(src), _ptr(dst), C.c_int64(ld), C.c_int32(rows), C.c_int64(n), _ptr(perm),
                                    _stream(stream)), "gs_permute_columns")


def gs_sort_temp_size(n, key_bits) -> int:
    b = C.c_size_t()
    _check(lib().gs_sort_temp_size(C.c_int64(n), C.c_int32(key_bits), C.byref(b)), "gs_sort_temp_size")
    return b.value


def gs_debug_sort_pairs(keys, vals, keys_alt, vals_alt, key_bits, temp, stream=None):
    _check(lib().gs_debug_sort_pairs(_ptr(keys), _ptr(vals), _ptr(keys_alt), _ptr(vals_alt),
                                     C.c_int64(keys.numel()), C.c_int32(key_bits), _ptr(temp),
                                     C.c_size_t(temp.numel()), _stream(stream)), "gs_debug_sort_pairs")


def gs_debug_workspace_view(ws, n, n_views, width, height) -> GsWsView:
    out = GsWsView()
    _check(lib().gs_debug_workspace_view(_ptr(ws), C.c_size_t(ws.numel()), C.c_int64(n), C.c_int32(n_views),
                                         C.c_int32(width), C.c_int32(height), C.byref(out)),
           "gs_debug_workspace_view")
    return out


def gs_set_render_stats(on: bool):
    """Diagnostic composited counts in the forward (n_composited); off by default."""
    _check(lib().gs_set_render_stats(C.c_int32(int(bool(on)))), "gs_set_render_stats")


def gs_set_binning(mode: int):
    """0 = tile buckets + in-tile sort (default), 1 = global onesweep LSD radix sort."""
    _check(lib().gs_set_binning(C.c_int32(mode)), "gs_set_binning")


def gs_profile_kernel(name: str | None):
    _check(lib().gs_profile_kernel(name.encode() if name else None), "gs_profile_kernel")


def gs_profile_read():
    """(total_ms, launches) of the profiled kernel since gs_profile_kernel; synchronises."""
    ms = C.c_double()
    n = C.c_int64()
    _check(lib().gs_profile_read(C.byref(ms), C.byref(n)), "gs_profile_read")
    return ms.value, n.value


def gs_debug_exp_scale(s: torch.Tensor, out: torch.Tensor, stream=None):
    _check(lib().gs_debug_exp_scale(_ptr(s), _ptr(out), C.c_int64(s.numel()), _stream(stream)),
           "gs_debug_exp_scale")
