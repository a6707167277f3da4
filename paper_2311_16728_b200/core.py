"""Torch-facing wrappers of the libgs.so entry points: parameter packing, workspaces and the
five stages of the path.  PyTorch only allocates device memory and provides streams; every
number is computed by the CUDA kernels behind include/gs.h."""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L

CLASS_ROWS = {"means": (0, 3), "quats": (3, 7), "log_scales": (7, 10), "opacity_logits": (10, 11)}


def param_rows(sh_degree: int) -> int:
    return 11 + 3 * (sh_degree + 1) ** 2


def pack_params(scene, device="cuda", ld: int | None = None) -> torch.Tensor:
    """Per-class arrays (synth.Scene) -> float32 [K, ld] structure-of-arrays (gs.h layout)."""
    n = scene.means.shape[0]
    D = int(round(math.sqrt(scene.sh.shape[1]))) - 1
    K = param_rows(D)
    ld = ld or ((n + 63) // 64) * 64
    host = np.zeros((K, ld), np.float32)
    host[0:3, :n] = scene.means.T
    host[3:7, :n] = scene.quats.T
    host[7:10, :n] = scene.log_scales.T
    host[10, :n] = scene.opacity_logits
    # SH coefficient-major: row 11 + 3 l + c
    host[11:, :n] = scene.sh.reshape(n, -1).T
    return torch.from_numpy(host).to(device)


def unpack(t: torch.Tensor, n: int, sh_degree: int) -> dict:
    """[K, ld] tensor (params, grads or moments) -> per-class numpy arrays like synth.Scene."""
    a = t.detach().float().cpu().numpy()[:, :n]
    NC = (sh_degree + 1) ** 2
    return dict(means=a[0:3].T.copy(), quats=a[3:7].T.copy(), log_scales=a[7:10].T.copy(),
                opacity_logits=a[10].copy(), sh=a[11:].T.reshape(n, NC, 3).copy())


class Workspace:
    """Render workspace of one (n, views, width, height, capacity) configuration."""

    def __init__(self, n: int, n_views: int, width: int, height: int, pair_capacity: int, device="cuda"):
        self.n, self.V, self.W, self.H = n, n_views, width, height
        self.capacity = pair_capacity
        self.bytes = L.gs_workspace_size(n, n_views, width, height, pair_capacity)
        self.buf = torch.empty(self.bytes, dtype=torch.uint8, device=device)
        self.tiles_x = (width + L.GS_TILE - 1) // L.GS_TILE
        self.tiles_y = (height + L.GS_TILE - 1) // L.GS_TILE

    # ---- debug views (bit-exact comparisons) ----
    def _slice(self, ptr: int, count: int, dtype: torch.dtype) -> torch.Tensor:
        off = ptr - self.buf.data_ptr()
        nbytes = count * torch.empty((), dtype=dtype).element_size()
        return self.buf[off:off + nbytes].view(dtype)

    def views(self) -> dict:
        v = L.gs_debug_workspace_view(self.buf, self.n, self.V, self.W, self.H)
        M = self.n * self.V
        tiles = self.tiles_x * self.tiles_y * self.V
        rec0 = self._slice(v.rec0, 4 * M, torch.float32).view(M, 4)
        rec1 = self._slice(v.rec1, 4 * M, torch.float32).view(M, 4)
        rec2 = self._slice(v.rec2, 4 * M, torch.float32).view(M, 4)
        return dict(mean2d=rec0[:, 0:2], conic=torch.stack([rec0[:, 2], rec0[:, 3], rec1[:, 0]], 1),
                    sigma=rec1[:, 1], rgb=torch.stack([rec1[:, 2], rec1[:, 3], rec2[:, 0]], 1), extent=rec2[:, 1:3],
                    depth=self._slice(v.depth, M, torch.float32),
                    radius=self._slice(v.radius, M, torch.int32),
                    rect=self._slice(v.rect, 4 * M, torch.int32).view(M, 4),
                    tiles_touched=self._slice(v.tiles_touched, M, torch.int32),
                    offsets=self._slice(v.offsets, M, torch.int32),
                    keys=self._slice(v.keys, v.capacity, torch.int64),
                    vals=self._slice(v.vals, v.capacity, torch.int32),
                    ranges=self._slice(v.ranges, 2 * tiles, torch.int32).view(tiles, 2),
                    n_contrib=self._slice(v.n_contrib, self.V * self.H * self.W, torch.int32),
                    n_composited=self._slice(v.n_composited, self.V * self.H * self.W, torch.int32))

    def status(self):
        """(status, flags, pairs) -- synchronises the current stream."""
        return L.gs_query_status(self.buf)

    def __del__(self):
        # the library's forward-state token is keyed by the buffer address, which the caching
        # allocator may hand to the next workspace: forget it with the buffer
        try:
            if getattr(self, "buf", None) is not None:
                L.gs_workspace_release(self.buf)
        except Exception:
            pass


class Renderer:
    """A1-A6 forward and A8-A9 backward over one workspace."""

    def __init__(self, n: int, sh_degree: int, n_views: int, width: int, height: int, pair_capacity: int,
                 device="cuda"):
        self.n, self.D = n, sh_degree
        self.ws = Workspace(n, n_views, width, height, pair_capacity, device)
        self.V, self.W, self.H = n_views, width, height
        self.rgb = torch.empty((n_views, 3, height, width), dtype=torch.float32, device=device)
        self.T = torch.empty((n_views, height, width), dtype=torch.float32, device=device)

    def forward(self, params: torch.Tensor, cams, bg=(0.0, 0.0, 0.0)):
        ps = L.params_struct(params, self.n, self.D)
        L.gs_preprocess(ps, cams, self.ws.buf)
        L.gs_render_forward(ps, cams, self.ws.buf, bg, self.rgb, self.T)
        return self.rgb, self.T

    def backward(self, params: torch.Tensor, cams, dL_drgb: torch.Tensor, grads: torch.Tensor,
                 grad2d_norm: torch.Tensor | None = None, bg=(0.0, 0.0, 0.0)):
        ps = L.params_struct(params, self.n, self.D)
        L.gs_render_backward(ps, cams, self.ws.buf, bg, dL_drgb, grads, grad2d_norm)
        return grads

    def backward_adam(self, params: torch.Tensor, cams, dL_drgb: torch.Tensor, opt: "Adam",
                      grad2d_norm: torch.Tensor | None = None, bg=(0.0, 0.0, 0.0)):
        """A8 + A9 + A11 fused (single GPU): backward and the optimiser step without a gradient array.
        With opt.device_step the step counter lives on the device (CUDA-graph replay)."""
        ps = L.params_struct(params, self.n, self.D)
        if opt.device_step:
            L.gs_render_backward_adam(ps, cams, self.ws.buf, bg, dL_drgb, opt.m, opt.v, opt.hp, 0, grad2d_norm,
                                      step_dev=opt.t_dev)
        else:
            opt.t += 1
            L.gs_render_backward_adam(ps, cams, self.ws.buf, bg, dL_drgb, opt.m, opt.v, opt.hp, opt.t, grad2d_norm)


class PhotometricLoss:
    """A7 for V images of H x W (Eq. 4)."""

    def __init__(self, V: int, H: int, W: int, lam: float = 0.2, device="cuda"):
        self.V, self.H, self.W, self.lam = V, H, W, lam
        self.ws = torch.empty(L.gs_loss_workspace_size(V, H, W), dtype=torch.uint8, device=device)
        self.loss = torch.empty(V, dtype=torch.float32, device=device)
        self.dL = torch.empty((V, 3, H, W), dtype=torch.float32, device=device)

    def __call__(self, render: torch.Tensor, gt: torch.Tensor, grad: bool = True):
        L.gs_photometric_loss(render, gt, self.lam, self.loss, self.dL if grad else None, self.ws)
        return self.loss, (self.dL if grad else None)


def level_shapes(H: int, W: int, n_levels: int):
    shapes = [(H, W)]
    for _ in range(n_levels):
        H, W = (H + 1) // 2, (W + 1) // 2
        shapes.append((H, W))
    return shapes


def gaussian_pyramid(img: torch.Tensor, n_levels: int) -> list:
    """A0: levels 0..n of [N, C, H, W] images (level 0 is the input itself)."""
    N, Cc, H, W = img.shape
    shapes = level_shapes(H, W, n_levels)
    sizes = [N * Cc * h * w for (h, w) in shapes[1:]]
    out = torch.empty(max(sum(sizes), 1), dtype=torch.float32, device=img.device)
    L.gs_pyramid(img, n_levels, out)
    levels, o = [img], 0
    for (h, w), s in zip(shapes[1:], sizes):
        levels.append(out[o:o + s].view(N, Cc, h, w))
        o += s
    return levels


@dataclass
class AdamConfig:
    """Per-class fixed learning rates (R20 -- 3DGS-calibrated defaults)."""
    lr_means: float = 1.6e-4
    lr_quats: float = 1e-3
    lr_log_scales: float = 5e-3
    lr_opacity: float = 5e-2
    lr_sh_dc: float = 2.5e-3
    lr_sh_rest: float = 1.25e-4
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-15
    sgd: bool = False
    scene_extent: float = 1.0

    def struct(self) -> L.GsAdamHparams:
        hp = L.GsAdamHparams()
        hp.lr[:] = [self.lr_means * self.scene_extent, self.lr_quats, self.lr_log_scales, self.lr_opacity,
                    self.lr_sh_dc, self.lr_sh_rest]
        hp.beta1, hp.beta2, hp.eps, hp.sgd_mode = self.beta1, self.beta2, self.eps, int(self.sgd)
        return hp


class Adam:
    """A11: fused Adam over the whole [K, ld] parameter buffer (or a Gaussian shard)."""

    def __init__(self, params: torch.Tensor, n: int, sh_degree: int, cfg: AdamConfig | None = None):
        self.params, self.n, self.D = params, n, sh_degree
        self.cfg = cfg or AdamConfig()
        self.hp = self.cfg.struct()
        self.m = torch.zeros_like(params)
        self.v = torch.zeros_like(params)
        self.t = 0
        self.device_step = False  # True: fused steps count on the device (t_dev), for graph replay
        self.t_dev = torch.zeros(1, dtype=torch.int64, device=params.device)

    def use_device_step(self):
        """Switch the fused backward+Adam to the device-resident step counter (keeps the count;
        a no-op once switched)."""
        if not self.device_step:
            self.t_dev.fill_(self.t)
        self.device_step = True

    def step(self, grads: torch.Tensor, zero_grads: bool = True, g_begin: int = 0, g_end: int | None = None):
        self.t += 1
        ps = L.params_struct(self.params, self.n, self.D)
        L.gs_adam_step(ps, grads, self.m, self.v, self.hp, self.t, g_begin, self.n if g_end is None else g_end,
                       zero_grads)


@dataclass
class DensifyConfig:
    """Densify-and-prune hyper-parameters (R27-R30)."""
    grad_threshold: float = 2e-4   # mean ||dL/dmean2d|| in pixels
    percent_dense: float = 0.01    # "large" above 1 % of the scene extent (SPEC)
    scene_extent: float = 1.0
    opacity_threshold: float = 0.005
    max_screen_frac: float = 0.5   # prune a pixel radius above this fraction of max(W, H)

    def struct(self, width: int, height: int) -> L.GsDensifyCfg:
        c = L.GsDensifyCfg()
        c.grad_threshold, c.percent_dense, c.scene_extent = self.grad_threshold, self.percent_dense, self.scene_extent
        c.opacity_threshold = self.opacity_threshold
        c.max_screen_px = int(self.max_screen_frac * max(width, height))
        return c


def densify(params: torch.Tensor, n: int, sh_degree: int, m, v, grad_accum: torch.Tensor, vis_count: torch.Tensor,
            max_radius: torch.Tensor, z: torch.Tensor, cfg: L.GsDensifyCfg, tags: torch.Tensor | None = None):
    """SURVEY f1 densify and prune: returns (new params [K, ld'], new m, new v, counts[, new tags]) with
    counts = (n_clone, n_split, n_prune, n_new).  m, v may be None (no optimiser state); tags: an
    optional per-Gaussian uint8 tensor carried to the new map."""
    ps = L.params_struct(params, n, sh_degree)
    temp = torch.empty(max(L.gs_densify_temp_size(n), 1), dtype=torch.uint8, device=params.device)
    counts = L.gs_densify_plan(ps, grad_accum, vis_count, max_radius, cfg, temp)
    nn = counts[3]
    out = torch.zeros((param_rows(sh_degree), L.param_ld(max(nn, 1))), dtype=torch.float32, device=params.device)
    om = torch.zeros_like(out) if m is not None else None
    ov = torch.zeros_like(out) if v is not None else None
    L.gs_densify_apply(ps, m, v, z, temp, L.params_struct(out, nn, sh_degree), om, ov)
    if tags is None:
        return out, om, ov, counts
    new_tags = torch.zeros(max(nn, 1), dtype=torch.uint8, device=params.device)
    L.gs_densify_tags(n, temp, tags, new_tags)
    return out, om, ov, counts, new_tags


def geometry_densify(cam, uv: torch.Tensor, active: torch.Tensor, kp_depth, depth_map, image: torch.Tensor,
                     mode: int, sh_degree: int, rho: float = 100.0):
    """new temporary primitives for the inactive keypoints of one
    keyframe.  Returns (params [K, ld] with `count` valid columns, count, src keypoint indices)."""
    nk = int(uv.shape[0])
    dev = uv.device
    out = torch.zeros((param_rows(sh_degree), L.param_ld(max(nk, 1))), dtype=torch.float32, device=dev)
    src = torch.zeros(max(nk, 1), dtype=torch.int32, device=dev)
    count = torch.zeros(1, dtype=torch.int32, device=dev)
    L.gs_geometry_densify(cam, uv, active, kp_depth, depth_map, image, mode, rho,
                          L.params_struct(out, nk, sh_degree), src, count)
    c = int(count.item())
    return out, c, src[:c]


def spatial_order(params: torch.Tensor, n: int, sh_degree: int) -> torch.Tensor:
    """Map layout (gs_spatial_order): int32 [n] device perm, perm[k] = index of the Gaussian
    that goes to position k (ascending Morton code of its mean)."""
    perm = torch.empty(max(n, 1), dtype=torch.int32, device=params.device)
    temp = torch.empty(L.gs_spatial_order_temp_size(n), dtype=torch.uint8, device=params.device)
    L.gs_spatial_order(L.params_struct(params, n, sh_degree), perm, temp)
    return perm[:n]


def permute_columns(t: torch.Tensor, perm: torch.Tensor, n: int) -> torch.Tensor:
    """New tensor with column k = column perm[k] of t for k < n (gs_permute_columns); t is
    [rows, ld] (parameter layout, Adam moments) or [>= n] (per-Gaussian array, 4-byte dtype)."""
    out = t.clone() if t.shape[-1] > n else torch.empty_like(t)  # columns >= n (padding) stay as they were
    rows = 1 if t.dim() == 1 else t.shape[0]
    ld = t.shape[-1]
    if t.element_size() != 4:
        raise ValueError("4-byte element type required")
    L.gs_permute_columns(t.view(torch.float32) if t.dtype != torch.float32 else t,
                         out.view(torch.float32) if out.dtype != torch.float32 else out, ld, rows, n, perm)
    return out
