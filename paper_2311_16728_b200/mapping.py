"""Photorealistic-mapping driver: Gaussian-pyramid schedule (Eq. 5), one mapping iteration
per level (render -> loss -> backward -> [all-reduce] -> Adam), keyframe-batch data
parallelism over torch.distributed (NCCL).  Host logic only; every stage is a libgs.so call.
"""
from __future__ import annotations

import math

import numpy as np
import torch
import torch.distributed as dist

from . import _lib as L
from .core import (Adam, AdamConfig, DensifyConfig, PhotometricLoss, Renderer, densify, gaussian_pyramid,
                   geometry_densify, level_shapes, pack_params, permute_columns)
from .core import spatial_order as core_spatial_order
from .levels import densify_samples, level_camera


def gp_level(iteration: int, n_levels: int, iters_per_level: int) -> int:
    """Eq. 5: start at the top level n, step down every iters_per_level
    iterations, stay at 0 (SPEC.md:443-451 gp_level; R21/R26)."""
    if iteration < 0 or n_levels < 0 or iters_per_level <= 0:
        raise ValueError("gp_level: iteration >= 0, n >= 0, iters_per_level > 0")
    return max(0, n_levels - iteration // iters_per_level)


def shard_views(n_views: int, rank: int, world: int) -> list[int]:
    """Keyframe-batch partition: rank g takes views g, g+G, ..."""
    return list(range(rank, n_views, world))


def reduce_gradients(grads: torch.Tensor, group=None) -> torch.Tensor:
    """A10: sum of the per-rank gradients (R22) -- the only exchange step of the path."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(grads, op=dist.ReduceOp.SUM, group=group)
    return grads


def row_shard(K: int, rank: int, world: int) -> tuple[int, int, int]:
    """Parameter-row shard of the [K][ld] layout for the sharded optimiser:
    R = ceil(K / world) rows per rank (the buffer is padded to world * R rows so that every
    rank's rows are one contiguous, equally sized collective chunk); rank g owns rows
    [g R, min(K, (g + 1) R)).  Returns (R, row_begin, row_end)."""
    R = -(-K // world)
    return R, min(K, rank * R), min(K, (rank + 1) * R)


def _backend(group) -> str:
    return dist.get_backend(group)


def reduce_scatter_rows(buf: torch.Tensor, R: int, group=None) -> torch.Tensor:
    """A10 (sharded): after the call rows [g R, (g + 1) R) of the padded [world R][ld] buffer hold
    the sum over ranks (in-place NCCL reduce-scatter; other rows are left unspecified)."""
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    mine = buf[rank * R:(rank + 1) * R]
    if _backend(group) == "nccl":
        dist.reduce_scatter_tensor(mine, buf, op=dist.ReduceOp.SUM, group=group)
    else:  # gloo has no reduce-scatter: the same sums through an all-reduce
        dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
    return mine


def all_gather_rows(buf: torch.Tensor, R: int, group=None) -> torch.Tensor:
    """Every rank's rows [g R, (g + 1) R) of the padded buffer to every rank (in place)."""
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    mine = buf[rank * R:(rank + 1) * R]
    if _backend(group) == "nccl":
        dist.all_gather_into_tensor(buf, mine, group=group)
    else:
        dist.all_gather(list(buf.chunk(world)), mine.clone(), group=group)
    return buf


class ShardedAdam:
    """A11 sharded by parameter rows (SURVEY §8(e) extension f3): reduce-scatter of the gradient
    rows, Adam on this rank's rows only (gs_adam_step_rows; m and v exist for those rows only,
    1/world of the optimiser state), all-gather of the updated parameter rows.  Same NVLink volume
    as the all-reduce, 1/world of the Adam bytes.  `params` / `grads` are the first K rows of
    padded [world R][ld] buffers (`padded_params`, `padded_grads`).

    The backward ADDS into `grads` (gs.h gs_render_backward), so after a step the whole padded
    gradient buffer is zeroed: the reduce-scatter leaves partial or summed gradients in the rows
    other ranks own, and re-adding them next iteration would apply stale gradient."""

    def __init__(self, padded_params: torch.Tensor, padded_grads: torch.Tensor, n: int, sh_degree: int,
                 cfg: AdamConfig | None = None, group=None):
        from .core import param_rows
        self.group = group
        self.world, self.rank = dist.get_world_size(group), dist.get_rank(group)
        self.K = param_rows(sh_degree)
        self.R, self.r0, self.r1 = row_shard(self.K, self.rank, self.world)
        self.n, self.D = n, sh_degree
        self.cfg = cfg or AdamConfig()
        self.hp = self.cfg.struct()
        self._t = 0
        self.device_step = False  # True: the step counter lives on the device (CUDA-graph replay)
        self.t_dev = torch.zeros(1, dtype=torch.int64, device=padded_params.device)
        self.rebind(padded_params, padded_grads, n)

    @property
    def t(self) -> int:
        return int(self.t_dev.item()) if self.device_step else self._t

    def use_device_step(self):
        """Count steps on the device (gs_adam_step_rows_dev), so a captured step replays with the
        right bias corrections; keeps the count."""
        if not self.device_step:
            self.t_dev.fill_(self._t)
        self.device_step = True

    def rebind(self, padded_params: torch.Tensor, padded_grads: torch.Tensor, n: int,
               m_full: torch.Tensor | None = None, v_full: torch.Tensor | None = None):
        """New parameter / gradient buffers (after densification); m_full / v_full: the full
        [>= K][ld] moments of the new map (every rank passes the same), of which this rank keeps
        its rows; None = zero moments."""
        assert padded_params.shape[0] == self.world * self.R and padded_grads.shape == padded_params.shape
        self.padded_params, self.padded_grads = padded_params, padded_grads
        self.params, self.grads = padded_params[:self.K], padded_grads[:self.K]
        self.n = n
        ld = padded_params.shape[1]
        # R rows (not r1 - r0): every rank's moment chunk has the same size for full_state()'s gather
        self.m = torch.zeros((self.R, ld), dtype=torch.float32, device=padded_params.device)
        self.v = torch.zeros_like(self.m)
        for mine, full in ((self.m, m_full), (self.v, v_full)):
            if full is not None and self.r1 > self.r0:
                mine[:self.r1 - self.r0] = full[self.r0:self.r1]

    def full_state(self) -> tuple:
        """All-gather of the moment rows: (m, v) as [world R][ld] tensors, rows [0, K) valid --
        what densification needs to move the optimiser state with its Gaussians."""
        out = []
        for mine in (self.m, self.v):
            full = torch.zeros((self.world * self.R, mine.shape[1]), dtype=mine.dtype, device=mine.device)
            full[self.rank * self.R:(self.rank + 1) * self.R] = mine
            all_gather_rows(full, self.R, self.group)
            out.append(full)
        return tuple(out)

    def _adam_rows(self):
        from . import _lib as L
        ps = L.params_struct(self.params, self.n, self.D)
        if self.device_step:
            L.gs_adam_step_rows_dev(ps, self.grads, self.m, self.v, self.hp, self.t_dev, self.r0, self.r1, False)
        else:
            L.gs_adam_step_rows(ps, self.grads, self.m, self.v, self.hp, self._t, self.r0, self.r1, False)

    def step(self):
        reduce_scatter_rows(self.padded_grads, self.R, self.group)   # A10
        if not self.device_step:
            self._t += 1
        if self.r1 > self.r0:
            self._adam_rows()                                          # A11 on this rank's rows
        all_gather_rows(self.padded_params, self.R, self.group)       # replicas identical again
        self.padded_grads.zero_()                                      # no row may carry into the next +=


class MappingEngine:
    """Optimises one Gaussian map against the keyframes of this rank.

    scene: synth.Scene (initial parameters); cams: this rank's keyframe cameras (level 0);
    gts: [V, 3, H, W] level-0 targets (numpy or torch); n_levels: top pyramid level n (n=2,
    PAPER.md:568)."""

    def __init__(self, scene, cams, gts, n_levels: int = 2, lam: float = 0.2, adam: AdamConfig | None = None,
                 device: str = "cuda", capacity_margin: float = 1.3, group=None, bg=(0.0, 0.0, 0.0),
                 shard_optimizer: bool = True, densify_cfg: DensifyConfig | None = None,
                 spatial_order: bool = True, comm: str = "nccl"):
        self.device = device
        self.n = scene.means.shape[0]
        self.D = int(round(math.sqrt(scene.sh.shape[1]))) - 1
        self.group = group
        packed = pack_params(scene, device)
        # map layout (order.cu): Gaussians in Morton order of their means, so that the ones that
        # land on the same tiles are neighbours in memory.  order[k] = index in `scene` of the
        # Gaussian at position k (None once densification has changed the map).  Every rank
        # computes the same permutation from the same parameters.
        self.spatial_order = spatial_order
        self.order = None
        if spatial_order and self.n > 0:
            perm = core_spatial_order(packed, self.n, self.D)
            packed = permute_columns(packed, perm, self.n)
            self.order = perm.to(torch.int64)
        self.sharded = None
        self.peer = None
        self._pipe = None
        self._status = None
        self.graph = None
        self.adam_cfg = adam
        if comm not in ("nccl", "peer"):
            raise ValueError("comm: 'nccl' (collectives) or 'peer' (fused kernel over peer memory)")
        if comm == "peer" and dist.is_available() and dist.is_initialized():
            # A10 + A11 as one kernel over symmetric peer memory (comm.py, gs_reduce_adam_bcast)
            from .comm import PeerAdam
            self.peer = PeerAdam(self.n, self.D, adam, group, device)
            self.peer.params[:, :packed.shape[1]] = packed
            self.params, self.grads = self.peer.params, self.peer.grads
        elif shard_optimizer and dist.is_available() and dist.is_initialized():
            # reduce-scatter -> row-sharded Adam -> all-gather (parameters / gradients live in
            # the first K rows of buffers padded to world x R rows)
            pp = self._padded(packed)
            self.sharded = ShardedAdam(pp, torch.zeros_like(pp), self.n, self.D, adam, group)
            self.params, self.grads = self.sharded.params, self.sharded.grads
        else:
            self.params = packed
            self.grads = torch.zeros_like(self.params)
        self.grad2d_norm = torch.zeros(self.n, dtype=torch.float32, device=device)
        # densification statistics: visible (iteration, view) pairs and max pixel radius
        self.densify_cfg = densify_cfg
        self.vis_count = torch.zeros(self.n, dtype=torch.float32, device=device)
        self.max_radius = torch.zeros(self.n, dtype=torch.int32, device=device)
        # 1 = temporary primitive from geometry-based densification
        self.temporary = torch.zeros(self.n, dtype=torch.uint8, device=device)
        # replicated optimiser state (single GPU / unsharded DP); the sharded one keeps its rows only
        self.adam = Adam(self.params, self.n, self.D, adam) if self.sharded is None and self.peer is None else None
        self.cams0 = list(cams)
        self.V = len(self.cams0)
        self.n_levels = n_levels
        self.lam = lam
        self.bg = bg
        self.group = group
        H, W = self.cams0[0].height, self.cams0[0].width
        self.shapes = level_shapes(H, W, n_levels)
        self.cams = [[level_camera(c, l) for c in self.cams0] for l in range(n_levels + 1)]
        self.gt0 = torch.empty((self.V, 3, H, W), dtype=torch.float32, device=device)
        self.set_keyframes(gts)
        self.losses = [PhotometricLoss(self.V, h, w, lam, device) for (h, w) in self.shapes]
        self.renderers = [None] * (n_levels + 1)
        self.margin = capacity_margin
        self.calibrate()

    # ------------------------------------------------------------------ keyframes / A0
    def set_keyframes(self, gts):
        g = torch.as_tensor(np.asarray(gts, np.float32) if not torch.is_tensor(gts) else gts)
        self.gt0.copy_(g.to(self.device, non_blocking=True).view_as(self.gt0))
        self.build_pyramids()

    def add_keyframe(self, cam, gt):
        """A new keyframe (keyframes reach photorealistic mapping one at a time):
        its level-0 camera and [3, H, W] target join the batch this engine maps; parameters and
        optimiser state carry on; the pyramids, losses and level workspaces are rebuilt, and
        captured graphs (which refer to the old buffers) are dropped."""
        g = torch.as_tensor(np.asarray(gt, np.float32) if not torch.is_tensor(gt) else gt).to(self.device)
        H, W = self.cams0[0].height, self.cams0[0].width
        if (cam.height, cam.width) != (H, W) or tuple(g.shape) != (3, H, W):
            raise ValueError("add_keyframe: camera / target size differs from the engine's keyframes")
        self.cams0.append(cam)
        self.V = len(self.cams0)
        self.cams = [[level_camera(c, l) for c in self.cams0] for l in range(self.n_levels + 1)]
        gt0 = torch.empty((self.V, 3, H, W), dtype=torch.float32, device=self.device)
        gt0[:-1] = self.gt0
        gt0[-1] = g
        self.gt0 = gt0
        self.build_pyramids()
        self.losses = [PhotometricLoss(self.V, h, w, self.lam, self.device) for (h, w) in self.shapes]
        self.renderers = [None] * (self.n_levels + 1)
        self.graph = None
        self._pipe = None
        self.calibrate()
        return self.V - 1

    def build_pyramids(self, overlap: bool = False):
        """A0: GP^l(I_gt), l = 1..n, once per keyframe.  overlap: build them on a
        side stream; the first loss that needs them waits for it (iteration), so the pyramid
        runs concurrently with the first level's projection, binning and rendering."""
        if not overlap or not self.device.startswith("cuda"):
            self.pyr = gaussian_pyramid(self.gt0, self.n_levels)
            self._pyr_pending = False
            return
        if getattr(self, "_side", None) is None:
            self._side = torch.cuda.Stream(device=self.gt0.device)
            self._pyr_event = torch.cuda.Event()
        self._side.wait_stream(torch.cuda.current_stream())  # after the targets' copy
        with torch.cuda.stream(self._side):
            self.pyr = gaussian_pyramid(self.gt0, self.n_levels)
            self._pyr_event.record()
        self._pyr_pending = True

    def _pyramid(self, level: int):
        if getattr(self, "_pyr_pending", False):
            torch.cuda.current_stream().wait_event(self._pyr_event)
            self._pyr_pending = False
        return self.pyr[level]

    # ------------------------------------------------------------------ capacity
    def calibrate(self, min_capacity: int = 1 << 16):
        """Size each level's pair capacity from a measured pair count (one sync, setup only)."""
        for l, (h, w) in enumerate(self.shapes):
            r = self.renderers[l]
            if r is None:
                r = Renderer(self.n, self.D, self.V, w, h, min_capacity, self.device)
            r.forward(self.params, self.cams[l], self.bg)
            st, flags, pairs = r.ws.status()
            need = int(pairs * self.margin) + 4096
            if need > r.ws.capacity or r.ws.capacity > 4 * need:
                r = Renderer(self.n, self.D, self.V, w, h, max(need, min_capacity), self.device)
            self.renderers[l] = r

    def check(self):
        """Synchronises; raises if any level overflowed its pair capacity (then re-calibrate)."""
        for r in self.renderers:
            st, flags, pairs = r.ws.status()
            if flags & 1:
                raise RuntimeError(f"pair capacity exceeded ({pairs} > {r.ws.capacity})")

    # ------------------------------------------------------------------ iteration
    def render(self, level: int = 0):
        return self.renderers[level].forward(self.params, self.cams[level], self.bg)

    def distributed(self) -> bool:
        return dist.is_available() and dist.is_initialized() and dist.get_world_size(self.group) > 1

    def iteration(self, level: int, fused: bool | None = None) -> torch.Tensor:
        """One optimiser step at pyramid level `level` (Eq. 4 against GP^level, R19).  On one GPU
        the backward and Adam run fused (no gradient array); with data parallelism the gradient
        is materialised, all-reduced (A10) and then stepped."""
        r = self.renderers[level]
        cams = self.cams[level]
        rgb, _ = r.forward(self.params, cams, self.bg)                       # A1-A6
        if self._status is not None:  # overflow flag + pair count, read back with the losses
            L.gs_status_async(r.ws.buf, self._status[level])
        if self.densify_cfg is not None:                                     # f1 statistics
            L.gs_densify_stats(L.params_struct(self.params, self.n, self.D), cams, r.ws.buf, self.vis_count,
                               self.max_radius)
        loss, dL = self.losses[level](rgb, self._pyramid(level))             # A7
        if fused is None:
            fused = self.sharded is None and self.peer is None and not self.distributed()
        if fused:
            r.backward_adam(self.params, cams, dL, self.adam, self.grad2d_norm, self.bg)  # A8-A9 + A11
        else:
            r.backward(self.params, cams, dL, self.grads, self.grad2d_norm, self.bg)  # A8-A9
            if self.peer is not None:
                self.peer.step()                                             # A10 + A11 fused, peer memory
            elif self.sharded is not None:
                self.sharded.step()                                          # A10 + A11, row-sharded
            else:
                reduce_gradients(self.grads, self.group)                     # A10
                self.adam.step(self.grads, zero_grads=True)                  # A11
        return loss

    def step(self) -> list:
        """One pass of the Eq. 5 schedule: iterations at levels n, n-1, ..., 0."""
        return [self.iteration(l) for l in range(self.n_levels, -1, -1)]

    # ------------------------------------------------------------------ map replacement
    def _padded(self, p: torch.Tensor) -> torch.Tensor:
        """[K][ld] -> [world R][ld] (rows K.. zero), the sharded optimiser's buffer shape."""
        world = dist.get_world_size(self.group)
        R, _, _ = row_shard(p.shape[0], 0, world)
        pp = torch.zeros((world * R, p.shape[1]), dtype=torch.float32, device=p.device)
        pp[:p.shape[0]] = p
        return pp

    def _moments(self) -> tuple:
        """The full [K][ld] Adam moments of the current map (all-gathered when row-sharded)."""
        if self.peer is not None:
            return self.peer.full_state()
        if self.sharded is not None:
            m, v = self.sharded.full_state()
            K = self.params.shape[0]
            return m[:K], v[:K]
        return self.adam.m, self.adam.v

    def _install(self, p: torch.Tensor, m: torch.Tensor, v: torch.Tensor, n: int):
        """Replace the map by p (moments m, v; [K][ld'], n Gaussians): optimiser state, gradient
        buffers and per-level workspaces follow; captured graphs refer to the old buffers and are
        dropped."""
        self.n = n
        if self.peer is not None:
            from .comm import PeerAdam
            t = self.peer.t
            self.peer = PeerAdam(n, self.D, self.adam_cfg, self.group, p.device)
            self.peer.params[:, :p.shape[1]] = p[:, :self.peer.ld]
            self.peer.load_state(m, v, t)
            self.params, self.grads = self.peer.params, self.peer.grads
        elif self.sharded is not None:
            pp = self._padded(p)
            self.sharded.rebind(pp, torch.zeros_like(pp), n, m, v)
            self.params, self.grads = self.sharded.params, self.sharded.grads
        else:
            self.params = p
            self.adam.params, self.adam.m, self.adam.v, self.adam.n = p, m, v, n
            self.grads = torch.zeros_like(p)
        self.renderers = [None] * (self.n_levels + 1)
        self.graph = None   # a captured step refers to the old buffers
        self._pipe = None
        self.calibrate()

    # ------------------------------------------------------------------ densify and prune (f1)
    def densify_and_prune(self, seed: int) -> tuple:
        """SPEC.md:463-471 with the statistics gathered since the last call (needs densify_cfg):
        clone / split / prune, the Adam moments follow their Gaussians (new ones start at 0), the
        statistics are reset and the level workspaces re-sized.  Returns (n_cloned, n_split,
        n_pruned).  With replicated data parallelism the statistics are combined first (sum /
        max) so every rank takes the same decisions with the same samples."""
        if self.densify_cfg is None:
            raise RuntimeError("densify_and_prune needs MappingEngine(densify_cfg=...)")
        if self.distributed():
            dist.all_reduce(self.grad2d_norm, group=self.group)
            dist.all_reduce(self.vis_count, group=self.group)
            dist.all_reduce(self.max_radius, op=dist.ReduceOp.MAX, group=self.group)
        z = torch.from_numpy(densify_samples(self.n, seed)).to(self.params.device)
        H, W = self.shapes[0]
        cfg = self.densify_cfg.struct(W, H)
        m0, v0 = self._moments()
        p, m, v, counts, tags = densify(self.params, self.n, self.D, m0, v0, self.grad2d_norm,
                                        self.vis_count, self.max_radius, z, cfg, tags=self.temporary)
        n = counts[3]
        if self.spatial_order and n > 0:  # clones and split children went to the end: re-order
            perm = core_spatial_order(p, n, self.D)
            p, m, v = (permute_columns(x, perm, n) for x in (p, m, v))
            tags = permute_columns(tags.to(torch.int32), perm, n).to(torch.uint8)
        self.order = None
        self.temporary = tags
        dev = p.device
        self.grad2d_norm = torch.zeros(max(n, 1), dtype=torch.float32, device=dev)
        self.vis_count = torch.zeros(max(n, 1), dtype=torch.float32, device=dev)
        self.max_radius = torch.zeros(max(n, 1), dtype=torch.int32, device=dev)
        self._install(p, m, v, n)
        return counts[:3]

    # ------------------------------------------------------------------ geometry densification (f2)
    def add_keyframe_features(self, view: int, uv, active, kp_depth, depth_map, image, mode: int,
                              rho: float = 100.0) -> int:
        """temporary primitives for the inactive keypoints of keyframe `view`
        (level-0 camera), appended to the map with zero Adam moments; the workspaces are re-sized.
        uv [n, 2], active [n] (0/1), kp_depth [n] (mono), depth_map [H, W] (RGB-D, mode 1),
        image [3, H, W]; numpy or device tensors.  Returns the number of primitives added."""
        dev = self.params.device
        t = lambda a, dt: None if a is None else torch.as_tensor(np.asarray(a) if not torch.is_tensor(a) else a,  # noqa: E731
                                                                 dtype=dt).to(dev).contiguous()
        newp, cnt, _ = geometry_densify(self.cams0[view], t(uv, torch.float32), t(active, torch.int32),
                                        t(kp_depth, torch.float32), t(depth_map, torch.float32),
                                        t(image, torch.float32), mode, self.D, rho)
        if cnt == 0:
            return 0
        n0, n1 = self.n, self.n + cnt
        K = self.params.shape[0]
        ld = L.param_ld(n1)
        m0, v0 = self._moments()
        p = torch.zeros((K, ld), dtype=torch.float32, device=dev)
        p[:, :n0] = self.params[:, :n0]
        p[:, n0:n1] = newp[:, :cnt]
        m = torch.zeros_like(p)
        v = torch.zeros_like(p)
        m[:, :n0] = m0[:, :n0]
        v[:, :n0] = v0[:, :n0]
        grow = lambda a, fill: torch.cat([a[:n0], torch.full((cnt,), fill, dtype=a.dtype, device=dev)])  # noqa: E731
        self.temporary = grow(self.temporary, 1)
        self.grad2d_norm, self.vis_count, self.max_radius = (grow(self.grad2d_norm, 0), grow(self.vis_count, 0),
                                                             grow(self.max_radius, 0))
        if self.spatial_order:  # the new primitives went to the end: re-order
            perm = core_spatial_order(p, n1, self.D)
            p, m, v = (permute_columns(x, perm, n1) for x in (p, m, v))
            self.temporary = permute_columns(self.temporary.to(torch.int32), perm, n1).to(torch.uint8)
            self.grad2d_norm, self.vis_count = (permute_columns(x, perm, n1) for x in (self.grad2d_norm, self.vis_count))
            self.max_radius = permute_columns(self.max_radius, perm, n1)
        self.order = None
        self._install(p, m, v, n1)
        return cnt

    # ------------------------------------------------------------------ CUDA graphs
    def capture(self, gts_pinned: torch.Tensor | None = None, out_pinned: torch.Tensor | None = None):
        """Capture one step -- A0 + the Eq. 5 pass (and, with pinned host buffers, the H2D copy of
        the targets and the D2H copy of the losses) -- into a CUDA graph; `replay()` then runs it
        with a single launch.  The single-GPU fused path, the peer-memory DP step, and the
        row-sharded NCCL DP step (its reduce-scatter and all-gather are captured with it; the
        optimiser counts steps on the device).  Not the replicated all-reduce path."""
        if self.distributed() and self.peer is None and self.sharded is None:
            raise RuntimeError("graph capture: the single-GPU fused path or a sharded / peer-memory DP step")
        if self.adam is not None:
            self.adam.use_device_step()
        if self.sharded is not None:
            self.sharded.use_device_step()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        host = gts_pinned is not None

        def body():
            if host:
                self.step_host(gts_pinned, out_pinned)
            else:
                self.build_pyramids(overlap=True)
                self.graph_losses = torch.stack(self.step())

        with torch.cuda.stream(side):  # warm-up run on the capture stream (also a real step)
            body()
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            body()
        self.graph = g
        return g

    def replay(self):
        self.graph.replay()

    def capture_pipelined(self, gts_pinned: list, out_pinned: list):
        """The end-to-end step (`step_host` with prefetch) as two compute-only CUDA graphs, single GPU.

        gts_pinned / out_pinned: two pinned host buffers each ([V, 3, H, W] targets, [levels, V]
        losses).  Graph i runs A0 and the Eq. 5 pass on device target buffer i.  Call k of
        `step_pipelined()` replays graph k % 2; on a copy stream it brings gts_pinned[(k+1) % 2]
        (the NEXT step's targets, which the caller fills before call k) into the other buffer while
        the graph runs, and reads this step's losses back into out_pinned[k % 2] once it is done --
        neither copy sits on the compute stream.  `pipeline_join()` makes the current stream wait
        for the copies.  Use either this pair or `capture()`/`replay()` on an engine, not both.
        (Measured on B200, TUM config: 0.625 ms/step vs 0.664 ms with the copies inside two
        graphs and 0.607 ms for the device-only replay, tools/e2e_probe.py.)"""
        if self.distributed() or self.sharded is not None:
            raise RuntimeError("graph capture is for the single-GPU fused path")
        self.adam.use_device_step()
        bufs = [self.gt0, torch.empty_like(self.gt0)]
        dev = bufs[0].device
        self._status = torch.zeros((self.n_levels + 1, 2), dtype=torch.int32, device=dev)
        graphs, losses = [], []
        try:
            for i in range(2):  # capture() also runs one real (warm-up) step on targets i
                self.gt0 = bufs[i]
                bufs[i].copy_(gts_pinned[i], non_blocking=True)
                graphs.append(self.capture())
                losses.append(self.graph_losses)
        finally:
            status = self._status
            self._status = None
        self.gt0 = bufs[0]
        self.graph = None
        self._pipe = dict(graphs=graphs, losses=losses, bufs=bufs, gts=gts_pinned, out=out_pinned, k=0,
                          copy=torch.cuda.Stream(device=dev), status=status,
                          status_host=[torch.zeros_like(status, device="cpu").pin_memory() for _ in range(2)],
                          ev_in=[torch.cuda.Event() for _ in range(2)],
                          ev_done=[torch.cuda.Event() for _ in range(2)],
                          ev_out=[torch.cuda.Event() for _ in range(2)], pending=[False, False])
        return graphs

    def _pipe_check(self, i: int):
        """Raise if step slot i's read-back status (host wait on its copy) shows a capacity
        overflow: that step rendered nothing on the overflowing level (gs.h gs_status_async)."""
        pp = self._pipe
        if not pp["pending"][i]:
            return
        pp["ev_out"][i].synchronize()
        pp["pending"][i] = False
        st = pp["status_host"][i]
        if int(st[:, 0].bitwise_and(1).any()):
            lv = [l for l in range(st.shape[0]) if int(st[l, 0]) & 1]
            raise RuntimeError(f"pair capacity exceeded at GP level(s) {lv} (pairs {st[:, 1].tolist()}); "
                               "re-calibrate (MappingEngine.calibrate) and re-capture")

    def step_pipelined(self) -> torch.Tensor:
        """Call k of the pipelined end-to-end step (see capture_pipelined): returns the pinned
        losses buffer it fills (valid after pipeline_join() and a synchronise).  Call 0 also copies
        its own targets (gts_pinned[0]); later calls' targets were prefetched by the previous call.
        Call k first checks the status read back by call k - 2 (which used the same pinned
        buffers) and raises on a pair-capacity overflow."""
        pp = self._pipe
        if pp is None:
            raise RuntimeError("step_pipelined needs capture_pipelined() (again, after the map was replaced)")
        k = pp["k"]
        i = k % 2
        self._pipe_check(i)
        cs, cp = torch.cuda.current_stream(), pp["copy"]
        if k == 0:
            pp["bufs"][i].copy_(pp["gts"][i], non_blocking=True)
            cp.wait_stream(cs)
        else:
            cs.wait_event(pp["ev_in"][i])          # this step's targets have arrived
            cp.wait_event(pp["ev_done"][1 - i])    # the previous step is done with the other buffer
        with torch.cuda.stream(cp):                # the next step's targets, during this step
            pp["bufs"][1 - i].copy_(pp["gts"][1 - i], non_blocking=True)
            pp["ev_in"][1 - i].record(cp)
        pp["graphs"][i].replay()
        pp["ev_done"][i].record(cs)
        cp.wait_event(pp["ev_done"][i])
        with torch.cuda.stream(cp):                # this step's losses and status, off the compute stream
            pp["out"][i].copy_(pp["losses"][i], non_blocking=True)
            pp["status_host"][i].copy_(pp["status"], non_blocking=True)
            pp["ev_out"][i].record(cp)
        pp["pending"][i] = True
        pp["k"] = k + 1
        return pp["out"][i]

    def pipeline_join(self):
        """The current stream waits for the pipelined step's copies (losses read back, prefetch)."""
        torch.cuda.current_stream().wait_stream(self._pipe["copy"])

    def pipeline_check(self):
        """Host wait for the outstanding read-backs; raises on a pair-capacity overflow."""
        for i in range(2):
            self._pipe_check(i)

    def step_host(self, gts_pinned: torch.Tensor, out_pinned: torch.Tensor,
                  next_gts_pinned: torch.Tensor | None = None):
        """End-to-end public API: new keyframe targets from pinned host memory (H2D), A0,
        the Eq. 5 pass, per-level losses back to pinned host memory (D2H).

        next_gts_pinned: the targets of the NEXT call, copied on a copy stream into a second
        device buffer while this step computes (double buffering); the next call then starts
        from them instead of copying gts_pinned.  Every call still moves its targets host->device
        and its losses device->host."""
        cur = torch.cuda.current_stream()
        if getattr(self, "_staged", None) is not None:  # prefetched by the previous call
            buf, ev = self._staged
            cur.wait_event(ev)
            self._gt_spare, self.gt0 = self.gt0, buf
            self._staged = None
        else:
            self.gt0.copy_(gts_pinned, non_blocking=True)
        self.build_pyramids(overlap=True)
        if next_gts_pinned is not None:
            if getattr(self, "_copy_stream", None) is None:
                self._copy_stream = torch.cuda.Stream(device=self.gt0.device)
            if getattr(self, "_gt_spare", None) is None:
                self._gt_spare = torch.empty_like(self.gt0)
            free = torch.cuda.Event()
            free.record(cur)  # the spare buffer's last reader (the previous step) is queued before this
            self._copy_stream.wait_event(free)
            with torch.cuda.stream(self._copy_stream):
                self._gt_spare.copy_(next_gts_pinned, non_blocking=True)
                done = torch.cuda.Event()
                done.record()
            self._staged = (self._gt_spare, done)
            self._gt_spare = None
        losses = self.step()
        out_pinned.copy_(torch.stack(losses), non_blocking=True)
        return out_pinned
