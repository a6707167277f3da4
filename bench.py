#!/usr/bin/env python
"""Benchmark of the Photo-SLAM photorealistic-mapping hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config tum] [--impl ours|reference]

A *step* is one pass of the whole hot path over this rank's keyframe batch: the Gaussian
pyramid of the new keyframe targets (A0) and one mapping iteration at each pyramid level
n = 2, 1, 0 (Eq. 5; each iteration = preprocess, bin, sort, composite, Eq. 4 loss, backward,
NCCL gradient all-reduce when N > 1, fused Adam).  `value` = keyframe-view mapping
iterations per second over all ranks (weak scaling: one keyframe view per GPU for the
single-view configs).  Inputs are synthetic (synth/) and resident in HBM; the parameter +
Adam working set (4 x 47 MB at the TUM config) exceeds the 126 MB L2, so no flush is needed.

--impl reference times the CPU oracle (oracle/) on a bounded sample of the same workload
(the only reference this paper has; rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "mapping iters/sec (fwd+bwd) and render FPS at 1/2/4/8 B200; % HBM roofline"
# FP32 operations of the raster backward (A8; SURVEY §8(d)'s ALU model counts per
# evaluated (pixel, Gaussian) pair).  Every list entry up to the pixel's last contributor is
# evaluated: power 9, exp 2, alpha 2 -> 13.  A composited entry adds T recovery 2, colour grads
# 3, dL/dalpha 10, acc update 9, dL/dsigma 1, dL/dpower 1, mean2d moments 10, conic moments 9
# -> 45 (58 in total).
BWD_FLOP_PER_EVAL = 13
BWD_FLOP_PER_COMP = 45
BWD_FLOP_PER_PAIR = BWD_FLOP_PER_EVAL + BWD_FLOP_PER_COMP


# Forward (A6) FLOPs (SURVEY §8(d) ALU model): every list entry up to the pixel's stop is
# evaluated -- dx, dy, the quadratic form and the cutoff, sigma e^power, the alpha clamp and skip
# (12); a composited entry adds the colour update 3 x fma and the transmittance update (9).
FWD_FLOP_PER_EVAL = 12
FWD_FLOP_PER_COMP = 9


def survey_step_bytes(K: int, n: int, b: int, lv: dict, world: int, eng) -> float:
    """SURVEY §8(d) algorithmic bytes of one iteration (one GP level) per GPU with b local views,
    the measured visible count V and pair count P per view: A1 4KN + b(8N + 40V), A2 b 8N,
    A3 b(20V + 12P), A4 b 24P, A5 b(8P + 8 tiles), A6 b(40P + 20 Npx), A7 b 36 Npx,
    A8 b(40P + 20 Npx + 36V), A9 8KN + b 36V, A11 28KN (28KN/G row-sharded)."""
    V, P, px, tiles = lv["V"], lv["P"], lv["px"], lv["tiles"]
    a11 = 28 * K * n / (world if getattr(eng, "sharded", None) is not None else 1)
    return (4 * K * n + b * (8 * n + 40 * V) + b * 8 * n + b * (20 * V + 12 * P) + b * 24 * P
            + b * (8 * P + 8 * tiles) + b * (40 * P + 20 * px) + b * 36 * px + b * (40 * P + 20 * px + 36 * V)
            + 8 * K * n + b * 36 * V + a11)


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json copy)"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if r[2 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ----------------------------------------------------------------------------- workload
def workload_config(name: str, world: int) -> dict:
    """The `config` object of the JSON line (both arms print the same one)."""
    from synth import config
    cfg = config(name)
    K = 11 + 3 * (cfg["sh_degree"] + 1) ** 2
    ld = (cfg["n"] + 63) // 64 * 64
    views = 1 if cfg["views"] == 1 else cfg["views"]
    per_gpu = 1 if cfg["views"] == 1 else len(range(0, views, world))
    total = world if cfg["views"] == 1 else views
    return {"workload": name, "n_gaussians": cfg["n"], "sh_degree": cfg["sh_degree"], "width": cfg["width"],
            "height": cfg["height"], "gp_levels": cfg["levels"] + 1, "views_per_gpu": per_gpu,
            "global_batch": total, "iters_per_step": cfg["levels"] + 1, "parallelism": f"dp{world}",
            "l2": f"working set {4 * K * ld * 4 / 1e6:.0f} MB (params+grads+Adam m,v) > 126 MB L2; no flush",
            "layout": "Gaussians in Morton order (MappingEngine spatial_order, once at setup; the input recipe "
                      "shuffles them)"}


# ----------------------------------------------------------------------------- oracle (CPU)
_ORACLE_SCENES = {}


def oracle_fraction_step(cfg_name: str, level0_pixels: int, seed: int = 0, rank_view: int = 0):
    """The CPU oracle on a fraction f = level0_pixels / (H W) of one step of the workload, every
    stage at the same fraction: for each GP level n..0, render + backward on f H_l W_l random
    pixels (dL masked to them), Eq. 4 on an f-high band of rows, and the fp64 Adam step of an f
    share of the Gaussians.  Returns (seconds, iteration-equivalents done = (n+1) f, description):
    throughput = iteration-equivalents / seconds, all of it measured (no extrapolation)."""
    import oracle.oracle as orc
    from synth import config, make_cameras, make_scene, perturb
    cfg = config(cfg_name)
    if cfg_name not in _ORACLE_SCENES:  # input construction, not oracle work
        _ORACLE_SCENES[cfg_name] = (perturb(make_scene(cfg), 99), make_cameras(cfg, rank_view + 1)[rank_view])
    scene, cam0 = _ORACLE_SCENES[cfg_name]
    n_levels = cfg["levels"]
    f = min(1.0, level0_pixels / (cam0.width * cam0.height))
    rng = np.random.default_rng(seed)
    n = scene.n
    ng = max(1, int(round(f * n)))
    spent = 0.0
    for level in range(n_levels, -1, -1):
        cam = orc.level_camera(cam0, level)
        H, W = cam.height, cam.width
        k = max(1, int(round(f * H * W)))
        idx = rng.choice(H * W, size=k, replace=False)
        pix = np.stack([np.zeros(k, int), idx // W, idx % W], 1).astype(np.int32)
        band = max(1, int(round(f * H)))
        gt = rng.uniform(0.05, 0.95, size=(3, band, W))
        crop = rng.uniform(0.05, 0.95, size=(3, band, W))
        G = rng.normal(size=(k, 3))
        t0 = time.perf_counter()
        orc.render(scene, [cam], "recipe", pixels=pix)
        orc.loss(crop, gt, 0.2)
        g = orc.backward(scene, [cam], G, "recipe", pixels=pix)
        for cls, lr in (("means", 1.6e-4), ("quats", 1e-3), ("log_scales", 5e-3), ("opacity_logits", 5e-2),
                        ("sh", 2.5e-3)):
            arr = getattr(scene, cls)[:ng].reshape(-1).astype(np.float64)
            orc.adam(arr, g[cls][:ng].reshape(-1), np.zeros(arr.size), np.zeros(arr.size), lr=lr, step=1)
        spent += time.perf_counter() - t0
    desc = (f"{cfg_name}: fraction f = {f:.5f} of one step (levels {n_levels}..0: render + backward on f H W "
            f"random pixels, Eq. 4 on an f-high row band, fp64 Adam on f of the {n} Gaussians); "
            f"iteration-equivalents = {n_levels + 1} f per step, measured, not extrapolated")
    return spent, (n_levels + 1) * f, desc


def oracle_full_frame(cfg_name: str = "tiny", threads: int | None = None):
    """The oracle over a whole frame (every pixel): render + Eq. 4 + backward + Adam of the tiny
    config (configs[0]), with the given OpenMP thread count; seconds."""
    import oracle.oracle as orc
    from synth import make_cameras, make_scene, noise_image
    scene = make_scene(cfg_name)
    cam = make_cameras(cfg_name, 1)[0]
    gt = noise_image(cam.height, cam.width, 1)
    old = orc.threads()
    if threads:
        orc.set_threads(threads)
    try:
        t0 = time.perf_counter()
        r = orc.render(scene, [cam], "recipe")
        _, _, dL = orc.loss(r["rgb"][0], gt, 0.2)
        g = orc.backward(scene, [cam], dL[None], "recipe")
        for cls in ("means", "quats", "log_scales", "opacity_logits", "sh"):
            arr = getattr(scene, cls).reshape(-1).astype(np.float64)
            orc.adam(arr, g[cls].reshape(-1), np.zeros(arr.size), np.zeros(arr.size), lr=1e-3, step=1)
        return time.perf_counter() - t0, orc.threads()
    finally:
        orc.set_threads(old)


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    import oracle.oracle as orc
    for w in range(args.warmup):
        oracle_fraction_step(args.config, args.ref_pixels, seed=1000 + w)
    secs, work = 0.0, 0.0
    for s in range(args.steps):
        t, wk, desc = oracle_fraction_step(args.config, args.ref_pixels, seed=s)
        secs += t
        work += wk
    value = work / secs
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "iters/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": secs / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(args.config, world),
            "cpu_baseline": {"value": value, "unit": "iters/s", "cores": orc.threads(), "kind": "oracle",
                             "sample": desc},
            "e2e": {"value": value, "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "iteration_equivalents_per_step": work / args.steps}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- GPU arm
def use_chunked(view_tiles: int, cap: int) -> bool:
    """Mirror of gs_internal.cuh use_chunked: the chunk-parallel raster path (few lists, or up to
    8192 lists with a pair capacity of >= 1024 per list)."""
    return view_tiles < 1000 or (view_tiles <= 8192 and cap >= 1024 * view_tiles)
FUSED_SCHEDULE_TILES = 8192  # views x tiles up to this: one-CTA tile scan + schedule (raster.cu)


def launches_per_iteration(key_bits: int, fused: bool, binning: int = 0, chunked: bool = False,
                           view_tiles: int = 0) -> int:
    """Kernels libgs.so launches per mapping iteration (api.cu sequencing): preprocess + scan (2);
    binning 0: bucket scatter, short- and long-bucket tile sorts with the pair-record gather (3) /
    binning 1: duplicate, sort histogram, one pass per 8-bit digit, fixup, ranges, pair gather
    (5 + passes); raster fwd (1); the raster schedule (chunk index on levels with few tiles, else
    the longest-first tile order) (1) -- built inside the bucket path's tile scan when
    views x tiles <= 8192 (0); loss (2); fused: raster bwd + preprocess bwd + Adam (3), else +
    gradient accumulate (4)."""
    passes = (key_bits + 7) // 8
    binning_kernels = 3 if binning == 0 else 5 + passes
    schedule = 0 if binning == 0 and view_tiles <= FUSED_SCHEDULE_TILES else 1
    return 2 + binning_kernels + 1 + schedule + 2 + (3 if fused else 4)


def run_ours(args):
    import torch
    import torch.distributed as dist
    rank, world, local = dist_env()
    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    from paper_2311_16728_b200 import _lib as L
    from paper_2311_16728_b200.build import build
    from paper_2311_16728_b200.core import Renderer, pack_params
    from paper_2311_16728_b200.mapping import MappingEngine, shard_views
    from synth import config, make_cameras, make_scene, perturb
    if rank == 0:
        build()
    if world > 1:
        dist.barrier()
    L.lib()
    cfg = config(args.config)
    n_views_global = max(cfg["views"], world) if cfg["views"] == 1 else cfg["views"]
    if cfg["views"] == 1:
        n_views_global = world  # weak scaling: one keyframe per GPU
    my_views = shard_views(n_views_global, rank, world)
    scene = make_scene(cfg)
    cams_all = make_cameras(cfg, n_views_global)
    cams = [cams_all[v] for v in my_views]
    D = cfg["sh_degree"]
    n = scene.n
    # targets: renders of the unperturbed scene (SURVEY §8(d) 'Ground truth'), by this path
    rtmp = Renderer(n, D, len(cams), cams[0].width, cams[0].height, 8 << 20)
    p0 = pack_params(scene)
    gt = rtmp.forward(p0, cams)[0].clone()
    del rtmp, p0
    eng = MappingEngine(perturb(scene, 99), cams, gt, n_levels=cfg["levels"], comm=args.comm)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    iters_per_step = cfg["levels"] + 1

    def step():
        eng.build_pyramids(overlap=True)
        return eng.step()

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    eng.check()
    if args.launch_list:
        # exactly one step inside a cudaProfilerStart/Stop range (ncu --profile-from-start off)
        torch.cuda.profiler.start()
        step()
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        if rank == 0:
            print(json.dumps({"launch_list": True, "config": args.config}), flush=True)
        return 0

    if args.quick:  # A/B runs: the headline graph replay only
        use_graph = (world == 1 or eng.peer is not None or eng.sharded is not None) and not args.no_graph
        if use_graph:
            eng.capture()
            for _ in range(3):
                eng.replay()
        torch.cuda.synchronize()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for _ in range(args.steps):
            eng.replay() if use_graph else step()
        t1.record(stream)
        torch.cuda.synchronize()
        eng.check()
        ms = t0.elapsed_time(t1) / args.steps
        if rank == 0:
            print(json.dumps({"quick": True, "config": args.config, "value": iters_per_step * len(cams) * world / (ms * 1e-3),
                              "ms_per_step": ms}), flush=True)
        return 0

    # ---- per-stage breakdown (separate instrumented pass; not the headline)
    stage = {k: 0.0 for k in ("pyramid", "preprocess", "render_fwd", "loss", "backward", "allreduce", "adam")}
    reps = 5
    for _ in range(reps):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record(); eng.build_pyramids(); ev[1].record(); torch.cuda.synchronize()
        stage["pyramid"] += ev[0].elapsed_time(ev[1])
        for level in range(cfg["levels"], -1, -1):
            r = eng.renderers[level]
            c = eng.cams[level]
            e = [torch.cuda.Event(enable_timing=True) for _ in range(7)]
            ps = L.params_struct(eng.params, n, D)
            e[0].record(); L.gs_preprocess(ps, c, r.ws.buf)
            e[1].record(); L.gs_render_forward(ps, c, r.ws.buf, eng.bg, r.rgb, r.T)
            e[2].record(); loss, dL = eng.losses[level](r.rgb, eng.pyr[level])
            if eng.distributed():
                e[3].record(); r.backward(eng.params, c, dL, eng.grads, eng.grad2d_norm, eng.bg)
                e[4].record()
                from paper_2311_16728_b200.mapping import all_gather_rows, reduce_gradients, reduce_scatter_rows
                if eng.peer is not None:  # barrier | fused reduce + Adam + broadcast over peer memory
                    e[5].record()
                    eng.peer.step()
                elif eng.sharded is not None:  # reduce-scatter | row-sharded Adam + all-gather
                    sh = eng.sharded
                    reduce_scatter_rows(sh.padded_grads, sh.R)
                    e[5].record()
                    sh.t += 1
                    sh._adam_rows()
                    all_gather_rows(sh.padded_params, sh.R)
                    sh.padded_grads.zero_()
                else:
                    reduce_gradients(eng.grads)
                    e[5].record(); eng.adam.step(eng.grads, zero_grads=True)
                e[6].record()
            else:  # fused backward + Adam (single GPU)
                e[3].record(); r.backward_adam(eng.params, c, dL, eng.adam, eng.grad2d_norm, eng.bg)
                e[4].record(); e[5].record(); e[6].record()
            torch.cuda.synchronize()
            for k, name in enumerate(("preprocess", "render_fwd", "loss", "backward", "allreduce", "adam")):
                stage[name] += e[k].elapsed_time(e[k + 1])
    stage = {k: v / reps for k, v in stage.items()}

    # ---- algorithmic work of the raster kernels per level: composited (pixel, Gaussian) pairs
    # and evaluated pairs (list entries up to each pixel's last contributor, which the
    # back-to-front replay visits)
    comp_pairs, eval_pairs, levels_meas = [], [], []
    L.gs_set_render_stats(True)  # the composited counts are a diagnostic output (off when timed)
    for level in range(cfg["levels"], -1, -1):
        eng.render(level)
        torch.cuda.synchronize()
        rw = eng.renderers[level].ws
        v = rw.views()
        comp_pairs.append(int(v["n_composited"].sum().item()))
        eval_pairs.append(int(v["n_contrib"].to(torch.int64).sum().item()))
        _, _, P_l = rw.status()
        levels_meas.append({"level": level, "V": int((v["radius"] > 0).sum().item()) / len(cams), "P": P_l / len(cams),
                            "px": rw.W * rw.H, "tiles": rw.tiles_x * rw.tiles_y})
    L.gs_set_render_stats(False)
    pairs_per_step = sum(comp_pairs)
    flops_per_step = BWD_FLOP_PER_EVAL * sum(eval_pairs) + BWD_FLOP_PER_COMP * pairs_per_step

    # ---- live kernel timing (eager launches): each kernel family of the step is bracketed with
    # CUDA events recorded by libgs.so on its launching stream (gs_profile_kernel), one family per
    # pass of K eager steps; share = its summed launch time / the pass's step time
    live = {}
    akern = "k_adam_fused" if world == 1 else ("k_reduce_adam_bcast" if eng.peer is not None else "k_adam")
    families = ["k_preprocess", "k_tile_scan", "k_bin_scatter", "k_tile_sort", "k_raster_fwd", "k_ssim",
                "k_raster_bwd", "k_preprocess_bwd", akern]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for kname in families:
        L.gs_profile_kernel(kname)
        torch.cuda.synchronize()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for _ in range(args.steps):
            step()
        t1.record(stream)
        torch.cuda.synchronize()
        live[kname] = L.gs_profile_read() + (t0.elapsed_time(t1),)
    L.gs_profile_kernel(None)
    eager_ms = statistics.median(v[2] for v in live.values())
    shares = {k: v[0] / v[2] for k, v in live.items()}

    # ---- headline: K timed steps, one CUDA-graph replay per step: one GPU, the peer-memory DP
    # step, or the row-sharded NCCL DP step (its reduce-scatter / all-gather captured with it);
    # eager launches only for the replicated all-reduce path
    use_graph = (world == 1 or eng.peer is not None or eng.sharded is not None) and not args.no_graph
    graph_note = None
    if use_graph:
        try:
            eng.capture()
        except Exception as ex:  # noqa: BLE001  (multi-rank NCCL capture is unmeasured: fall back to eager)
            if world == 1:
                raise
            use_graph, graph_note = False, f"capture failed, eager launches: {type(ex).__name__}: {ex}"[:300]
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
    if use_graph:
        for _ in range(2):
            eng.replay()
        torch.cuda.synchronize()
    # the map trains during the run (every step is a real optimiser step), so its pair counts
    # drift; the e2e region below restarts from this snapshot: both time K steps of the same map
    snap = None
    if world == 1 and eng.adam is not None:
        snap = [(t, t.clone()) for t in (eng.params, eng.adam.m, eng.adam.v, eng.adam.t_dev)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for _ in range(args.steps):
            eng.replay() if use_graph else step()
        t1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = t0.elapsed_time(t1)
    ms_t = torch.tensor([ms], device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    eng.check()

    # ---- render FPS: A1-A6 at level 0 for this rank's views, eager launches and (one GPU) the
    # replay of a CUDA graph of the same calls (the eager number carries the host's per-call cost)
    def frame_ms(fn, nr, graph):
        if graph:
            g = torch.cuda.CUDAGraph()
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                fn()
            torch.cuda.current_stream().wait_stream(side)
            with torch.cuda.graph(g):
                fn()
            fn = g.replay
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(nr):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / nr

    nr = 50
    render_ms_eager = frame_ms(lambda: eng.render(0), nr, False)
    render_ms = frame_ms(lambda: eng.render(0), nr, world == 1) if world == 1 else render_ms_eager

    # ---- context for BASELINE.md's only comparable paper number (Table 1 render FPS on Replica
    # 1200x680, 911-1084 FPS on an RTX 4090 with ~130-140K trained Gaussians): A1-A6 of one
    # Replica-like keyframe view (500K Gaussians, SH 3) on this GPU
    replica = None
    if rank == 0 and world == 1 and not args.no_replica and args.config != "replica":
        rscene = make_scene("replica")
        rcam = make_cameras("replica", 1)
        rr = Renderer(rscene.n, 3, 1, rcam[0].width, rcam[0].height, 1 << 23)
        rp = pack_params(rscene)
        rr.forward(rp, rcam)
        torch.cuda.synchronize()
        st, flags, pairs = rr.ws.status()
        replica_eager_ms = frame_ms(lambda: rr.forward(rp, rcam), nr, False)
        replica_ms = frame_ms(lambda: rr.forward(rp, rcam), nr, True)
        replica = {"workload": "replica 1200x680, 500000 Gaussians, SH 3, 1 view", "pairs": int(pairs),
                   "render_fps": 1000.0 / replica_ms, "render_fps_eager": 1000.0 / replica_eager_ms,
                   "paper_render_fps_rtx4090": [911.262, 1084.017],
                   "paper_note": "PAPER.md:416-417,444-445 (mono, RGB-D; trained maps of 31-35 MB): context only"}
        del rr, rp

    # ---- e2e through the public API: pinned H2D of every step's targets + D2H of its losses
    # (MappingEngine.step_host, eager launches; step k+1's targets are copied on a copy stream
    # while step k computes -- the first step's copy is inside the timed region, the last step
    # prefetches nothing)
    gts_pinned = [eng.gt0.cpu().pin_memory() for _ in range(2)]
    out_pinned = torch.empty((iters_per_step, len(cams)), dtype=torch.float32).pin_memory()
    e2e_graph = world == 1 and not args.no_graph
    if e2e_graph:  # single GPU: the same API as two CUDA graphs (MappingEngine.capture_pipelined)
        outs = [out_pinned, torch.empty_like(out_pinned).pin_memory()]
        eng.capture_pipelined(gts_pinned, outs)

        def run_e2e(k, last):
            eng.step_pipelined()
    else:
        def run_e2e(k, last):
            eng.step_host(gts_pinned[k % 2], out_pinned, None if last else gts_pinned[(k + 1) % 2])
    # warm-up: W steps, and on one GPU on for at least 0.3 s -- the graph captures above leave
    # the GPU idle long enough for its clocks to drop, and a short warm-up then times the ramp
    # (measured: 0.67 -> 0.617 ms per TUM step over the first ~100 ms, tools/e2e_var.py).  Under
    # torchrun every rank runs the same fixed count (each step holds collectives).
    t_w, k = time.perf_counter(), 0
    n_w = max(args.warmup, 3) + (0 if world == 1 else 16)
    while k < n_w or (world == 1 and time.perf_counter() - t_w < 0.3):
        run_e2e(k, False)
        k += 1
        if k % 8 == 0:
            torch.cuda.synchronize()
    if not e2e_graph:
        run_e2e(k, True)  # drain the prefetch chain
    if e2e_graph:
        eng.pipeline_join()
    torch.cuda.synchronize()
    if snap is not None:  # the headline's starting map (outside the timed region)
        for dst, src in snap:
            dst.copy_(src)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for k in range(args.steps):
        run_e2e(k, k == args.steps - 1)
    if e2e_graph:
        eng.pipeline_join()  # the last step's losses are read back inside the timed region
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = torch.tensor([e0.elapsed_time(e1)], device=dev)
    if world > 1:
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    e2e_ms = float(e2e_ms.item())
    if e2e_graph:
        eng.pipeline_check()  # raises if a timed step overflowed its pair capacity (rendered nothing)
    eng.check()

    # ---- rooflines.  Per kernel family: the raster kernels (A6, A8) are FP32-ALU bound
    # (algorithmic FLOPs per evaluated / composited pair) against 148 SMs x 128 FP32
    # lanes x 2 x the SM clock sampled during the run; the per-Gaussian kernels are HBM bound
    # (SURVEY §8(d) algorithmic bytes with the measured V, P) against the measured copy peak.
    # `roofline` is the family with the largest measured share of the step.
    K = 11 + 3 * (D + 1) ** 2
    ld = eng.params.shape[1]
    clocks = clk.summary()
    sm_mhz = clocks.get("sm_mhz") or 1965.0
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    fp32_peak = sms * 128 * 2 * sm_mhz * 1e6 / 1e12  # TFLOP/s
    peak, peak_src = load_peaks()
    b = len(cams)
    bytes_model = {  # algorithmic bytes per step (all levels), measured V and P
        "k_preprocess": sum(4 * K * n + b * (8 * n + 40 * lv["V"]) for lv in levels_meas),
        "k_tile_scan": sum(b * 8 * lv["tiles"] for lv in levels_meas),
        "k_bin_scatter": sum(b * (20 * lv["V"] + 12 * lv["P"]) for lv in levels_meas),
        "k_tile_sort": sum(b * (24 + 8) * lv["P"] for lv in levels_meas),
        "k_ssim": sum(b * 36 * lv["px"] for lv in levels_meas),
        "k_preprocess_bwd": sum(8 * K * n + b * 36 * lv["V"] for lv in levels_meas),
    }
    if world == 1:
        adam_bytes = K * n * 24 + 4 * n  # fused: p, m, v read + written, a 4-byte slot per Gaussian
    elif eng.peer is not None:  # this rank's range: G gradients read, m, v read + written, p read, G p + G g written
        adam_bytes = (eng.peer.e1 - eng.peer.e0) * 4 * (world + 5 + 2 * world)
    elif eng.sharded is not None:  # this rank's rows only
        adam_bytes = (eng.sharded.r1 - eng.sharded.r0) * ld * 32
    else:
        adam_bytes = K * ld * 32
    bytes_model[akern] = adam_bytes * len(levels_meas)
    flops_model = {"k_raster_bwd": flops_per_step,
                   "k_raster_fwd": FWD_FLOP_PER_EVAL * sum(eval_pairs) + FWD_FLOP_PER_COMP * pairs_per_step}
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get(args.config, {})
        except Exception:  # noqa: BLE001
            traffic = {}

    def roof(kname):
        ms_k, launches_k, wall = live[kname]
        per_step = ms_k / args.steps
        common = {"kernel": kname, "avg_launch_ms": ms_k / max(launches_k, 1), "launches_per_step":
                  launches_k / args.steps, "share_of_step": ms_k / wall,
                  "traffic": (traffic or {}).get(kname),
                  "timing": "CUDA events around each launch on its stream, eager pass of K steps"}
        if kname in flops_model:
            ach = flops_model[kname] / (per_step * 1e-3) / 1e12
            return {"bound": "alu", "achieved": ach, "peak": fp32_peak, "unit": "TFLOP/s", "frac": ach / fp32_peak,
                    "peak_source": f"{sms} SMs x 128 FP32 lanes x 2 FLOP x {sm_mhz:.0f} MHz (sampled)",
                    "algorithmic_flops_per_launch": flops_model[kname] / max(launches_k / args.steps, 1), **common}
        ach = bytes_model[kname] / (per_step * 1e-3) / 1e9
        return {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                "peak_source": peak_src, "algorithmic_bytes_per_launch": bytes_model[kname] /
                max(launches_k / args.steps, 1), **common}

    kernel_roofs = {k: roof(k) for k in families if (k in flops_model or k in bytes_model) and live[k][0] > 0}
    dominant = max(kernel_roofs, key=lambda k: kernel_roofs[k]["share_of_step"])
    roofline = dict(kernel_roofs[dominant])
    roofline["chosen_by"] = "largest measured share of the step"
    roofline["evaluated_pairs_per_level"] = eval_pairs
    roofline["composited_pairs_per_level"] = comp_pairs
    # step-level HBM fraction (the metric's third part): SURVEY §8(d) algorithmic bytes of every
    # stage at every level with the measured V and P, over the measured step time
    step_bytes = sum(survey_step_bytes(K, n, b, lv, world, eng) for lv in levels_meas)
    ms_step = ms_max / args.steps
    roofline_step = {"bound": "hbm", "algorithmic_bytes_per_step": step_bytes, "peak": peak, "unit": "GB/s",
                     "achieved": step_bytes / (ms_step * 1e-3) / 1e9,
                     "frac": step_bytes / (ms_step * 1e-3) / 1e9 / peak,
                     "levels": [{k: lv[k] for k in ("level", "V", "P", "px", "tiles")} for lv in levels_meas],
                     "model": "SURVEY §8(d): A1 4KN+b(8N+40V), A2 b8N, A3 b(20V+12P), A4 b24P, A5 b(8P+8 tiles), "
                              "A6 b(40P+20Npx), A7 b36Npx, A8 b(40P+20Npx+36V), A9 8KN+b36V, A11 28KN (/G sharded)"}

    total_views = len(cams) * world
    value = iters_per_step * total_views * args.steps / (ms_max * 1e-3)
    e2e_value = iters_per_step * total_views * args.steps / (e2e_ms * 1e-3)
    launches_step = 2  # pyramid levels (k_pyr_down)
    for r in eng.renderers:
        t = r.ws.tiles_x * r.ws.tiles_y * len(cams)
        bits = 32 + max(1, math.ceil(math.log2(max(t, 2))))
        launches_step += launches_per_iteration(bits, world == 1, chunked=use_chunked(t, r.ws.capacity), view_tiles=t)
        if world > 1 and eng.peer is not None:  # peer barrier + fused reduce/Adam/broadcast + barrier for Adam
            launches_step += 2
        elif world > 1 and eng.sharded is not None and use_graph:  # device step counter of the row Adam
            launches_step += 1
    launches = args.steps * launches_step

    # ---- sorted keys/s (A4): the level-0 pairs of this step (keys (tile << 32 | depth bits),
    # Gaussian ids), randomly permuted, through the onesweep LSD radix sort (gs_debug_sort_pairs);
    # and the default bucket path's rate: pairs / (bin scatter + tile sorts) per level-0 launch
    sorted_keys = None
    if rank == 0:
        rw = eng.renderers[0].ws
        eng.render(0)
        torch.cuda.synchronize()
        v0 = rw.views()
        _, _, P0 = rw.status()  # this render's pairs (the map has trained since levels_meas)
        bits = 32 + max(1, math.ceil(math.log2(max(rw.tiles_x * rw.tiles_y * len(cams), 2))))
        perm = torch.randperm(P0, device=dev)
        k_src, v_src = v0["keys"][:P0][perm].clone(), v0["vals"][:P0][perm].clone()
        kk, vv = torch.empty_like(k_src), torch.empty_like(v_src)
        k2, v2 = torch.empty_like(k_src), torch.empty_like(v_src)
        temp = torch.empty(L.gs_sort_temp_size(P0, bits), dtype=torch.uint8, device=dev)
        reps, tot = 20, 0.0
        for r_ in range(reps + 3):
            kk.copy_(k_src)
            vv.copy_(v_src)
            a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a_.record(stream)
            L.gs_debug_sort_pairs(kk, vv, k2, v2, bits, temp)
            b_.record(stream)
            torch.cuda.synchronize()
            if r_ >= 3:
                tot += a_.elapsed_time(b_)
        # keys equal the bucket path's order; equal keys (same tile, equal fp32 depth) keep the
        # permuted input order in the stable radix sort, so values are compared as per-key sets
        ok = bool(torch.equal(kk, v0["keys"][:P0]) and
                  torch.equal((kk * 0 + vv.to(torch.int64)).sum(), v0["vals"][:P0].to(torch.int64).sum()))
        radix_ms = tot / reps
        bucket_ms = None
        if True:
            # level-0 share of the bucket kernels: launches are per level, level 0 is the last of each step
            L.gs_profile_kernel("k_tile_sort")
            eng.render(0)
            tms = L.gs_profile_read()
            L.gs_profile_kernel("k_bin_scatter")
            eng.render(0)
            bms = L.gs_profile_read()
            L.gs_profile_kernel(None)
            bucket_ms = tms[0] + bms[0]
        sorted_keys = {"pairs": P0, "key_bits": bits, "radix_onesweep_keys_per_s": P0 / (radix_ms * 1e-3),
                       "radix_ms": radix_ms, "radix_keys_equal_bucket_order": ok,
                       "bucket_keys_per_s": (P0 / (bucket_ms * 1e-3)) if bucket_ms else None,
                       "bucket_ms": bucket_ms,
                       "note": "level-0 pairs of this step; radix = gs_debug_sort_pairs on a random permutation; "
                               "bucket = bin scatter + per-tile bitonic sorts (the default A3+A4 path)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle.oracle as orc
        secs, work, desc = oracle_fraction_step(args.config, args.ref_pixels)
        full_1, _ = oracle_full_frame("tiny", threads=1)
        full_n, nth = oracle_full_frame("tiny")
        cpu = {"value": work / secs, "unit": "iters/s", "cores": orc.threads(), "kind": "oracle",
               "sample": desc + f"; {secs:.1f} s measured",
               "full_frame_tiny": {"seconds_1_thread": full_1, "seconds_all_threads": full_n, "threads": nth,
                                   "what": "configs[0] (1000 Gaussians, 64x48): render + Eq. 4 + backward + Adam "
                                           "over every pixel, one iteration"}}
    if rank == 0:
        H, W = cams[0].height, cams[0].width
        line = {
            "metric": METRIC, "value": value, "unit": "iters/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": workload_config(args.config, world),
            "roofline": roofline,
            "roofline_step": roofline_step,
            "roofline_hbm": kernel_roofs[akern],
            "kernel_rooflines": kernel_roofs,
            "sorted_keys_per_s": sorted_keys,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "iters/s",
                    "h2d_bytes_per_step": int(gts_pinned[0].numel() * 4),
                    "d2h_bytes_per_step": int(out_pinned.numel() * 4),
                    "api": ("MappingEngine.step_pipelined (two compute-only CUDA graphs; next step's targets copied "
                            "H2D while this step computes)") if e2e_graph else
                           "MappingEngine.step_host (eager launches, prefetch on a copy stream)"},
            "gpu_launches": launches,
            "clocks": clocks,
            "render_fps": 1000.0 / render_ms * len(cams) * world,
            "render_fps_eager": 1000.0 / render_ms_eager * len(cams) * world,
            "render_replica": replica,
            "stage_ms_per_step": {k: round(v, 4) for k, v in stage.items()},
            "timing": {"headline": "CUDA graph replay per step" if use_graph else (graph_note or "eager launches"),
                       "eager_ms_per_step": eager_ms / args.steps},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="replica",
                    help="workload (synth CONFIGS); the headline is configs[2], the Replica-like keyframe")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-replica", action="store_true", help="skip the Replica render-FPS context line")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-pixels", type=int, default=2048,
                    help="oracle sample: level-0 pixels per step (the same fraction of every level and stage)")
    ap.add_argument("--launch-list", action="store_true", help="profile exactly one step (ncu range)")
    ap.add_argument("--no-graph", action="store_true", help="time eager launches instead of graph replays")
    ap.add_argument("--quick", action="store_true", help="A/B experiments: headline timing only (no extra keys)")
    ap.add_argument("--comm", default="nccl", choices=["nccl", "peer"],
                    help="N>1 optimiser exchange: NCCL reduce-scatter + row-sharded Adam + all-gather, or the "
                         "fused reduce + Adam + broadcast kernel over peer memory (unmeasured on >1 GPU)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
