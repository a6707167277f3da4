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


# ----------------------------------------------------------------------------- oracle (CPU)
def oracle_sample_step(cfg_name: str, rank_view: int = 0, n_pix: int = 4096, seed: int = 0):
    """The CPU oracle on a bounded sample of one step of the workload: for each GP level,
    render + backward on n_pix random pixels (dL masked to them), Eq. 4 on the full level image,
    and the fp64 Adam step over every parameter.  Returns (seconds extrapolated to the full
    step, seconds actually spent, description)."""
    import oracle.oracle as orc
    from synth import config, make_cameras, make_scene, perturb
    scaled_camera = orc.level_camera
    cfg = config(cfg_name)
    scene = perturb(make_scene(cfg), 99)
    cam0 = make_cameras(cfg, rank_view + 1)[rank_view]
    n_levels = cfg["levels"]
    rng = np.random.default_rng(seed)
    spent = 0.0
    extrap = 0.0
    K = scene.sh.shape[1]
    n = scene.n
    for level in range(n_levels, -1, -1):
        cam = scaled_camera(cam0, level)
        H, W = cam.height, cam.width
        k = min(n_pix, H * W)
        idx = rng.choice(H * W, size=k, replace=False)
        pix = np.stack([np.zeros(k, int), idx // W, idx % W], 1).astype(np.int32)
        gt = rng.uniform(0.05, 0.95, size=(3, H, W))
        t0 = time.perf_counter()
        r = orc.render(scene, [cam], "recipe", pixels=pix)
        t1 = time.perf_counter()
        img = np.zeros((3, H, W))
        img[:, pix[:, 1], pix[:, 2]] = r["rgb"].T
        loss, _, dL = orc.loss(img, gt, 0.2)
        t2 = time.perf_counter()
        g = orc.backward(scene, [cam], dL[:, pix[:, 1], pix[:, 2]].T, "recipe", pixels=pix)
        t3 = time.perf_counter()
        for cls, lr in (("means", 1.6e-4), ("quats", 1e-3), ("log_scales", 5e-3), ("opacity_logits", 5e-2),
                        ("sh", 2.5e-3)):
            arr = getattr(scene, cls)
            orc.adam(arr.reshape(-1), g[cls].reshape(-1), np.zeros(arr.size), np.zeros(arr.size), lr=lr, step=1)
        t4 = time.perf_counter()
        scale = (H * W) / k
        spent += t4 - t0
        extrap += (t1 - t0) * scale + (t2 - t1) + (t3 - t2) * scale + (t4 - t3)
    desc = (f"{cfg_name}: per GP level {n_levels}..0, render+backward on {n_pix} random pixels "
            f"(extrapolated x H*W/{n_pix}), full-image Eq. 4 loss, fp64 Adam over all {n}x{11 + 3 * K} params")
    return extrap, spent, desc


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    import oracle.oracle as orc
    from synth import config
    cfg = config(args.config)
    iters_per_step = cfg["levels"] + 1
    for _ in range(args.warmup):
        oracle_sample_step(args.config, n_pix=args.ref_pixels)
    ext = []
    for s in range(args.steps):
        e, _, desc = oracle_sample_step(args.config, n_pix=args.ref_pixels, seed=s)
        ext.append(e)
    sec = float(np.mean(ext))
    value = iters_per_step / sec
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "iters/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.config},
            "cpu_baseline": {"value": value, "unit": "iters/s", "cores": orc.threads(), "kind": "oracle",
                             "sample": desc},
            "e2e": {"value": value, "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- GPU arm
CHUNK_MAX_TILES = 600  # views x tiles below this use the chunked raster path (gs_internal.cuh)
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
    eng = MappingEngine(perturb(scene, 99), cams, gt, n_levels=cfg["levels"])
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
                if eng.sharded is not None:  # reduce-scatter | row-sharded Adam + all-gather
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
    comp_pairs, eval_pairs = [], []
    for level in range(cfg["levels"], -1, -1):
        eng.render(level)
        torch.cuda.synchronize()
        v = eng.renderers[level].ws.views()
        comp_pairs.append(int(v["n_composited"].sum().item()))
        eval_pairs.append(int(v["n_contrib"].to(torch.int64).sum().item()))
    pairs_per_step = sum(comp_pairs)
    flops_per_step = BWD_FLOP_PER_EVAL * sum(eval_pairs) + BWD_FLOP_PER_COMP * pairs_per_step

    # ---- live kernel timing (eager launches): the dominant kernels are bracketed with CUDA
    # events recorded by libgs.so on their launching stream (gs_profile_kernel)
    live = {}
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for kname in ("k_raster_bwd", "k_adam_fused" if world == 1 else "k_adam"):
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
    eager_ms = min(v[2] for v in live.values())

    # ---- headline: K timed steps (one CUDA-graph replay per step on a single GPU; eager
    # launches under torchrun, where the NCCL all-reduce sits inside the iteration)
    use_graph = world == 1 and not args.no_graph
    if use_graph:
        eng.capture()
        for _ in range(2):
            eng.replay()
        torch.cuda.synchronize()
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
    if rank == 0 and world == 1 and not args.no_replica:
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

    # ---- rooflines.  Dominant kernel: the raster backward (A8), FP32-ALU bound: algorithmic
    # FLOPs = evaluated pairs x 13 + composited pairs x 45 against 148 SMs x 128 FP32
    # lanes x 2 x the SM clock sampled during the run.  Second: the fused Adam (A11), HBM bound.
    K = 11 + 3 * (D + 1) ** 2
    ld = eng.params.shape[1]
    clocks = clk.summary()
    sm_mhz = clocks.get("sm_mhz") or 1965.0
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    fp32_peak = sms * 128 * 2 * sm_mhz * 1e6 / 1e12  # TFLOP/s
    bwd_ms, bwd_launches, _ = live["k_raster_bwd"]
    bwd_flops = flops_per_step * args.steps
    bwd_achieved = bwd_flops / (bwd_ms * 1e-3) / 1e12
    akern = "k_adam_fused" if world == 1 else "k_adam"
    adam_ms, adam_launches, _ = live[akern]
    if world == 1:
        adam_bytes = K * n * 24 + 4 * n
    elif eng.sharded is not None:  # this rank's rows only
        adam_bytes = (eng.sharded.r1 - eng.sharded.r0) * ld * 32
    else:
        adam_bytes = K * ld * 32
    peak, peak_src = load_peaks()
    adam_achieved = adam_bytes * adam_launches / (adam_ms * 1e-3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get(args.config, {})
        except Exception:  # noqa: BLE001
            traffic = {}

    total_views = len(cams) * world
    value = iters_per_step * total_views * args.steps / (ms_max * 1e-3)
    e2e_value = iters_per_step * total_views * args.steps / (e2e_ms * 1e-3)
    launches_step = 2  # pyramid levels (k_pyr_down)
    for r in eng.renderers:
        t = r.ws.tiles_x * r.ws.tiles_y * len(cams)
        bits = 32 + max(1, math.ceil(math.log2(max(t, 2))))
        launches_step += launches_per_iteration(bits, world == 1, chunked=t < CHUNK_MAX_TILES, view_tiles=t)
    launches = args.steps * launches_step

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        import oracle.oracle as orc
        ext, spent, desc = oracle_sample_step(args.config, n_pix=args.ref_pixels)
        cpu = {"value": iters_per_step / ext, "unit": "iters/s", "cores": orc.threads(), "kind": "oracle",
               "sample": desc + f"; {spent:.1f} s measured"}
    if rank == 0:
        H, W = cams[0].height, cams[0].width
        line = {
            "metric": METRIC, "value": value, "unit": "iters/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": args.config, "n_gaussians": n, "sh_degree": D, "width": W, "height": H,
                       "gp_levels": cfg["levels"] + 1, "views_per_gpu": len(cams), "global_batch": total_views,
                       "iters_per_step": iters_per_step, "parallelism": f"dp{world}",
                       "l2": f"working set {4 * K * ld * 4 / 1e6:.0f} MB (params+grads+Adam m,v) > 126 MB L2; no flush",
                       "layout": "Gaussians in Morton order (MappingEngine spatial_order, once at setup; the "
                                 "input recipe shuffles them)"},
            "roofline": {"bound": "alu", "kernel": "k_raster_bwd (A8)", "achieved": bwd_achieved,
                         "peak": fp32_peak, "unit": "TFLOP/s", "frac": bwd_achieved / fp32_peak,
                         "traffic": (traffic or {}).get("k_raster_bwd"),
                         "peak_source": f"{sms} SMs x 128 FP32 lanes x 2 FLOP x {sm_mhz:.0f} MHz (sampled)",
                         "algorithmic_flops_per_launch": flops_per_step / len(comp_pairs),
                         "flop_per_evaluated_pair": BWD_FLOP_PER_EVAL,
                         "flop_per_composited_pair_extra": BWD_FLOP_PER_COMP,
                         "evaluated_pairs_per_level": eval_pairs, "composited_pairs_per_level": comp_pairs,
                         "avg_launch_ms": bwd_ms / max(bwd_launches, 1),
                         "share_of_step": bwd_ms / live["k_raster_bwd"][2],
                         "timing": "CUDA events around each launch, eager pass of K steps"},
            "roofline_hbm": {"bound": "hbm", "kernel": f"{akern} (A11)", "achieved": adam_achieved, "peak": peak,
                             "unit": "GB/s", "frac": adam_achieved / peak, "traffic": (traffic or {}).get(akern),
                             "peak_source": peak_src, "algorithmic_bytes_per_launch": adam_bytes,
                             "avg_launch_ms": adam_ms / max(adam_launches, 1),
                             "share_of_step": adam_ms / live[akern][2]},
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
            "timing": {"headline": "CUDA graph replay per step" if use_graph else "eager launches",
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
    ap.add_argument("--config", default="tum")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-replica", action="store_true", help="skip the Replica render-FPS context line")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-pixels", type=int, default=4096)
    ap.add_argument("--launch-list", action="store_true", help="profile exactly one step (ncu range)")
    ap.add_argument("--no-graph", action="store_true", help="time eager launches instead of graph replays")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
