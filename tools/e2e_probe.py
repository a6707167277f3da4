"""Where does the end-to-end step lose time against the device-resident graph replay?
Times, on one GPU, K steps of: (A) capture()/replay(), (B) capture_pipelined with pinned host
targets, (C) the same with device-resident 'host' buffers (D2D copies), (D) capture() with
pinned host targets (step_host inside the graph, no prefetch).  Prints one JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2311_16728_b200.build import build  # noqa: E402
from paper_2311_16728_b200.core import Renderer, pack_params  # noqa: E402
from paper_2311_16728_b200.mapping import MappingEngine  # noqa: E402
from synth import config, make_cameras, make_scene, perturb  # noqa: E402


def main(cname="tum", K=40):
    build()
    cfg = config(cname)
    scene = make_scene(cfg)
    cams = make_cameras(cfg, cfg["views"])
    rt = Renderer(scene.n, cfg["sh_degree"], len(cams), cams[0].width, cams[0].height, 8 << 20)
    gt = rt.forward(pack_params(scene), cams)[0].clone()
    del rt
    L = cfg["levels"] + 1

    def timed(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(K):
            fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / K

    out = {}
    eng = MappingEngine(perturb(scene, 99), cams, gt, n_levels=cfg["levels"])
    eng.capture()
    out["A_replay_ms"] = timed(eng.replay)
    del eng
    for name, mk in (("B_pipelined_pinned_ms", lambda: gt.cpu().pin_memory()),
                     ("C_pipelined_device_ms", lambda: gt.clone())):
        eng = MappingEngine(perturb(scene, 99), cams, gt, n_levels=cfg["levels"])
        g = [mk() for _ in range(2)]
        o = [torch.empty((L, len(cams))).pin_memory() for _ in range(2)]
        eng.capture_pipelined(g, o)
        out[name] = timed(eng.step_pipelined)
        del eng
    # E: compute-only graph; the next step's targets copied H2D on a copy stream into a staging
    # buffer (eager), a D2D copy into the graph's input, the losses read back eagerly
    eng = MappingEngine(perturb(scene, 99), cams, gt, n_levels=cfg["levels"])
    eng.capture()
    stage = [gt.clone() for _ in range(2)]
    hosts = [gt.cpu().pin_memory() for _ in range(2)]
    outp = torch.empty((L, len(cams))).pin_memory()
    cp = torch.cuda.Stream()
    ev_copy = [torch.cuda.Event() for _ in range(2)]
    ev_free = [torch.cuda.Event() for _ in range(2)]
    st = {"k": 0}

    def step_e():
        k = st["k"]
        i = k % 2
        cs = torch.cuda.current_stream()
        cs.wait_event(ev_copy[i]) if k > 0 else stage[i].copy_(hosts[i], non_blocking=True)
        eng.gt0.copy_(stage[i])
        ev_free[i].record(cs)
        cp.wait_event(ev_free[1 - i]) if k > 0 else cp.wait_stream(cs)
        with torch.cuda.stream(cp):
            stage[1 - i].copy_(hosts[1 - i], non_blocking=True)
            ev_copy[1 - i].record(cp)
        eng.replay()
        outp.copy_(eng.graph_losses, non_blocking=True)
        st["k"] = k + 1
    out["E_graph_plus_eager_copies_ms"] = timed(step_e)
    del eng
    # F: two compute-only graphs (graph i reads target buffer i directly: no D2D copy); the next
    # step's H2D and this step's loss D2H on the copy stream, off the compute stream
    eng = MappingEngine(perturb(scene, 99), cams, gt, n_levels=cfg["levels"])
    bufs = [eng.gt0, torch.empty_like(eng.gt0)]
    gr = []
    for i in range(2):
        eng.gt0 = bufs[i]
        gr.append((eng.capture(), eng.graph_losses))
    outs = [torch.empty((L, len(cams))).pin_memory() for _ in range(2)]
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_done = [torch.cuda.Event() for _ in range(2)]
    st2 = {"k": 0}

    def step_f():
        k = st2["k"]
        i = k % 2
        cs = torch.cuda.current_stream()
        if k == 0:
            bufs[i].copy_(hosts[i], non_blocking=True)
            cp.wait_stream(cs)
        else:
            cs.wait_event(ev_in[i])
            cp.wait_event(ev_done[1 - i])  # step k - 1 is done with buffer 1 - i
        with torch.cuda.stream(cp):  # the next step's targets, during this step
            bufs[1 - i].copy_(hosts[1 - i], non_blocking=True)
            ev_in[1 - i].record(cp)
        gr[i][0].replay()
        ev_done[i].record(cs)
        cp.wait_event(ev_done[i])
        with torch.cuda.stream(cp):  # this step's losses, off the compute stream
            outs[i].copy_(gr[i][1], non_blocking=True)
        st2["k"] = k + 1

    def timed_f():
        for _ in range(3):
            step_f()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(K):
            step_f()
        torch.cuda.current_stream().wait_stream(cp)
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / K
    out["F_two_graphs_copies_off_stream_ms"] = timed_f()
    del eng
    eng = MappingEngine(perturb(scene, 99), cams, gt, n_levels=cfg["levels"])
    gp = gt.cpu().pin_memory()
    op = torch.empty((L, len(cams))).pin_memory()
    eng.capture(gp, op)
    out["D_replay_host_serial_ms"] = timed(eng.replay)
    out["h2d_MB"] = gt.numel() * 4 / 1e6
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main(*(sys.argv[1:2] or ["tum"]))
