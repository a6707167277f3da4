"""Data-parallel host logic on CPU (gloo, world_size 2): keyframe views are sharded over ranks
(SURVEY §8(e)), per-rank gradients are summed by the all-reduce (A10, R22) and every rank then
applies the identical optimiser step, so replicas stay bitwise equal.  The per-view gradients
come from the CPU oracle here (test infrastructure); on GPUs they come from libgs.so."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2311_16728_b200.mapping import reduce_gradients, shard_views


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _flat_grad(scene, cams, G):
    import oracle.oracle as orc
    g = orc.backward(scene, cams, G, "recipe")
    return np.concatenate([g[k].reshape(-1) for k in ("means", "quats", "log_scales", "opacity_logits", "sh")])


def _views():
    from synth import make_cameras, make_scene
    from tests.helpers import camera
    scene = make_scene("tiny", n=300)
    base = make_cameras("tiny", 1)[0]
    cams = []
    for v in range(4):
        t = base.t + np.array([0.03 * v, -0.02 * v, 0.05 * v], np.float32)
        cams.append(camera(fx=base.fx, fy=base.fy, cx=base.cx, cy=base.cy, width=base.width, height=base.height,
                           R=base.R, t=t, lim=base.lim_x))
    G = np.random.default_rng(0).normal(size=(4, 3, base.height, base.width))
    return scene, cams, G


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        scene, cams, G = _views()
        mine = shard_views(len(cams), rank, world)
        g = _flat_grad(scene, [cams[v] for v in mine], G[mine])
        t = torch.from_numpy(g.copy())
        reduce_gradients(t)
        p = np.concatenate([scene.means.reshape(-1), scene.quats.reshape(-1), scene.log_scales.reshape(-1),
                            scene.opacity_logits.reshape(-1), scene.sh.reshape(-1)]).astype(np.float64)
        p_new = p - 1e-3 * t.numpy()  # identical step on every rank
        np.save(os.path.join(out_dir, f"g{rank}.npy"), t.numpy())
        np.save(os.path.join(out_dir, f"p{rank}.npy"), p_new)
        np.save(os.path.join(out_dir, f"v{rank}.npy"), np.array(mine))
    finally:
        dist.destroy_process_group()


def test_shard_views_partition():
    for n in (1, 2, 5, 16, 64):
        for world in (1, 2, 3, 8):
            parts = [shard_views(n, r, world) for r in range(world)]
            flat = sorted(v for p in parts for v in p)
            assert flat == list(range(n))
            assert max(len(p) for p in parts) - min(len(p) for p in parts) <= 1


def test_reduce_is_noop_without_process_group():
    t = torch.ones(5)
    assert torch.equal(reduce_gradients(t), torch.ones(5))


def test_gloo_world2_allreduce_equals_batched_gradient(tmp_path):
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    g0, g1 = np.load(tmp_path / "g0.npy"), np.load(tmp_path / "g1.npy")
    p0, p1 = np.load(tmp_path / "p0.npy"), np.load(tmp_path / "p1.npy")
    v0, v1 = np.load(tmp_path / "v0.npy"), np.load(tmp_path / "v1.npy")
    assert sorted(list(v0) + list(v1)) == [0, 1, 2, 3] and not set(v0) & set(v1)
    assert np.array_equal(g0, g1) and np.array_equal(p0, p1)  # replicas bitwise equal
    scene, cams, G = _views()
    batched = _flat_grad(scene, cams, G)  # one process, all views (R22: sum over the batch)
    np.testing.assert_allclose(g0, batched, rtol=1e-9, atol=1e-12 * np.abs(batched).max())
