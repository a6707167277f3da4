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


# ------------------------------------------------------------------ sharded optimiser (f3)
def _row_lr(row: int) -> float:
    # per-class rates of AdamConfig() in the [K][ld] row order (R20)
    from paper_2311_16728_b200.core import AdamConfig
    c = AdamConfig()
    lrs = [c.lr_means, c.lr_quats, c.lr_log_scales, c.lr_opacity, c.lr_sh_dc, c.lr_sh_rest]
    cls = 0 if row < 3 else 1 if row < 7 else 2 if row < 10 else 3 if row == 10 else 4 if row < 14 else 5
    return lrs[cls]


def _oracle_adam_rows(P, G, M, V, r0, r1, step):
    """fp64 oracle Adam on parameter rows [r0, r1) (M, V hold those rows only)."""
    import oracle.oracle as orc
    for r in range(r0, r1):
        p, m, v = orc.adam(P[r].numpy(), G[r].numpy(), M[r - r0].numpy(), V[r - r0].numpy(), lr=_row_lr(r), step=step)
        P[r] = torch.from_numpy(p)
        M[r - r0] = torch.from_numpy(m)
        V[r - r0] = torch.from_numpy(v)
        G[r] = 0.0


STEPS = 3


def _step_grad(g: torch.Tensor, step: int) -> torch.Tensor:
    """A different per-rank gradient every step (the engine's backward output changes as the map
    moves), so a stale row from an earlier step cannot cancel out."""
    return g * (1.0 + 0.5 * step)


def _sharded_worker(rank, world, port, out_dir):
    from paper_2311_16728_b200.mapping import ShardedAdam, row_shard
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        scene, cams, G = _views()
        K, n = 14, scene.means.shape[0]  # D = 0 (tiny): 11 + 3 rows
        mine = shard_views(len(cams), rank, world)
        g = torch.from_numpy(_flat_grad(scene, [cams[v] for v in mine], G[mine]).reshape(K, n).copy())
        p0 = np.concatenate([scene.means.T, scene.quats.T, scene.log_scales.T, scene.opacity_logits[None],
                             scene.sh.reshape(n, -1).T]).astype(np.float64)
        R, _, _ = row_shard(K, rank, world)
        pp = torch.zeros((world * R, n), dtype=torch.float64)
        pp[:K] = torch.from_numpy(p0)
        pg = torch.zeros_like(pp)
        opt = ShardedAdam(pp, pg, n, 0)
        opt.m = torch.zeros((opt.R, n), dtype=torch.float64)
        opt.v = torch.zeros_like(opt.m)
        # gs_adam_step_rows semantics, zero_grads=False as ShardedAdam calls it: only this rank's
        # rows of params / moments change, the gradient rows are left as they are
        opt._adam_rows = lambda: _oracle_adam_rows(opt.params, opt.grads.clone(), opt.m, opt.v, opt.r0, opt.r1, opt.t)
        # replicated path in the same process: all-reduce of the full gradient, Adam on every row
        P = torch.from_numpy(p0.copy())
        Pg = torch.zeros_like(P)
        M, V = torch.zeros_like(P), torch.zeros_like(P)
        traj_s, traj_r = [], []
        for step in range(STEPS):
            gs = _step_grad(g, step)
            pg[:K] += gs           # the engine's backward ADDS into the gradient buffer (gs.h)
            opt.step()
            Pg += gs
            dist.all_reduce(Pg)
            _oracle_adam_rows(P, Pg, M, V, 0, K, step + 1)   # zeroes Pg (zero_grads=True)
            traj_s.append(opt.params.numpy().copy())
            traj_r.append(P.numpy().copy())
            assert float(pg.abs().max()) == 0.0  # nothing left over for the next +=
        np.save(os.path.join(out_dir, f"sp{rank}.npy"), np.stack(traj_s))
        np.save(os.path.join(out_dir, f"rp{rank}.npy"), np.stack(traj_r))
        np.save(os.path.join(out_dir, f"rows{rank}.npy"), np.array([opt.r0, opt.r1]))
    finally:
        dist.destroy_process_group()


def test_row_shard_partition():
    from paper_2311_16728_b200.mapping import row_shard
    for K in (14, 59):
        for world in (1, 2, 3, 8):
            rows = [row_shard(K, r, world) for r in range(world)]
            R = rows[0][0]
            assert all(x[0] == R for x in rows) and R * world >= K
            covered = [i for _, a, b in rows for i in range(a, b)]
            assert covered == list(range(K))


def test_gloo_world2_sharded_adam_equals_replicated(tmp_path):
    """reduce-scatter -> row-sharded Adam -> all-gather, with the engine's += gradient pattern over
    3 steps, gives every rank the parameters of the replicated all-reduce + full Adam path bit for
    bit at every step (the update is elementwise), and both equal the batched oracle."""
    world = 2
    mp.start_processes(_sharded_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    s0, s1 = np.load(tmp_path / "sp0.npy"), np.load(tmp_path / "sp1.npy")
    rp0 = np.load(tmp_path / "rp0.npy")
    assert np.array_equal(s0, s1)            # replicas identical
    assert np.array_equal(s0, rp0)           # sharded == replicated, every step, bitwise
    r0, r1 = np.load(tmp_path / "rows0.npy"), np.load(tmp_path / "rows1.npy")
    assert r0[0] == 0 and r0[1] == r1[0] and r1[1] == 14
    # batched reference: one process, gradient summed over all views (R22), full Adam on every row
    scene, cams, G = _views()
    K, n = 14, scene.means.shape[0]
    g = torch.from_numpy(_flat_grad(scene, cams, G).reshape(K, n).copy())
    P = torch.from_numpy(np.concatenate([scene.means.T, scene.quats.T, scene.log_scales.T,
                                         scene.opacity_logits[None], scene.sh.reshape(n, -1).T]).astype(np.float64))
    M, V = torch.zeros_like(P), torch.zeros_like(P)
    for step in range(STEPS):
        _oracle_adam_rows(P, _step_grad(g, step).clone(), M, V, 0, K, step + 1)
        np.testing.assert_allclose(s0[step], P.numpy(), rtol=1e-12, atol=1e-15)


def _stale_worker(rank, world, port, out_dir):
    """The pre-fix ShardedAdam (only this rank's gradient rows zeroed after the step): the
    regression the fixed step must not show."""
    from paper_2311_16728_b200.mapping import ShardedAdam
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        K, n = 14, 8
        pp = torch.zeros((K, n), dtype=torch.float64)
        pg = torch.zeros_like(pp)
        opt = ShardedAdam(pp, pg, n, 0)

        def sgd_rows():  # SGD with lr 1 on this rank's rows
            opt.params[opt.r0:opt.r1] -= opt.grads[opt.r0:opt.r1]
        opt._adam_rows = sgd_rows
        for _ in range(3):
            pg[:K] += 1.0 + rank  # per-rank gradient (sum over ranks = 3)
            opt.step()
        np.save(os.path.join(out_dir, f"stale{rank}.npy"), opt.params.numpy())
    finally:
        dist.destroy_process_group()


def test_gloo_world2_sharded_step_leaves_no_stale_gradient(tmp_path):
    """3 SGD steps of the summed gradient 3 move every row to exactly -9 (a stale row re-added
    in later steps gives -18 and more)."""
    mp.start_processes(_stale_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True,
                       start_method="spawn")
    for r in range(2):
        assert np.array_equal(np.load(tmp_path / f"stale{r}.npy"), np.full((14, 8), -9.0))


def _state_worker(rank, world, port, out_dir):
    from paper_2311_16728_b200.mapping import ShardedAdam
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        K, n = 14, 5
        R = 7
        pp = torch.zeros((world * R, n), dtype=torch.float64)
        opt = ShardedAdam(pp, torch.zeros_like(pp), n, 0)
        opt.m = torch.zeros((opt.R, n), dtype=torch.float64)
        opt.v = torch.zeros_like(opt.m)
        rows = torch.arange(opt.r0, opt.r1, dtype=torch.float64)[:, None]
        opt.m[:opt.r1 - opt.r0] = rows * 10 + torch.arange(n)
        opt.v[:opt.r1 - opt.r0] = -(rows * 10 + torch.arange(n))
        m, v = opt.full_state()
        np.save(os.path.join(out_dir, f"m{rank}.npy"), m.numpy())
        # densification: a new map of n' = 3 Gaussians with full moments; each rank keeps its rows
        m_new = torch.arange(world * R * 3, dtype=torch.float64).view(world * R, 3)
        pp2 = torch.zeros((world * R, 3), dtype=torch.float64)
        opt.rebind(pp2, torch.zeros_like(pp2), 3, m_new, -m_new)
        np.save(os.path.join(out_dir, f"mine{rank}.npy"), opt.m.numpy())
        np.save(os.path.join(out_dir, f"v{rank}.npy"), v.numpy())
    finally:
        dist.destroy_process_group()


def test_gloo_world2_sharded_state_gather_and_rebind(tmp_path):
    """Densification under the row-sharded optimiser: full_state() all-gathers every rank's
    moment rows into the full layout; rebind() keeps exactly this rank's rows of the new map's
    moments (rows [r0, r1), zero padding after)."""
    mp.start_processes(_state_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True,
                       start_method="spawn")
    want = np.arange(14)[:, None] * 10.0 + np.arange(5)
    for r in range(2):
        m = np.load(tmp_path / f"m{r}.npy")
        assert np.array_equal(m[:14], want)
        assert np.array_equal(np.load(tmp_path / f"v{r}.npy")[:14], -want)
        mine = np.load(tmp_path / f"mine{r}.npy")
        full = np.arange(14 * 3, dtype=np.float64).reshape(14, 3)
        assert np.array_equal(mine, full[7 * r:7 * (r + 1)])


def test_comm_shard_partition():
    """gs_comm_shard (C ABI, host arithmetic): the world ranges tile [0, K ld) in order, each a
    whole number of float4s, every rank but the last the same length."""
    from paper_2311_16728_b200.comm import comm_shard
    from paper_2311_16728_b200 import _lib as L
    from paper_2311_16728_b200.core import param_rows
    for n, D in ((1, 0), (1000, 0), (200_000, 3), (77, 2)):
        total = param_rows(D) * L.param_ld(n)
        for world in (1, 2, 3, 8):
            rs = [comm_shard(n, D, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            assert all(e0 % 4 == 0 and e1 % 4 == 0 for e0, e1 in rs)
            assert len({e1 - e0 for e0, e1 in rs[:-1]}) <= 1
    with pytest.raises(L.GsError):
        comm_shard(10, 0, 2, 2)
