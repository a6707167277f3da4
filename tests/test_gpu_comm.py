"""The fused data-parallel optimiser step over peer memory (comm.cu,
gs_reduce_adam_bcast between two gs_peer_barrier) on one GPU: an NCCL process group of one rank
with torch symmetric memory.  At world size 1 the kernel is exactly gs_adam_step (same
arithmetic, bit for bit); the engine with comm='peer' optimises like the single-GPU engine,
replays as a CUDA graph and densifies.  (More ranks need more GPUs than the pool gives: the
multi-rank sum / broadcast is unmeasured on hardware.)"""
import numpy as np
import pytest
import torch
import torch.distributed as dist

from paper_2311_16728_b200 import _lib as L
from paper_2311_16728_b200.core import Adam, AdamConfig, DensifyConfig, Renderer, pack_params
from paper_2311_16728_b200.mapping import MappingEngine
from synth import make_cameras, make_scene, perturb

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pg(tmp_path_factory):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2311_16728_b200.build import build
    build()
    L.lib()
    path = tmp_path_factory.mktemp("pg") / "store"
    dist.init_process_group("nccl", init_method=f"file://{path}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    yield dist.group.WORLD
    dist.destroy_process_group()


@pytest.mark.parametrize("sgd", [False, True])
def test_peer_adam_world1_equals_adam_step(pg, sgd):
    from paper_2311_16728_b200.comm import PeerAdam
    scene = make_scene("tum", n=3001)
    n, D = scene.n, 3
    cfg = AdamConfig(sgd=sgd, lr_means=1e-2)
    peer = PeerAdam(n, D, cfg)
    p0 = pack_params(scene)
    peer.params.copy_(p0)
    ref_p = p0.clone()
    ref = Adam(ref_p, n, D, cfg)
    gen = torch.Generator("cuda").manual_seed(3)
    for step in range(3):
        g = torch.randn(p0.shape, device="cuda", generator=gen)
        g[:, n:] = 0
        peer.grads.copy_(g)
        peer.step()
        ref.step(g.clone(), zero_grads=True)
        torch.cuda.synchronize()
        assert torch.equal(peer.params, ref_p), step
        assert float(peer.grads.abs().max()) == 0.0
        if not sgd:
            m, v = peer.full_state()
            assert torch.equal(m, ref.m) and torch.equal(v, ref.v)
    assert peer.t == 3


def _engines(comm):
    scene = make_scene("tiny")
    cams = make_cameras("tiny", 1)
    r = Renderer(scene.n, 0, 1, cams[0].width, cams[0].height, 1 << 16)
    gt = r.forward(pack_params(scene), cams)[0].clone()
    return MappingEngine(perturb(scene, 4), cams, gt, n_levels=1, comm=comm, shard_optimizer=False,
                         densify_cfg=DensifyConfig(grad_threshold=1e-3, scene_extent=1.0))


def test_engine_peer_step_matches_single_gpu_and_replays(pg):
    eng = _engines("peer")
    assert eng.peer is not None and eng.adam is None
    ref = _engines("nccl")  # replicated all-reduce of a one-rank group: the reference optimiser path
    for _ in range(4):
        la = [x.item() for x in eng.step()]
        lb = [x.item() for x in ref.step()]
        np.testing.assert_allclose(la, lb, rtol=1e-4)
    n = eng.n
    # the raster backward's fp32 atomics add in no fixed order: trajectories agree to rounding
    torch.testing.assert_close(eng.params[:, :n], ref.params[:, :n], rtol=1e-4, atol=1e-5)
    eng.capture()  # no NCCL call inside the peer step: capturable
    before = eng.peer.t
    for _ in range(3):
        eng.replay()
    torch.cuda.synchronize()
    assert eng.peer.t == before + 3 * 2  # two levels per step
    assert torch.isfinite(eng.params[:, :n]).all()


def test_engine_peer_densify(pg):
    eng = _engines("peer")
    for _ in range(5):
        eng.build_pyramids()
        eng.step()
    t = eng.peer.t
    m0, _ = eng._moments()
    nc, ns, npr = eng.densify_and_prune(seed=2)
    assert nc + ns > 0 and eng.peer.n == eng.n and eng.peer.t == t
    m1, _ = eng._moments()
    assert m1.shape[1] == eng.params.shape[1] and float(m1.abs().sum()) > 0
    for _ in range(2):
        eng.build_pyramids()
        assert np.isfinite([x.item() for x in eng.step()]).all()


@pytest.mark.parametrize("world", [2, 3, 8])
def test_reduce_adam_bcast_multi_rank_arithmetic(world):
    """The peer path of gs_reduce_adam_bcast for `world` ranks, emulated on one GPU without the
    barriers (nothing waits on anything): `world` parameter / gradient buffers on this device
    stand for the ranks' symmetric buffers; calling the kernel for every rank in turn must leave
    every rank's parameters equal to one gs_adam_step on the summed gradient, every gradient
    buffer zeroed, and each rank's moment shard equal to its range of the full moments."""
    from paper_2311_16728_b200.comm import comm_shard
    scene = make_scene("tum", n=5003)
    n, D = scene.n, 3
    cfg = AdamConfig(lr_means=1e-2)
    p0 = pack_params(scene)
    K, ld = p0.shape
    gen = torch.Generator("cuda").manual_seed(5)
    params = [p0.clone() for _ in range(world)]
    grads = [torch.randn(p0.shape, device="cuda", generator=gen) for _ in range(world)]
    for g in grads:
        g[:, n:] = 0
    gsum = torch.stack(grads).sum(0)  # rank order 0..world-1, as the kernel sums
    gsum_seq = grads[0].clone()
    for g in grads[1:]:
        gsum_seq += g
    ref_p = p0.clone()
    ref = Adam(ref_p, n, D, cfg)
    ref.step(gsum_seq.clone(), zero_grads=True)
    shards = []
    for r in range(world):
        e0, e1 = comm_shard(n, D, r, world)
        q = -(-(K * ld) // 4 // world) * 4
        m = torch.zeros(q, device="cuda")
        v = torch.zeros(q, device="cuda")
        L.gs_reduce_adam_bcast(L.params_struct(params[r], n, D), [p.data_ptr() for p in params],
                               [g.data_ptr() for g in grads], 0, 0, m, v, cfg.struct(), 1, None, r, world)
        shards.append((e0, e1, m, v))
    torch.cuda.synchronize()
    for r in range(world):
        assert torch.equal(params[r], ref_p), r
        assert float(grads[r].abs().max()) == 0.0
    mflat, vflat = ref.m.reshape(-1), ref.v.reshape(-1)
    for e0, e1, m, v in shards:
        assert torch.equal(m[:e1 - e0], mflat[e0:e1]) and torch.equal(v[:e1 - e0], vflat[e0:e1])


@pytest.mark.parametrize("sgd", [False, True])
def test_adam_step_rows_dev_equals_host_step(pg, sgd):
    """gs_adam_step_rows_dev (step counter on the device, advanced by the call) takes the same
    steps, bit for bit, as gs_adam_step_rows with the host's 1-based counter."""
    scene = make_scene("tum", n=2003)
    n, D = scene.n, 3
    cfg = AdamConfig(sgd=sgd, lr_means=1e-2)
    hp = cfg.struct()
    p0 = pack_params(scene)
    K = p0.shape[0]
    r0, r1 = 4, 41
    pa, pb = p0.clone(), p0.clone()
    ma, va = torch.zeros((r1 - r0, p0.shape[1]), device="cuda"), torch.zeros((r1 - r0, p0.shape[1]), device="cuda")
    mb, vb = ma.clone(), va.clone()
    t_dev = torch.zeros(1, dtype=torch.int64, device="cuda")
    gen = torch.Generator("cuda").manual_seed(7)
    for step in range(1, 4):
        g = torch.randn(p0.shape, device="cuda", generator=gen)
        L.gs_adam_step_rows(L.params_struct(pa, n, D), g, ma, va, hp, step, r0, r1, False)
        L.gs_adam_step_rows_dev(L.params_struct(pb, n, D), g, mb, vb, hp, t_dev, r0, r1, False)
        torch.cuda.synchronize()
        assert torch.equal(pa, pb) and int(t_dev.item()) == step
        if not sgd:
            assert torch.equal(ma, mb) and torch.equal(va, vb)
    assert torch.equal(pa[:r0], p0[:r0]) and torch.equal(pa[r1:K], p0[r1:K])  # other rows untouched


def test_engine_sharded_nccl_step_captures_and_replays(pg):
    """The row-sharded NCCL DP step (reduce-scatter -> Adam on the rank's rows -> all-gather ->
    zeroed gradients) captured in a CUDA graph: replays continue the eager trajectory (same
    losses as an engine stepping eagerly from the same state) and count steps on the device."""
    def make():
        scene = make_scene("tiny")
        cams = make_cameras("tiny", 1)
        r = Renderer(scene.n, 0, 1, cams[0].width, cams[0].height, 1 << 16)
        gt = r.forward(pack_params(scene), cams)[0].clone()
        return MappingEngine(perturb(scene, 4), cams, gt, n_levels=1, comm="nccl", shard_optimizer=True)
    eng, ref = make(), make()
    assert eng.sharded is not None
    for _ in range(2):
        eng.step()
        ref.step()
    eng.capture()  # also runs one (warm-up) step
    ref.step()
    assert eng.sharded.t == ref.sharded.t
    for _ in range(3):
        eng.replay()
        lb = [x.item() for x in ref.step()]
    torch.cuda.synchronize()
    la = eng.graph_losses.cpu().numpy().reshape(-1)
    np.testing.assert_allclose(la, np.ravel(lb), rtol=1e-3)
    assert eng.sharded.t == ref.sharded.t == 2 * 6
    n = eng.n
    torch.testing.assert_close(eng.params[:, :n], ref.params[:, :n], rtol=1e-4, atol=1e-5)
