"""GPU parity of densify and prune against the oracle, the
statistics kernel, and the mapping engine with densification (decisions in fp32 on both sides:
classes and counts must match exactly; copies bitwise; new positions / log-scales to rounding)."""
import numpy as np
import pytest
import torch

import oracle.oracle as orc
from paper_2311_16728_b200 import _lib as L
from paper_2311_16728_b200.core import DensifyConfig, Renderer, densify, pack_params
from paper_2311_16728_b200.mapping import MappingEngine
from synth import densify_samples, make_cameras, make_scene, perturb

pytestmark = pytest.mark.gpu


def _records(t: torch.Tensor, n: int) -> np.ndarray:
    return t[:, :n].T.contiguous().cpu().numpy()


@pytest.mark.parametrize("n,extent", [(6000, 2.0), (777, 0.5)])
def test_densify_matches_oracle(n, extent):
    scene = make_scene("tum", n=n)
    rng = np.random.default_rng(n)
    vis = rng.integers(0, 5, n).astype(np.float32)
    ga = (rng.uniform(0, 2e-3, n) * vis).astype(np.float32)
    mr = rng.integers(0, 400, n).astype(np.int32)
    scene.opacity_logits[rng.choice(n, n // 30, replace=False)] = -7.0
    small = rng.choice(n, n // 2, replace=False)  # half small enough to clone, the rest mostly split
    scene.log_scales[small] = np.log(rng.uniform(0.001, 0.004, (small.size, 3))).astype(np.float32)
    z = densify_samples(n, 11)
    params = pack_params(scene)
    gen = torch.Generator("cuda").manual_seed(2)
    m = torch.randn(params.shape, device="cuda", generator=gen)
    v = torch.rand(params.shape, device="cuda", generator=gen)
    c = DensifyConfig(grad_threshold=5e-4, scene_extent=extent).struct(640, 480)
    cuda = lambda a: torch.from_numpy(a).cuda()  # noqa: E731
    new_p, new_m, new_v, counts = densify(params, n, 3, m, v, cuda(ga), cuda(vis), cuda(mr), cuda(z), c)
    ref = orc.densify(orc.scene_records(scene), _records(m, n), _records(v, n), ga, vis, mr, z, c.grad_threshold,
                      c.percent_dense, c.scene_extent, c.opacity_threshold, c.max_screen_px)
    assert counts == (ref["n_clone"], ref["n_split"], ref["n_prune"], ref["n_new"])
    assert min(counts[:3]) > 0  # every branch exercised
    nn = counts[3]
    got, gm, gv = _records(new_p, nn), _records(new_m, nn), _records(new_v, nn)
    nk = nn - ref["n_clone"] - 2 * ref["n_split"]
    assert np.array_equal(got[:nk], ref["rec"][:nk].astype(np.float32))  # kept originals: bitwise
    assert np.array_equal(gm[:nk], ref["m"][:nk].astype(np.float32))
    assert np.array_equal(gv[:nk], ref["v"][:nk].astype(np.float32))
    assert (gm[nk:] == 0).all() and (gv[nk:] == 0).all()
    new, rnew = got[nk:].astype(np.float64), ref["rec"][nk:]
    np.testing.assert_allclose(new[:, :3], rnew[:, :3], rtol=0, atol=2e-6)       # P + R S z (fp32)
    np.testing.assert_allclose(new[:, 7:10], rnew[:, 7:10], rtol=0, atol=2e-6)   # log s (- ln 1.6)
    assert np.array_equal(new[:, 3:7], rnew[:, 3:7]) and np.array_equal(new[:, 10:], rnew[:, 10:])
    # untouched rows of the padded layout stay zero
    assert (new_p[:, nn:] == 0).all()


def test_densify_everything_pruned_and_noop():
    scene = make_scene("tiny", n=100)
    params = pack_params(scene)
    n = 100
    z = torch.from_numpy(densify_samples(n, 1)).cuda()
    zeros = torch.zeros(n, device="cuda")
    mr = torch.zeros(n, dtype=torch.int32, device="cuda")
    c = DensifyConfig(opacity_threshold=0.999).struct(64, 48)  # every sigmoid(logit) < 0.999? logit <= 4
    p, _, _, counts = densify(params, n, 0, None, None, zeros, zeros, mr, z, c)
    assert counts == (0, 0, n, 0)
    c = DensifyConfig(opacity_threshold=1e-6).struct(64, 48)
    p, _, _, counts = densify(params, n, 0, None, None, zeros, zeros, mr, z, c)
    assert counts == (0, 0, 0, n) and torch.equal(p[:, :n], params[:, :n])


def test_densify_stats_counts_visible_views():
    scene = make_scene("tum", n=20000)
    cams = make_cameras("tum", 3)
    params = pack_params(scene)
    r = Renderer(scene.n, 3, 3, cams[0].width, cams[0].height, 1 << 20)
    r.forward(params, cams)
    vc = torch.zeros(scene.n, device="cuda")
    mr = torch.full((scene.n,), 2, dtype=torch.int32, device="cuda")
    ps = L.params_struct(params, scene.n, 3)
    L.gs_densify_stats(ps, cams, r.ws.buf, vc, mr)
    L.gs_densify_stats(ps, cams, r.ws.buf, vc, mr)
    rad = r.ws.views()["radius"].view(3, scene.n)
    assert torch.equal(vc, 2 * (rad > 0).sum(0).float())
    assert torch.equal(mr, torch.maximum(rad.max(0).values, torch.full_like(mr, 2)))
    with pytest.raises(L.GsError) as e:
        L.gs_densify_stats(ps, cams[:2], r.ws.buf, vc, mr)
    assert e.value.status in (L.GS_ERR_STALE_STATE, L.GS_ERR_SHAPE)


def test_mapping_engine_densify_and_prune():
    scene = make_scene("tiny")
    cams = make_cameras("tiny", 1)
    params = pack_params(scene)
    r = Renderer(scene.n, 0, 1, cams[0].width, cams[0].height, 1 << 16)
    gt = r.forward(params, cams)[0].clone()
    start = perturb(scene, 4)
    eng = MappingEngine(start, cams, gt, n_levels=1, densify_cfg=DensifyConfig(grad_threshold=1e-3, scene_extent=1.0))
    for _ in range(6):
        eng.build_pyramids()
        eng.step()
    n0 = eng.n
    assert eng.vis_count.sum().item() > 0 and eng.grad2d_norm.sum().item() > 0
    nc, ns, npr = eng.densify_and_prune(seed=3)
    assert eng.n == n0 - npr + nc + ns and nc + ns > 0
    assert eng.params.shape[1] >= eng.n and eng.adam.m.shape == eng.params.shape
    assert eng.vis_count.sum().item() == 0
    losses = []
    for _ in range(4):
        eng.build_pyramids()
        losses.append([x.item() for x in eng.step()])
    assert np.isfinite(np.array(losses)).all()


# ------------------------------------------------------------------ f2: geometry-based densification
@pytest.mark.parametrize("mode", [0, 1])
def test_geometry_densify_matches_oracle(mode):
    from paper_2311_16728_b200.core import geometry_densify
    from synth import make_keypoints
    cam = make_cameras("tum", 1)[0]
    uv, active, kd, depth, img = make_keypoints(cam, 1500, 5)
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    out, cnt, src = geometry_densify(cam, cu(uv), cu(active), cu(kd), cu(depth) if mode else None, cu(img), mode, 3)
    ref = orc.geometry_densify(cam, uv, active, kd, depth if mode else None, img, mode, D=3)
    assert cnt == ref["count"] > 100
    assert np.array_equal(src.cpu().numpy(), ref["src"])
    got = _records(out, cnt).astype(np.float64)
    r = ref["rec"]
    np.testing.assert_allclose(got[:, :3], r[:, :3], rtol=2e-7, atol=1e-6)        # back-projection (fp64 -> fp32)
    assert np.array_equal(got[:, 3:7], r[:, 3:7])
    np.testing.assert_allclose(got[:, 7:14], r[:, 7:14], rtol=2e-7, atol=1e-6)   # log s, logit, SH DC
    assert (got[:, 14:] == 0).all()


def test_densify_tags_follow_their_gaussians():
    scene = make_scene("tum", n=3000)
    n = scene.n
    rng = np.random.default_rng(9)
    vis = np.full(n, 2, np.float32)
    ga = (rng.uniform(0, 2e-3, n) * 2).astype(np.float32)
    mr = np.zeros(n, np.int32)
    scene.opacity_logits[rng.choice(n, 100, replace=False)] = -7.0
    small = rng.choice(n, n // 2, replace=False)
    scene.log_scales[small] = np.log(0.002)
    z = densify_samples(n, 4)
    params = pack_params(scene)
    tags = torch.from_numpy(rng.integers(0, 200, n).astype(np.uint8)).cuda()
    c = DensifyConfig(grad_threshold=5e-4, scene_extent=1.0).struct(640, 480)
    cuda = lambda a: torch.from_numpy(a).cuda()  # noqa: E731
    _, _, _, counts, new_tags = densify(params, n, 3, None, None, cuda(ga), cuda(vis), cuda(mr), cuda(z), c, tags=tags)
    ref = orc.densify(orc.scene_records(scene), np.zeros((n, 59), np.float32), np.zeros((n, 59), np.float32), ga, vis,
                      mr, z, c.grad_threshold, c.percent_dense, c.scene_extent, c.opacity_threshold, c.max_screen_px)
    cls, t = ref["cls"], tags.cpu().numpy()
    expect = np.concatenate([t[cls <= 1], t[cls == 1], np.repeat(t[cls == 2], 2)])
    assert counts[3] == expect.size and np.array_equal(new_tags[:counts[3]].cpu().numpy(), expect)


def test_mapping_engine_geometry_densify():
    from synth import make_keypoints
    scene = make_scene("tiny")
    cams = make_cameras("tiny", 1)
    params = pack_params(scene)
    r = Renderer(scene.n, 0, 1, cams[0].width, cams[0].height, 1 << 16)
    gt = r.forward(params, cams)[0].clone()
    eng = MappingEngine(perturb(scene, 4), cams, gt, n_levels=1,
                        densify_cfg=DensifyConfig(grad_threshold=1e-3, scene_extent=1.0))
    uv, active, kd, depth, img = make_keypoints(cams[0], 120, 2)
    n0 = eng.n
    added = eng.add_keyframe_features(0, uv, active, kd, depth, img, mode=1)
    assert added > 0 and eng.n == n0 + added
    assert int(eng.temporary[:eng.n].sum().item()) == added  # flags follow their primitives (any layout)
    for _ in range(3):
        eng.build_pyramids()
        losses = [x.item() for x in eng.step()]
    assert np.isfinite(losses).all()
    nc, ns, npr = eng.densify_and_prune(seed=1)
    assert eng.temporary.shape[0] >= eng.n


def test_mapping_engine_densify_with_row_sharded_optimizer(tmp_path):
    """Densify and prune with shard_optimizer=True (NCCL process group of one rank, so the
    reduce-scatter / all-gather are real NCCL calls): the new map and its Adam moments equal what
    core.densify makes of the engine's state before the call (moments all-gathered from the
    shards), bit for bit; the engine keeps stepping afterwards."""
    import torch.distributed as dist
    from paper_2311_16728_b200.core import permute_columns
    from paper_2311_16728_b200.core import spatial_order as sorder
    from paper_2311_16728_b200.levels import densify_samples as dsamples
    dist.init_process_group("nccl", init_method=f"file://{tmp_path}/pg", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        scene = make_scene("tiny")
        cams = make_cameras("tiny", 1)
        r = Renderer(scene.n, 0, 1, cams[0].width, cams[0].height, 1 << 16)
        gt = r.forward(pack_params(scene), cams)[0].clone()
        cfg = DensifyConfig(grad_threshold=1e-3, scene_extent=1.0)
        eng = MappingEngine(perturb(scene, 4), cams, gt, n_levels=1, densify_cfg=cfg)
        assert eng.sharded is not None and eng.adam is None
        for _ in range(6):
            eng.build_pyramids()
            eng.step()
        n = eng.n
        m, v = eng._moments()
        assert float(m[:, :n].abs().sum()) > 0  # the sharded Adam has stepped
        z = torch.from_numpy(dsamples(n, 3)).cuda()
        p_e, m_e, v_e, counts, _ = densify(eng.params.clone(), n, 0, m.clone(), v.clone(), eng.grad2d_norm.clone(),
                                           eng.vis_count.clone(), eng.max_radius.clone(), z,
                                           cfg.struct(cams[0].width, cams[0].height), tags=eng.temporary.clone())
        nn = counts[3]
        perm = sorder(p_e, nn, 0)
        p_e, m_e, v_e = (permute_columns(x, perm, nn) for x in (p_e, m_e, v_e))
        nc, ns, npr = eng.densify_and_prune(seed=3)
        assert (nc, ns, npr) == counts[:3] and nc + ns > 0 and eng.n == nn
        m2, v2 = eng._moments()
        assert torch.equal(eng.params[:, :nn], p_e[:, :nn])
        assert torch.equal(m2[:, :nn], m_e[:, :nn]) and torch.equal(v2[:, :nn], v_e[:, :nn])
        assert float(eng.grads.abs().max()) == 0.0
        for _ in range(3):
            eng.build_pyramids()
            losses = [x.item() for x in eng.step()]
        assert np.isfinite(losses).all()
        # geometry densification under the sharded optimiser: moments of the old map carried over
        from synth import make_keypoints
        uv, active, kd, depth, img = make_keypoints(cams[0], 120, 2)
        n0 = eng.n
        m0, _ = eng._moments()
        mass = float(m0[:, :n0].abs().sum())
        added = eng.add_keyframe_features(0, uv, active, kd, depth, img, mode=1)
        assert added > 0 and eng.n == n0 + added
        m1, _ = eng._moments()
        assert abs(float(m1[:, :eng.n].abs().sum()) - mass) <= 1e-6 * mass  # same values, new order
        eng.build_pyramids()
        assert np.isfinite([x.item() for x in eng.step()]).all()
    finally:
        dist.destroy_process_group()


def test_mapping_engine_add_keyframe_keeps_state():
    """Keyframes arrive one at a time: add_keyframe grows the batch; parameters
    and Adam state carry on; an iteration then renders and optimises both views."""
    scene = make_scene("tiny")
    cams = make_cameras("tiny", 2)
    params = pack_params(scene)
    r = Renderer(scene.n, 0, 2, cams[0].width, cams[0].height, 1 << 16)
    gts = r.forward(params, cams)[0].clone()
    eng = MappingEngine(perturb(scene, 4), cams[:1], gts[:1], n_levels=1)
    for _ in range(3):
        eng.step()
    p_before = eng.params.clone()
    m_before = eng.adam.m.clone()
    k = eng.add_keyframe(cams[1], gts[1])
    assert k == 1 and eng.V == 2 and eng.gt0.shape[0] == 2
    assert torch.equal(eng.params, p_before) and torch.equal(eng.adam.m, m_before)
    losses = eng.step()
    assert all(l.shape[0] == 2 for l in losses) and np.isfinite([l.cpu().numpy() for l in losses]).all()
    with pytest.raises(ValueError):
        eng.add_keyframe(make_cameras("tum", 1)[0], torch.zeros(3, 480, 640))
