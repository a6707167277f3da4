"""Map layout (order.cu, include/gs.h gs_spatial_order / gs_permute_columns): the Morton
permutation against its definition recomputed in numpy float32, the column gather, and the
mapping engine giving the same optimisation with and without the spatial order."""
import numpy as np
import pytest
import torch

from paper_2311_16728_b200 import _lib as L
from paper_2311_16728_b200.core import Renderer, pack_params, permute_columns, spatial_order
from paper_2311_16728_b200.mapping import MappingEngine
from synth import make_cameras, make_scene, perturb

pytestmark = pytest.mark.gpu


def _spread3(x):
    out = np.zeros_like(x)
    for b in range(10):
        out |= ((x >> b) & 1) << (3 * b)
    return out


def _morton_ref(means: np.ndarray) -> np.ndarray:
    """gs.h definition: per axis cell = min(1023, (int)((x - lo) * (1024 / (hi - lo)))), fp32."""
    m = means.astype(np.float32)
    lo, hi = m.min(0), m.max(0)
    ext = (hi - lo).astype(np.float32)
    sc = np.where(ext > 0, np.float32(1024.0) / np.where(ext > 0, ext, np.float32(1)), np.float32(0)).astype(np.float32)
    t = ((m - lo).astype(np.float32) * sc).astype(np.float32)
    cell = np.clip(t.astype(np.int64), 0, 1023)
    return _spread3(cell[:, 0]) | _spread3(cell[:, 1]) << 1 | _spread3(cell[:, 2]) << 2


@pytest.mark.parametrize("n", [1, 37, 5000, 70000])
def test_spatial_order_is_stable_morton_sort(n):
    scene = make_scene("tum", n=n)
    params = pack_params(scene)
    perm = spatial_order(params, n, 3).cpu().numpy()
    assert np.array_equal(np.sort(perm), np.arange(n))
    codes = _morton_ref(scene.means)
    np.testing.assert_array_equal(perm, np.argsort(codes, kind="stable"))


def test_spatial_order_flat_axis_and_ties():
    scene = make_scene("tiny")
    scene.means[:, 2] = 2.0                     # flat axis -> cell 0
    scene.means[10:20] = scene.means[10]        # equal codes keep index order
    params = pack_params(scene)
    perm = spatial_order(params, scene.n, 0).cpu().numpy()
    np.testing.assert_array_equal(perm, np.argsort(_morton_ref(scene.means), kind="stable"))


def test_permute_columns_gathers_and_keeps_padding():
    g = torch.Generator().manual_seed(3)
    n, ld, K = 1000, 1024, 59
    a = torch.randn((K, ld), generator=g).cuda()
    perm = torch.randperm(n, generator=g).to(torch.int32).cuda()
    b = permute_columns(a, perm, n)
    assert torch.equal(b[:, :n], a[:, perm.long()])
    assert torch.equal(b[:, n:], a[:, n:])
    ints = torch.arange(n, dtype=torch.int32).cuda()
    assert torch.equal(permute_columns(ints, perm, n), perm)
    with pytest.raises(L.GsError):
        L.gs_permute_columns(a, a, ld, K, n, perm)   # src == dst


def test_engine_with_spatial_order_optimises_the_same_map():
    """The Morton layout changes where Gaussians sit in memory, not what the method computes:
    renders agree and three optimiser steps (SGD mode: -lr g, no Adam normalisation of
    last-bit noise) move every Gaussian the same way up to fp32 summation order."""
    from paper_2311_16728_b200.core import AdamConfig
    scene = make_scene("tum", n=30000)
    cams = make_cameras("tum", 1)
    params = pack_params(scene)
    r = Renderer(scene.n, 3, 1, cams[0].width, cams[0].height, 1 << 20)
    gt = r.forward(params, cams)[0].clone()
    start = perturb(scene, 5)
    cfg = AdamConfig(sgd=True)
    a = MappingEngine(start, cams, gt, n_levels=2, spatial_order=True, adam=cfg)
    b = MappingEngine(start, cams, gt, n_levels=2, spatial_order=False, adam=cfg)
    order = a.order
    assert torch.equal(a.params[:, :a.n], b.params[:, order])  # the same Gaussians, re-ordered
    p0 = b.params[:, order].clone()
    ra, _ = a.render(0)
    rb, _ = b.render(0)
    # the index only breaks ties between equal fp32 depths (SPEC.md:348 (3)); this map has ~60
    # tied depth values among its 30000 Gaussians, so the pixels two tied, overlapping Gaussians
    # share may differ -- all others agree to rounding
    d = (ra - rb).abs().amax(dim=1)
    assert (d > 1e-5).float().mean().item() <= 3e-3 and d.max().item() <= 5e-2  # measured 1.5e-3
    for _ in range(3):
        a.build_pyramids()
        b.build_pyramids()
        la = torch.stack(a.step()).cpu().numpy()
        lb = torch.stack(b.step()).cpu().numpy()
        np.testing.assert_allclose(la, lb, rtol=1e-5)
    diff = (a.params[:, :a.n] - b.params[:, order]).abs()
    moved = (b.params[:, order] - p0).abs()
    tol = 1e-3 * moved + 4 * torch.finfo(torch.float32).eps * p0.abs() + 1e-9
    bad = diff > tol
    assert bad.float().mean().item() <= 1e-4, (int(bad.sum()), float(diff.max()))
