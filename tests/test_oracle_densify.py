"""Pins of the oracle's densify-and-prune.

SPEC's three worked examples (no-op, one clone, one prune), the split branch, the footprint
prune, the untouched-primitive invariant (SPEC.md "densify_and_prune preserves the invariant
fields of untouched primitives bitwise"), and the geometry of the new positions checked against
scipy's rotation (an independent library route): offset = R(q) diag(e^s) z, so over many z the
offsets' covariance is Sigma3 = R diag(e^2s) R^T."""
import math

import numpy as np
import pytest
from scipy.spatial.transform import Rotation

import oracle.oracle as orc

K = 14  # D = 0: P 3 | q 4 | log s 3 | logit 1 | SH 3
HP = dict(grad_thr=2e-4, percent_dense=0.01, extent=5.0, op_thr=0.005, max_screen=320)


def _map(n, seed=0):
    rng = np.random.default_rng(seed)
    rec = np.zeros((n, K), np.float32)
    rec[:, 0:3] = rng.uniform(-1, 1, (n, 3))
    q = rng.normal(size=(n, 4))
    rec[:, 3:7] = q / np.linalg.norm(q, axis=1, keepdims=True) * rng.uniform(0.5, 2, (n, 1))
    rec[:, 7:10] = np.log(rng.uniform(0.005, 0.03, (n, 3)))  # 0.005..0.03 < 1% of 5 m... mostly
    rec[:, 7:10] = np.minimum(rec[:, 7:10], math.log(0.04))
    rec[:, 10] = rng.uniform(-2, 4, n)
    rec[:, 11:14] = rng.normal(size=(n, 3))
    m = rng.normal(size=(n, K)).astype(np.float32)
    v = rng.uniform(0, 1, (n, K)).astype(np.float32)
    return rec, m, v


def _run(rec, m, v, ga, vc, mr, z, **kw):
    hp = dict(HP, **kw)
    return orc.densify(rec, m, v, ga, vc, mr, z, hp["grad_thr"], hp["percent_dense"], hp["extent"], hp["op_thr"],
                       hp["max_screen"])


def _stats(n, grad=1e-5):
    return np.full(n, grad * 4, np.float32), np.full(n, 4, np.float32), np.full(n, 10, np.int32)


def _z(n, seed=1):
    return np.random.default_rng(seed).normal(size=(n, 2, 3)).astype(np.float32)


def test_all_healthy_is_a_noop():
    rec, m, v = _map(50)
    rec[:, 7:10] = math.log(0.02)
    ga, vc, mr = _stats(50)
    out = _run(rec, m, v, ga, vc, mr, _z(50))
    assert (out["n_clone"], out["n_split"], out["n_prune"]) == (0, 0, 0) and out["n_new"] == 50
    assert np.array_equal(out["rec"], rec.astype(np.float64)) and np.array_equal(out["m"], m.astype(np.float64))


def test_one_small_high_gradient_clone():
    n = 20
    rec, m, v = _map(n)
    rec[:, 7:10] = math.log(0.02)  # 0.02 <= 0.01 * 5: small
    ga, vc, mr = _stats(n)
    ga[7] = 1e-3 * 4  # mean 1e-3 >= 2e-4
    z = _z(n)
    out = _run(rec, m, v, ga, vc, mr, z)
    assert (out["n_clone"], out["n_split"], out["n_prune"]) == (1, 0, 0) and out["n_new"] == n + 1
    assert out["cls"][7] == 1
    assert np.array_equal(out["rec"][:n], rec.astype(np.float64))  # originals untouched, in order
    clone = out["rec"][n]
    assert np.array_equal(clone[3:], rec[7, 3:].astype(np.float64))
    q = rec[7, 3:7].astype(np.float64)
    R = Rotation.from_quat([q[1], q[2], q[3], q[0]]).as_matrix()  # scipy: (x, y, z, w)
    off = R @ (np.exp(rec[7, 7:10].astype(np.float64)) * z[7, 0])
    np.testing.assert_allclose(clone[:3], rec[7, :3] + off, rtol=0, atol=1e-12)
    assert (out["m"][n] == 0).all() and (out["v"][n] == 0).all()
    assert np.array_equal(out["m"][:n], m.astype(np.float64))


def test_low_opacity_pruned():
    n = 10
    rec, m, v = _map(n)
    rec[:, 10] = 1.0
    rec[3, 10] = np.float32(math.log(0.001 / 0.999))
    ga, vc, mr = _stats(n)
    out = _run(rec, m, v, ga, vc, mr, _z(n))
    assert (out["n_clone"], out["n_split"], out["n_prune"]) == (0, 0, 1) and out["n_new"] == n - 1
    assert np.array_equal(out["rec"], np.delete(rec, 3, 0).astype(np.float64))


def test_split_large_high_gradient():
    n = 6
    rec, m, v = _map(n)
    rec[:, 7:10] = math.log(0.02)
    rec[2, 7:10] = [math.log(0.2), math.log(0.03), math.log(0.01)]  # 0.2 > 0.05: large
    ga, vc, mr = _stats(n)
    ga[2] = 1.0
    z = _z(n, 5)
    out = _run(rec, m, v, ga, vc, mr, z)
    assert (out["n_clone"], out["n_split"], out["n_prune"]) == (0, 1, 0) and out["n_new"] == n + 1
    assert np.array_equal(out["rec"][:n - 1], np.delete(rec, 2, 0).astype(np.float64))  # parent removed
    q = rec[2, 3:7].astype(np.float64)
    R = Rotation.from_quat([q[1], q[2], q[3], q[0]]).as_matrix()
    for c in range(2):
        child = out["rec"][n - 1 + c]
        np.testing.assert_allclose(np.exp(child[7:10]), np.exp(rec[2, 7:10].astype(np.float64)) / 1.6, rtol=1e-14)
        off = R @ (np.exp(rec[2, 7:10].astype(np.float64)) * z[2, c])
        np.testing.assert_allclose(child[:3], rec[2, :3] + off, atol=1e-12)
        assert np.array_equal(child[3:7], rec[2, 3:7].astype(np.float64)) and child[10] == rec[2, 10]
        assert np.array_equal(child[11:], rec[2, 11:].astype(np.float64))


def test_footprint_prune_and_threshold_edges():
    n = 8
    rec, m, v = _map(n)
    rec[:, 7:10] = math.log(0.02)
    rec[:, 10] = 2.0
    ga, vc, mr = _stats(n)
    mr[1] = 321  # > 320 px: pruned
    mr[2] = 320  # == : kept
    ga[4] = np.float32(2e-4) * 4  # mean == threshold: high (>=)
    vc[5] = 0.0
    ga[5] = 1.0  # never visible: mean 0, not high
    out = _run(rec, m, v, ga, vc, mr, _z(n))
    assert list(out["cls"]) == [0, 3, 0, 0, 1, 0, 0, 0]


def test_clone_offsets_have_the_gaussian_covariance():
    """Offsets R diag(e^s) z over 20000 samples: covariance -> R diag(e^2s) R^T (scipy R)."""
    n = 20000
    rec = np.zeros((n, K), np.float32)
    q = np.array([0.9, 0.2, -0.3, 0.25], np.float32)
    rec[:, 3:7] = q
    rec[:, 7:10] = np.log([0.004, 0.001, 0.002]).astype(np.float32)
    rec[:, 10] = 3.0
    z = _z(n, 11)
    ga, vc, mr = _stats(n, grad=1.0)
    out = _run(rec, np.zeros_like(rec), np.zeros_like(rec), ga, vc, mr, z)
    assert out["n_clone"] == n
    off = out["rec"][n:, :3] - rec[:, :3]
    R = Rotation.from_quat([q[1], q[2], q[3], q[0]]).as_matrix()
    S = np.diag(np.exp(2 * rec[0, 7:10].astype(np.float64)))
    cov = np.cov(off.T)
    np.testing.assert_allclose(cov, R @ S @ R.T, atol=0.05 * S.max())
