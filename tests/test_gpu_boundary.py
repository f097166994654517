"""GPU tests of the C-ABI boundary added for SURVEY §8(b) / row a10 / row a8: device-side
info reductions, support-vector compaction, device warm start, svm_debug on the
row-sharded entry point, and the LRU row cache's hit / miss counters (against a replay
of the oracle's pair trajectory through the same replacement policy).  Marked `gpu`."""
import numpy as np
import pytest

from gen import workloads as W
from oracle import oracle as O
from tests.helpers.lru import lru_replay

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S():
    import paper_2311_14908_b200 as S
    S.lib()
    return S


def _cuda(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def test_info_reduced_on_device(S):
    """n_sv and W = 1/2 sum alpha (1 - y f) (S:L176 identity) from the device reduction
    equal the oracle's state: n_sv exactly, W within 1e-12 relative of the oracle's
    f-form and within 1e-9 of the O(n^2) quadratic form."""
    w = W.get("W2")
    X, y = w.train(2000)
    r_or = O.train(X, y, w.C, w.kernel, w.gamma, w.tol)
    for api in ("host", "dev"):
        if api == "host":
            r = S.svm_train_ex(X, y, w.C, w.kernel, w.gamma, w.tol)
        else:
            r = S.svm_train_dev(_cuda(X), _cuda(y), w.C, w.kernel, w.gamma, w.tol)
        info = r["info"]
        assert info["n_sv"] == int(np.sum(r_or.alpha > 1e-8))
        W_f = O.dual_objective_from_f(r_or.alpha, y, r_or.f)
        assert abs(info["dual_objective"] - W_f) <= 1e-12 * abs(W_f)
        W_q = O.dual_objective(X, y, r_or.alpha, w.kernel, w.gamma)
        assert abs(info["dual_objective"] - W_q) <= 1e-9 * abs(W_q)
        assert (info["seconds_h2d"] > 0) == (api == "host")


@pytest.mark.parametrize("n", [1, 2, 257, 5000, 70001])
def test_support_vectors_compaction(S, n):
    """svm_support_vectors_dev: {alpha > eps} in ascending index, coef = alpha * y exactly,
    the rows bit for bit; ragged sizes; count-only; the empty set."""
    rng = np.random.default_rng(n)
    d = 37
    X = rng.normal(size=(n, d)).astype(np.float32)
    y = np.where(rng.random(n) < 0.5, 1, -1).astype(np.int8)
    alpha = np.where(rng.random(n) < 0.4, rng.uniform(0, 1, n), 0.0)
    alpha[rng.random(n) < 0.05] = 5e-9                           # below the threshold
    Xsv, coef, idx = S.svm_support_vectors_dev(_cuda(X), _cuda(y), _cuda(alpha), want_index=True)
    sv = np.flatnonzero(alpha > 1e-8)
    np.testing.assert_array_equal(idx.cpu().numpy(), sv)
    np.testing.assert_array_equal(coef.cpu().numpy(), alpha[sv] * y[sv])
    np.testing.assert_array_equal(Xsv.cpu().numpy(), X[sv])
    Xz, cz, _ = S.svm_support_vectors_dev(_cuda(X), _cuda(y), _cuda(np.zeros(n)))
    assert cz.shape == (0,) and Xz.shape == (0, d)


def test_device_warm_start_segment_parity(S):
    """svm_train_dev resumed from the oracle's state after k steps (device alpha0 / f0)
    reproduces the rest of the oracle's trajectory, alpha and f bit for bit."""
    w = W.get("W3")
    X, y = w.train(1200)
    full = O.train(X, y, w.C, w.kernel, w.gamma, w.tol, trace_cap=100000)
    k = full.iterations // 3
    part = O.train(X, y, w.C, w.kernel, w.gamma, w.tol, max_iter=k)
    r = S.svm_train_dev(_cuda(X), _cuda(y), w.C, w.kernel, w.gamma, w.tol, alpha0=_cuda(part.alpha),
                        f0=_cuda(part.f), want_f=True, trace_cap=100000)
    assert r["info"]["iterations"] == full.iterations - k
    np.testing.assert_array_equal(r["trace"], full.trace[k:])
    np.testing.assert_array_equal(r["alpha"].cpu().numpy(), full.alpha)
    np.testing.assert_array_equal(r["f"].cpu().numpy(), full.f)
    assert r["b"] == full.b


def test_train_shard_debug_world1(S):
    """svm_train_shard with svm_debug (NCCL bootstrap, world = 1): pair trace, final f and
    a warm start, all equal the oracle."""
    w = W.get("W5")
    X, y = w.train(2500)
    full = O.train(X, y, w.C, w.kernel, w.gamma, w.tol, trace_cap=100000)
    comm = S.svm_comm_init(0, 1, S.svm_comm_unique_id(), 0)
    try:
        r = S.svm_train_shard(comm, _cuda(X), _cuda(y), 0, len(y), w.C, w.kernel, w.gamma, w.tol,
                              trace_cap=100000, want_f=True)
        np.testing.assert_array_equal(r["trace"], full.trace)
        np.testing.assert_array_equal(r["f"].cpu().numpy(), full.f)
        np.testing.assert_array_equal(r["alpha"].cpu().numpy(), full.alpha)
        k = full.iterations // 2
        part = O.train(X, y, w.C, w.kernel, w.gamma, w.tol, max_iter=k)
        r2 = S.svm_train_shard(comm, _cuda(X), _cuda(y), 0, len(y), w.C, w.kernel, w.gamma, w.tol,
                               trace_cap=100000, alpha0=_cuda(part.alpha), f0=_cuda(part.f))
        np.testing.assert_array_equal(r2["trace"], full.trace[k:])
        np.testing.assert_array_equal(r2["alpha"].cpu().numpy(), full.alpha)
        assert r2["info"]["n_sv"] == int(np.sum(full.alpha > 1e-8))
    finally:
        S.svm_comm_destroy(comm)


@pytest.mark.parametrize("name,n,slots", [("W3", 2000, 16), ("W3", 2000, 64), ("W5", 3000, 8)])
def test_row_cache_counters_match_lru_replay(S, monkeypatch, name, n, slots):
    """cache_hits / cache_misses of the device directory equal the replay of the oracle's
    pair trajectory through the same LRU policy, and the solve equals the oracle."""
    monkeypatch.setenv("SVMB200_NO_RESIDENT", "1")
    w = W.get(name)
    X, y = w.train(n)
    r_or = O.train(X, y, w.C, w.kernel, w.gamma, w.tol, trace_cap=100000)
    r = S.svm_train_ex(X, y, w.C, w.kernel, w.gamma, w.tol, cache_rows=slots, trace_cap=100000)
    np.testing.assert_array_equal(r["trace"], r_or.trace)
    np.testing.assert_array_equal(r["alpha"], r_or.alpha)
    hits, misses = lru_replay(r_or.trace, slots)
    assert (r["info"]["cache_hits"], r["info"]["cache_misses"]) == (hits, misses)
    if name == "W3":
        assert hits > 0
