"""Window shrinking on the GPU (svm_params.shrink_window, DESIGN.md
reading R29) against the oracle with the same rule (oracle_svm_train_full(..., shrink)),
pinned in test_oracle_qp.py: identical pair trajectory, alpha, f and b -- on instances
where shrinking changes the selection, on the workload laws (where it does not), with the
second-order rule, max_iter inside and at the end of a window, a warm start, and the
compaction / replay at several sizes.  Marked `gpu`."""
import numpy as np
import pytest

from gen import workloads as W
from oracle import oracle as O
from tests.test_oracle_qp import _rand_problem

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S():
    import paper_2311_14908_b200 as S
    S.lib()
    return S


def _check(S, X, y, C, kern, gamma, tol, H, **kw):
    cap = 10 * len(y) + 10000
    wss = kw.get("wss", 1)
    ref = O.train(X, y, C, kern, gamma, tol, trace_cap=cap, shrink=H, wss=wss,
                  max_iter=kw.get("max_iter", 0), alpha0=kw.get("alpha0"), f0=kw.get("f0"))
    r = S.svm_train_ex(X, y, C, kern, gamma, tol, want_f=True, trace_cap=cap, shrink_window=H, **kw)
    assert r["info"]["iterations"] == ref.iterations
    assert bool(r["info"]["converged"]) == ref.converged
    np.testing.assert_array_equal(r["trace"], ref.trace)
    np.testing.assert_array_equal(r["alpha"], ref.alpha)
    np.testing.assert_array_equal(r["f"], ref.f)
    assert r["b"] == ref.b
    assert r["info"]["b_up"] == ref.b_up and r["info"]["b_low"] == ref.b_low
    return r, ref


@pytest.mark.parametrize("seed,H", [(1, 3), (1, 5), (2, 3), (3, 5), (7, 2)])
def test_shrinking_changed_trajectories(S, seed, H):
    X, y, C, kern = _rand_problem(seed)
    r, ref = _check(S, X, y, C, kern, 0.5, 1e-3, H)


def test_shrinking_changes_something_here(S):
    X, y, C, kern = _rand_problem(1)
    plain = O.train(X, y, C, kern, 0.5, 1e-3, trace_cap=100000)
    r, ref = _check(S, X, y, C, kern, 0.5, 1e-3, 3)
    assert plain.iterations != ref.iterations


@pytest.mark.parametrize("name,n,H", [("W1", 200, 20), ("W3", 2000, 100), ("W4", 6000, 100), ("W5", 3000, 100),
                                      ("W2", 2000, 50)])
def test_shrinking_workloads(S, name, n, H):
    w = W.get(name)
    X, y = w.train(n)
    _check(S, X, y, w.C, w.kernel, w.gamma, w.tol, H)


def test_shrinking_with_second_order_selection(S):
    w = W.get("W3")
    X, y = w.train(1500)
    _check(S, X, y, w.C, w.kernel, w.gamma, w.tol, 40, wss=2)
    X, y, C, kern = _rand_problem(2)
    _check(S, X, y, C, kern, 0.5, 1e-3, 3, wss=2)


@pytest.mark.parametrize("mi", [250, 300, 317])
def test_shrinking_max_iter(S, mi):
    """max_iter inside a window (317: the active rows' selection is reported) and at a
    window end (300 = 3 windows of 100: the selection over every row is)."""
    w = W.get("W5")
    X, y = w.train(3000)
    r, ref = _check(S, X, y, w.C, w.kernel, w.gamma, w.tol, 100, max_iter=mi)
    assert r["info"]["converged"] == 0


def test_shrinking_warm_start(S):
    w = W.get("W4")
    X, y = w.train(5000)
    full = O.train(X, y, w.C, w.kernel, w.gamma, w.tol)
    part = O.train(X, y, w.C, w.kernel, w.gamma, w.tol, max_iter=full.iterations // 2)
    _check(S, X, y, w.C, w.kernel, w.gamma, w.tol, 64, alpha0=part.alpha, f0=part.f)


def test_shrinking_sets_rows_aside_and_replays(S):
    """A state far into the solve (many multipliers at bounds): most rows are set aside in
    every window, so the result rests on the compaction and the replay of the window's
    updates (their f is checked bit for bit over all rows)."""
    w = W.get("W5")
    X, y = w.train(6000)
    part = O.train(X, y, w.C, w.kernel, w.gamma, w.tol, max_iter=3000)
    _check(S, X, y, w.C, w.kernel, w.gamma, w.tol, 37, alpha0=part.alpha, f0=part.f, max_iter=600)


def test_shrinking_device_api_and_errors(S):
    import torch
    w = W.get("W5")
    X, y = w.train(2000)
    ref = O.train(X, y, w.C, w.kernel, w.gamma, w.tol, shrink=100)
    r = S.svm_train_dev(torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda(), w.C, w.kernel, w.gamma, w.tol,
                        shrink_window=100, want_f=True)
    np.testing.assert_array_equal(r["alpha"].cpu().numpy(), ref.alpha)
    np.testing.assert_array_equal(r["f"].cpu().numpy(), ref.f)
    with pytest.raises(S.SvmError, match="rank"):
        S.svm_train_ex(X, y, w.C, w.kernel, w.gamma, w.tol, shrink_window=10, virtual_ranks=2)


def test_shrinking_with_row_cache_and_gram(S, monkeypatch):
    """The sub-problems keep a requested row cache (and the Gram path works per window):
    still the oracle's shrinking trajectory."""
    monkeypatch.setenv("SVMB200_NO_RESIDENT", "1")
    w = W.get("W3")
    X, y = w.train(1500)
    _check(S, X, y, w.C, w.kernel, w.gamma, w.tol, 50, cache_rows=16)
    monkeypatch.delenv("SVMB200_NO_RESIDENT")
    _check(S, X, y, w.C, w.kernel, w.gamma, w.tol, 50, gram=1)


def test_shrinking_replay_wide_rows(S):
    """d = 784 > 256: the rows set aside are replayed by the feature-chunked replay kernel
    (the row-resident one covers d <= 256); from a state far into the W3 solve."""
    w = W.get("W3")
    X, y = w.train(2000)
    full = O.train(X, y, w.C, w.kernel, w.gamma, w.tol)
    part = O.train(X, y, w.C, w.kernel, w.gamma, w.tol, max_iter=(2 * full.iterations) // 3)
    _check(S, X, y, w.C, w.kernel, w.gamma, w.tol, 29, alpha0=part.alpha, f0=part.f, max_iter=200)
