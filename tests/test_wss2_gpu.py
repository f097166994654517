"""Second-order working-set selection on the GPU (Fan, Chen & Lin
2005, cited at PAPER.md L140): svm_params.wss = 2 against the oracle's
oracle_svm_train_wss(..., 2) (pinned against scikit-learn's libsvm in
test_oracle_qp.py) -- identical pair trajectory, alpha, f and b, in every execution mode
(fp32 / dictionary / mixed rows, row cache, Gram, virtual ranks, launch chunking).
Marked `gpu`."""
import hashlib
import os

import numpy as np
import pytest

from gen import workloads as W
from oracle import oracle as O

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def S():
    import paper_2311_14908_b200 as S
    S.lib()
    return S


def _check(S, X, y, w, **params):
    cap = 10 * len(y) + 10000
    ref = O.train(X, y, w.C, w.kernel, w.gamma, w.tol, trace_cap=cap, wss=2,
                  max_iter=params.get("max_iter", 0))
    r = S.svm_train_ex(X, y, w.C, w.kernel, w.gamma, w.tol, want_f=True, trace_cap=cap, wss=2, **params)
    assert r["info"]["iterations"] == ref.iterations
    assert bool(r["info"]["converged"]) == ref.converged
    np.testing.assert_array_equal(r["trace"], ref.trace)
    np.testing.assert_array_equal(r["alpha"], ref.alpha)
    np.testing.assert_array_equal(r["f"], ref.f)
    assert r["b"] == ref.b
    return r, ref


@pytest.mark.parametrize("name,n", [("W1", 200), ("W2", 1500), ("W3", 1500), ("W4", 4000), ("W5", 2000)])
def test_wss2_trajectory_parity(S, name, n):
    w = W.get(name)
    X, y = w.train(n)
    r, ref = _check(S, X, y, w)
    # the second-order rule differs from the first-order one on these data
    r1 = O.train(X, y, w.C, w.kernel, w.gamma, w.tol, trace_cap=10 * n + 10000)
    assert r1.iterations != ref.iterations or not np.array_equal(r1.trace, ref.trace)


def test_wss2_ragged_linear_and_ties(S):
    rng = np.random.default_rng(12)
    for n, d in ((2, 1), (37, 7), (149, 5), (1031, 13)):
        X = rng.integers(0, 3, size=(n, d)).astype(np.float32)
        y = np.where(rng.random(n) < 0.5, 1, -1).astype(np.int8)
        y[0], y[-1] = 1, -1
        for kern, gamma in ((O.LINEAR, 0.0), (O.RBF, 0.3)):
            w = W.Workload("t", "", n, d, kern, gamma, 2.0, 1e-3, 0, 0, 0, None)
            _check(S, X, y, w)


@pytest.mark.parametrize("params,env", [
    ({"cache_rows": 16}, {"SVMB200_NO_RESIDENT": "1"}),
    ({"cache_rows": -1}, {"SVMB200_NO_RESIDENT": "1"}),
    ({"virtual_ranks": 3}, {}),
    ({"gram": 1}, {}),
    ({"iters_per_launch": 7}, {}),
    ({"max_iter": 101}, {}),
    ({"ctas": 9}, {"SVMB200_RPT": "1"}),
])
def test_wss2_modes(S, monkeypatch, params, env):
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    for name, n in (("W3", 1200), ("W1", 200), ("W4", 3000)):
        w = W.get(name)
        X, y = w.train(n)
        _check(S, X, y, w, **params)


def test_wss2_full_w3_against_stored_oracle(S):
    """Full W3 (60,000 x 784) under wss = 2 against the oracle result stored by
    oracle/tools/make_golden.py W3 0 2."""
    path = os.path.join(GOLD, "W3_wss2_oracle.npz")
    if not os.path.exists(path):
        pytest.skip("golden W3_wss2_oracle.npz not generated")
    g = np.load(path)
    w = W.get("W3")
    X, y = w.train()
    r = S.svm_train_ex(X, y, w.C, w.kernel, w.gamma, w.tol, want_f=True, wss=2,
                       trace_cap=int(g["iterations"]) + 1)
    assert r["info"]["iterations"] == int(g["iterations"])
    sha = hashlib.sha256(np.ascontiguousarray(r["trace"], dtype=np.int64).tobytes()).hexdigest()
    assert sha == str(g["trace_sha"])
    np.testing.assert_array_equal(r["alpha"], g["alpha"])
    np.testing.assert_array_equal(r["f"], g["f"])
    assert r["b"] == float(g["b"])


def test_wss2_rejected_by_batch(S):
    import torch
    X, y = W.get("W1").train(50)
    with pytest.raises(S.SvmError, match="wss"):
        S.svm_train_batch_dev([(torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda())], 1.0, S.LINEAR, wss=2)
