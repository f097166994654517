"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same
seeded inputs.  Marked `gpu`; run on a B200.

The arithmetic contract makes both sides take every decision in
fp64 on identical values, so beyond BASELINE.json's tolerances (dual objective 1e-5
relative, decision values 1e-4 absolute, identical labels, identical SV sets with alpha
within 1e-6 C) the tests also require the identical pair trajectory and bit-equal alpha.
"""
import hashlib
import types
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


def _assert_bj_parity(X, y, w, r_gpu, r_or, Xt=None):
    """BASELINE.json north_star tolerances."""
    C = w.C
    a_g, a_o = r_gpu["alpha"], r_or.alpha
    W_g = O.dual_objective_from_f(a_g, y, r_gpu["f"]) if "f" in r_gpu else None
    W_o = O.dual_objective_from_f(a_o, y, r_or.f)
    if W_g is not None:
        assert abs(W_g - W_o) <= 1e-5 * abs(W_o) + 1e-12
    assert np.max(np.abs(a_g - a_o)) <= 1e-6 * C
    sv_g, sv_o = a_g > 1e-8, a_o > 1e-8
    assert np.array_equal(sv_g, sv_o)
    if Xt is not None:
        sv = sv_o
        d_o = O.decision(X[sv], (a_o * y)[sv], r_or.b, w.kernel, w.gamma, Xt)
        d_g = O.decision(X[sv_g], (a_g * y)[sv_g], r_gpu["b"], w.kernel, w.gamma, Xt)
        assert np.max(np.abs(d_g - d_o)) <= 1e-4
        assert np.array_equal(np.sign(d_g), np.sign(d_o))


def _run_pair(S, w, X, y, trace=True, **params):
    cap = 10 * len(y) + 10000 if trace else 0
    r_or = O.train(X, y, w.C, w.kernel, w.gamma, w.tol, trace_cap=cap,
                   max_iter=params.get("max_iter", 0))
    r_g = S.svm_train_ex(X, y, w.C, w.kernel, w.gamma, w.tol, want_f=True, trace_cap=cap, **params)
    return r_g, r_or


def _assert_exact(r_g, r_or):
    info = r_g["info"]
    assert info["iterations"] == r_or.iterations
    assert bool(info["converged"]) == r_or.converged
    if "trace" in r_g and "trace" in r_or:
        np.testing.assert_array_equal(r_g["trace"], r_or.trace)
    np.testing.assert_array_equal(r_g["alpha"], r_or.alpha)
    np.testing.assert_array_equal(r_g["f"], r_or.f)
    assert r_g["b"] == r_or.b
    assert info["b_up"] == r_or.b_up and info["b_low"] == r_or.b_low


# ---------------------------------------------------------------- kernel value / exp
def test_device_exp_matches_oracle_through_predict(S):
    """One support vector at the origin, coef 1, b 0: dec(x) = exp(-gamma x^2), so the
    device exp is checked against the oracle on 2^16 arguments (the fp32 x makes x^2
    exact, the same fp64 argument reaches both exps)."""
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.uniform(0, 40, 40000), np.exp(rng.uniform(-30, 3.5, 25536))]).astype(np.float32)
    Xt = x.reshape(-1, 1)
    sv = np.zeros((1, 1), np.float32)
    for gamma in (0.5, 0.0125, 1.0 / 54):
        d_g = S.svm_predict(sv, np.ones(1), 0.0, S.RBF, gamma, Xt)
        d_o = O.decision(sv, np.ones(1), 0.0, O.RBF, gamma, Xt)
        np.testing.assert_array_equal(d_g, d_o)


# ---------------------------------------------------------------- closed forms via GPU
def test_two_point_closed_form(S):
    X = np.array([[1.0], [3.0]], np.float32); y = np.array([1, -1], np.int8)
    alpha, b = S.svm_train(X, y, 10.0, S.LINEAR, 0.0, 1e-3)
    np.testing.assert_allclose(alpha, [0.5, 0.5], atol=1e-15)
    assert b == pytest.approx(2.0, abs=1e-15)
    dec = S.svm_predict(X, alpha * y, b, S.LINEAR, 0.0, np.array([[2.0], [1.0]], np.float32))
    np.testing.assert_allclose(dec, [0.0, 1.0], atol=1e-14)


def test_eta_zero_and_clipping(S):
    X = np.array([[0.0], [0.0], [2.0]], np.float32); y = np.array([1, -1, -1], np.int8)
    w = W.Workload("eta0", "", 3, 1, O.RBF, 0.5, 1.0, 1e-3, 0, 0, 0, None)
    r_g, r_or = _run_pair(S, w, X, y)
    _assert_exact(r_g, r_or)
    X = np.array([[1.0], [3.0]], np.float32); y = np.array([1, -1], np.int8)
    w = W.Workload("clip", "", 2, 1, O.LINEAR, 0.0, 0.25, 1e-3, 0, 0, 0, None)
    r_g, r_or = _run_pair(S, w, X, y)
    _assert_exact(r_g, r_or)
    assert r_g["alpha"].tolist() == [0.25, 0.25]


# ---------------------------------------------------------------- full trajectories
SMALL = [("W1", 200), ("W2", 3000), ("W3", 1500), ("W4", 6000), ("W5", 3000)]


@pytest.mark.parametrize("name,n", SMALL)
def test_trajectory_parity(S, name, n):
    w = W.get(name)
    X, y = w.train(n)
    Xt, _ = w.test(500)
    r_g, r_or = _run_pair(S, w, X, y)
    _assert_exact(r_g, r_or)
    _assert_bj_parity(X, y, w, r_g, r_or, Xt)


@pytest.mark.parametrize("vr,ctas", [(1, 7), (2, 0), (3, 0), (8, 0), (4, 9)])
def test_partition_independence(S, vr, ctas):
    """Same result for any number of (virtual) ranks and CTAs (S:L197 deterministic
    combine): exercises the multi-rank mailbox protocol on one GPU."""
    w = W.get("W5")
    X, y = w.train(2500)
    r_g, r_or = _run_pair(S, w, X, y, virtual_ranks=vr, ctas=ctas)
    _assert_exact(r_g, r_or)


def _cluster_cases():
    rng = np.random.default_rng(31)
    cases = []
    w1 = W.get("W1")
    cases.append(("W1 d=2 (rows in records)", w1, *w1.train()))
    w2 = W.get("W2")
    X2, y2 = w2.train()
    cases.append(("W2 4000 rows, bit rows in records", w2, X2[:4000], y2[:4000]))
    for n, d in ((900, 10), (600, 40)):                  # d > 12: rows gathered from HBM
        X = rng.normal(size=(n, d)).astype(np.float32)
        y = np.where(X[:, 0] + 0.7 * rng.normal(size=n) > 0, 1, -1).astype(np.int8)
        w = types.SimpleNamespace(C=1.0, kernel=1, gamma=0.1, tol=1e-3)
        cases.append((f"dense n={n} d={d}", w, X, y))
    return cases


@pytest.mark.parametrize("cluster", [-1, 1, 2, 4, 8, 16])
def test_cluster_exchange_parity(S, cluster):
    """Cluster mode -- the rank's CTAs form one thread-block cluster and exchange their
    candidates through distributed shared memory, the candidates' rows travelling in the
    records when they are short -- gives the oracle's trajectory bit for bit, as does the
    global-mailbox exchange (cluster=-1), for every cluster size."""
    for label, w, X, y in _cluster_cases():
        r_g, r_or = _run_pair(S, w, X, y, cluster=cluster)
        _assert_exact(r_g, r_or)


def test_cluster_mode_errors(S):
    w = W.get("W1")
    X, y = w.train()
    with pytest.raises(S.SvmError, match="cluster"):
        S.svm_train_ex(X, y, w.C, w.kernel, w.gamma, w.tol, cluster=17)
    with pytest.raises(S.SvmError, match="cluster"):
        S.svm_train_ex(X, y, w.C, w.kernel, w.gamma, w.tol, cluster=2, virtual_ranks=2)
    X5, y5 = W.get("W5").train(20000)                    # 20,000 x 256 floats: not resident
    with pytest.raises(S.SvmError, match="cluster"):
        S.svm_train_ex(X5, y5, 1.0, 1, 1.0 / 256, 1e-3, cluster=2, max_iter=5)


def test_ragged_and_tiny(S):
    """n smaller than the CTA count (empty CTAs), odd d, duplicate rows with opposite
    labels, a ragged last tile."""
    rng = np.random.default_rng(4)
    for n, d in ((2, 1), (5, 3), (37, 7), (149, 5), (1031, 13)):
        X = rng.integers(0, 3, size=(n, d)).astype(np.float32)   # many duplicates / ties
        y = np.where(rng.random(n) < 0.5, 1, -1).astype(np.int8)
        y[0], y[-1] = 1, -1
        for kern, gamma in ((O.LINEAR, 0.0), (O.RBF, 0.3)):
            w = W.Workload("t", "", n, d, kern, gamma, 2.0, 1e-3, 0, 0, 0, None)
            r_g, r_or = _run_pair(S, w, X, y)
            _assert_exact(r_g, r_or)


def test_launch_chunking_and_max_iter(S):
    """Host convergence checks every set of iterations: splitting the solve
    into launches of 7 iterations gives the same result; max_iter stops early with
    converged = 0 exactly where the oracle stops."""
    w = W.get("W2")
    X, y = w.train(1200)
    r_g, r_or = _run_pair(S, w, X, y, iters_per_launch=7)
    _assert_exact(r_g, r_or)
    assert r_g["info"]["launches"] > 1
    r_g, r_or = _run_pair(S, w, X, y, max_iter=333)
    _assert_exact(r_g, r_or)
    assert r_g["info"]["converged"] == 0 and r_g["info"]["iterations"] == 333


def test_warm_start_segment_parity(S):
    """Resume from the oracle's state after k steps: the GPU then reproduces the rest of
    the oracle's trajectory."""
    w = W.get("W3")
    X, y = w.train(1200)
    full = O.train(X, y, w.C, w.kernel, w.gamma, w.tol, trace_cap=100000)
    k = full.iterations // 2
    part = O.train(X, y, w.C, w.kernel, w.gamma, w.tol, max_iter=k)
    r_g = S.svm_train_ex(X, y, w.C, w.kernel, w.gamma, w.tol, alpha0=part.alpha, f0=part.f,
                         want_f=True, trace_cap=100000)
    assert r_g["info"]["iterations"] == full.iterations - k
    np.testing.assert_array_equal(r_g["trace"], full.trace[k:])
    np.testing.assert_array_equal(r_g["alpha"], full.alpha)


def test_device_api_matches_host_api(S):
    import torch
    w = W.get("W4")
    X, y = w.train(5000)
    r_h = S.svm_train_ex(X, y, w.C, w.kernel, w.gamma, w.tol, want_f=True)
    Xd = torch.from_numpy(X).cuda(); yd = torch.from_numpy(y).cuda()
    r_d = S.svm_train_dev(Xd, yd, w.C, w.kernel, w.gamma, w.tol, want_f=True)
    np.testing.assert_array_equal(r_d["alpha"].cpu().numpy(), r_h["alpha"])
    assert r_d["b"] == r_h["b"]


def test_errors(S):
    X = np.zeros((4, 2), np.float32)
    with pytest.raises(S.SvmError, match="ESINGLECLASS"):
        S.svm_train(X, np.ones(4, np.int8), 1.0, S.LINEAR)
    with pytest.raises(S.SvmError, match="ELABEL"):
        S.svm_train(X, np.array([1, -1, 2, 1], np.int8), 1.0, S.LINEAR)
    Xn = X.copy(); Xn[1, 1] = np.nan
    with pytest.raises(S.SvmError, match="ENONFINITE"):
        S.svm_train(Xn, np.array([1, -1, 1, -1], np.int8), 1.0, S.LINEAR)


# ---------------------------------------------------------------- predict
@pytest.mark.parametrize("name,n,m", [("W1", 200, 300), ("W2", 2000, 1000), ("W3", 1000, 300)])
def test_predict_exact_parity(S, name, n, m):
    w = W.get(name)
    X, y = w.train(n)
    r = O.train(X, y, w.C, w.kernel, w.gamma, w.tol)
    sv = r.alpha > 1e-8
    Xt, _ = w.test(m)
    d_o = O.decision(X[sv], (r.alpha * y)[sv], r.b, w.kernel, w.gamma, Xt)
    d_g = S.svm_predict(X[sv], (r.alpha * y)[sv], r.b, w.kernel, w.gamma, Xt)
    np.testing.assert_array_equal(d_g, d_o)
    # n_sv = 0 -> dec = b
    d0 = S.svm_predict(np.zeros((0, X.shape[1]), np.float32), np.zeros(0), 0.25, w.kernel, w.gamma, Xt)
    assert np.all(d0 == 0.25)


# ---------------------------------------------------------------- full-size configs
@pytest.mark.parametrize("name,params", [
    ("W2", {}),                      # bench workload: binary bit rows, X resident
    ("W3", {}),                      # streamed X + automatic row cache (a8)
    ("W3", {"cache_rows": -1}),      # streamed X, every row recomputed
    ("W3", {"gram": 1}),             # full Gram matrix (a9)
])
def test_full_trajectory_matches_stored_oracle(S, name, params):
    """Full-size configs: the whole trajectory (W2: 42,790 steps, BASELINE.json
    configs[1], the bench workload; W3: 11,659 steps) against the oracle result stored
    by oracle/tools/make_golden.py, in each execution mode the solve can take."""
    path = os.path.join(GOLD, f"{name}_oracle.npz")
    if not os.path.exists(path):
        pytest.skip(f"golden {name}_oracle.npz not generated")
    g = np.load(path)
    w = W.get(name)
    X, y = w.train()
    r = S.svm_train_ex(X, y, w.C, w.kernel, w.gamma, w.tol, want_f=True,
                       trace_cap=int(g["iterations"]) + 1, **params)
    assert r["info"]["iterations"] == int(g["iterations"])
    sha = hashlib.sha256(np.ascontiguousarray(r["trace"], dtype=np.int64).tobytes()).hexdigest()
    assert sha == str(g["trace_sha"])
    np.testing.assert_array_equal(r["alpha"], g["alpha"])
    np.testing.assert_array_equal(r["f"], g["f"])
    assert r["b"] == float(g["b"])


@pytest.mark.parametrize("name,k", [("W3", 60), ("W4", 30), ("W5", 12)])
def test_full_size_prefix_parity(S, name, k):
    """Full-size configs in the bench launch configuration: the first k SMO steps equal
    the oracle's (alpha and f bit for bit over all n rows)."""
    w = W.get(name)
    X, y = w.train()
    r_or = O.train(X, y, w.C, w.kernel, w.gamma, w.tol, max_iter=k, trace_cap=k)
    r_g = S.svm_train_ex(X, y, w.C, w.kernel, w.gamma, w.tol, max_iter=k, want_f=True, trace_cap=k)
    _assert_exact(r_g, r_or)


@pytest.mark.parametrize("name", ["W3", "W4"])
def test_full_size_converged_properties(S, name):
    """Properties that hold at any size on the GPU's converged full-size solution:
    box feasibility, sum alpha y = 0, gap <= 2 tol, and f on 300 sampled rows equals
    the oracle's from-scratch sum_j alpha_j y_j K_ij - y_i."""
    w = W.get(name)
    X, y = w.train()
    r = S.svm_train_ex(X, y, w.C, w.kernel, w.gamma, w.tol, want_f=True)
    a, f = r["alpha"], r["f"]
    assert r["info"]["converged"] == 1
    assert np.all(a >= 0) and np.all(a <= w.C)
    assert abs(np.dot(a, y.astype(float))) <= 1e-9 * max(1.0, w.C * np.sqrt(len(y)))
    assert r["info"]["gap"] <= 2 * w.tol
    sv = a > 0
    rows = np.random.default_rng(1).choice(len(y), 300, replace=False)
    f_ref = O.decision(X[sv], (a * y)[sv], 0.0, w.kernel, w.gamma, X[rows]) - y[rows]
    np.testing.assert_allclose(f[rows], f_ref, atol=1e-6)


# ---------------------------------------------------------------- tensor-core predict
@pytest.mark.parametrize("name,n,m", [("W1", 200, 300), ("W2", 3000, 1500), ("W3", 1500, 400),
                                      ("W4", 4000, 600), ("W5", 3000, 700)])
def test_predict_tensor_core_tolerance(S, name, n, m):
    """tcgen05 3xTF32 path: decision values within BASELINE.json's 1e-4 of the oracle's,
    identical labels wherever the oracle's |dec| exceeds that tolerance (ragged m and
    n_sv: neither is a multiple of the 128-row tiles)."""
    w = W.get(name)
    X, y = w.train(n)
    r = O.train(X, y, w.C, w.kernel, w.gamma, w.tol)
    sv = r.alpha > 1e-8
    Xt, _ = w.test(m)
    d_o = O.decision(X[sv], (r.alpha * y)[sv], r.b, w.kernel, w.gamma, Xt)
    d_t = S.svm_predict(X[sv], (r.alpha * y)[sv], r.b, w.kernel, w.gamma, Xt, mode=S.PREDICT_TENSOR)
    err = np.max(np.abs(d_t - d_o))
    assert err <= 1e-4, err
    clear = np.abs(d_o) > 1e-4
    assert np.array_equal(np.sign(d_t[clear]), np.sign(d_o[clear]))


def test_predict_tensor_core_device_api(S):
    import torch
    w = W.get("W5")
    X, y = w.train(2000)
    r = O.train(X, y, w.C, w.kernel, w.gamma, w.tol)
    sv = r.alpha > 1e-8
    Xt, _ = w.test(1000)
    d_o = O.decision(X[sv], (r.alpha * y)[sv], r.b, w.kernel, w.gamma, Xt)
    dev = S.svm_predict_dev(torch.from_numpy(X[sv]).cuda(), torch.from_numpy((r.alpha * y)[sv]).cuda(), r.b,
                            w.kernel, w.gamma, torch.from_numpy(Xt).cuda(), mode=S.PREDICT_TENSOR)
    assert np.max(np.abs(dev.cpu().numpy() - d_o)) <= 1e-4


def test_binary_encoding_equals_fp_path(S, monkeypatch):
    """Exactly-binary X (Adult-like) runs on bit rows with popcount distances (compact
    encoding); the result must equal both the oracle and the fp32-row path."""
    w = W.get("W2")
    X, y = w.train(2500)
    r_or = O.train(X, y, w.C, w.kernel, w.gamma, w.tol, trace_cap=100000)
    r_bin = S.svm_train_ex(X, y, w.C, w.kernel, w.gamma, w.tol, want_f=True, trace_cap=100000)
    monkeypatch.setenv("SVMB200_NO_BINARY", "1")
    r_fp = S.svm_train_ex(X, y, w.C, w.kernel, w.gamma, w.tol, want_f=True, trace_cap=100000)
    _assert_exact(r_bin, r_or)
    _assert_exact(r_fp, r_or)
    # linear kernel on binary rows (dot = popcount of AND), ragged sizes, many ties
    rng = np.random.default_rng(8)
    for n, d in ((37, 5), (300, 70), (1031, 33)):
        Xb = (rng.random((n, d)) < 0.3).astype(np.float32)
        yb = np.where(rng.random(n) < 0.5, 1, -1).astype(np.int8)
        yb[0], yb[-1] = 1, -1
        for kern, gamma in ((O.LINEAR, 0.0), (O.RBF, 0.2)):
            wb = W.Workload("b", "", n, d, kern, gamma, 1.5, 1e-3, 0, 0, 0, None)
            monkeypatch.delenv("SVMB200_NO_BINARY", raising=False)
            r_g, r_o = _run_pair(S, wb, Xb, yb)
            _assert_exact(r_g, r_o)


@pytest.mark.parametrize("d", [300, 500])
def test_wide_binary_rows_kernel_variants(S, monkeypatch, d):
    """Binary rows wider than smo_bincl's 256 features take the cluster-specialised
    smo_persistent (d = 300: rows still travel in the records; d = 500: rows gathered
    from HBM), and the global-exchange path (cluster = -1); all equal the oracle."""
    rng = np.random.default_rng(d)
    n = 1500
    Xb = (rng.random((n, d)) < 0.05).astype(np.float32)
    yb = np.where(Xb[:, :20].sum(1) + 0.5 * rng.normal(size=n) > 1.0, 1, -1).astype(np.int8)
    wb = W.Workload("b", "", n, d, O.RBF, 0.05, 2.0, 1e-3, 0, 0, 0, None)
    r_g, r_o = _run_pair(S, wb, Xb, yb)
    _assert_exact(r_g, r_o)
    plan = S.last_plan()
    assert plan["mode"] == "binary-resident" and plan["kernel"].startswith("smo_persistent")
    r_g2 = S.svm_train_ex(Xb, yb, wb.C, wb.kernel, wb.gamma, wb.tol, want_f=True, cluster=-1)
    np.testing.assert_array_equal(r_g2["alpha"], r_o.alpha)


def test_last_plan_reports_the_kernel(S):
    """svm_last_plan: W2 runs on the binary-cluster kernel; a streamed problem on the
    148-CTA persistent kernel."""
    w = W.get("W2")
    X, y = w.train(4000)
    S.svm_train_ex(X, y, w.C, w.kernel, w.gamma, w.tol, max_iter=10)
    p = S.last_plan()
    assert p["kernel"] == "smo_bincl<1>" and p["mode"] == "binary-resident" and p["cluster"] >= 1
    w5 = W.get("W5")
    X5, y5 = w5.train(200000)                            # 1352 rows of 256 floats per CTA
    S.svm_train_ex(X5, y5, w5.C, w5.kernel, w5.gamma, w5.tol, max_iter=3)
    p = S.last_plan()
    assert p["kernel"].startswith("smo_persistent") and p["cluster"] == 0 and p["mode"].startswith("streamed")


def test_train_shard_single_rank(S):
    """The one-process-per-GPU entry point (NCCL bootstrap, IPC mailbox, system-scope
    exchange) with world = 1 on one GPU reproduces the oracle."""
    import torch
    w = W.get("W5")
    X, y = w.train(3000)
    uid = S.svm_comm_unique_id()
    comm = S.svm_comm_init(0, 1, uid, 0)
    try:
        r = S.svm_train_shard(comm, torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda(), 0, len(y),
                              w.C, w.kernel, w.gamma, w.tol)
    finally:
        S.svm_comm_destroy(comm)
    r_or = O.train(X, y, w.C, w.kernel, w.gamma, w.tol)
    assert r["info"]["iterations"] == r_or.iterations
    np.testing.assert_array_equal(r["alpha"].cpu().numpy(), r_or.alpha)
    assert r["b"] == r_or.b
    assert r["info"]["dual_objective"] == pytest.approx(O.dual_objective_from_f(r_or.alpha, y, r_or.f), rel=1e-12)


@pytest.mark.parametrize("name,n,kern", [("W3", 1500, None), ("W5", 2500, None), ("W1", 200, None),
                                         ("W4", 3000, None)])
def test_gram_path_parity(S, name, n, kern):
    """Full-Gram path: K precomputed once with the row pass's arithmetic,
    then rows of K read per iteration -- identical trajectory and alpha."""
    w = W.get(name)
    X, y = w.train(n)
    r_g, r_or = _run_pair(S, w, X, y, gram=1)
    _assert_exact(r_g, r_or)
    r_s = S.svm_train_ex(X, y, w.C, w.kernel, w.gamma, w.tol, want_f=True, gram=-1)
    np.testing.assert_array_equal(r_s["alpha"], r_g["alpha"])


def test_full_size_w3_streaming_prefix(S):
    """W3 at full size runs with the automatic row cache by default (the Gram path is
    opt-in); this keeps the plain streaming path (gram=-1, no cache decision
    forced) covered at full size too."""
    w = W.get("W3")
    X, y = w.train()
    k = 40
    r_or = O.train(X, y, w.C, w.kernel, w.gamma, w.tol, max_iter=k, trace_cap=k)
    r_g = S.svm_train_ex(X, y, w.C, w.kernel, w.gamma, w.tol, max_iter=k, want_f=True, trace_cap=k, gram=-1)
    _assert_exact(r_g, r_or)


@pytest.mark.parametrize("name,n,slots", [("W3", 2000, 4), ("W3", 2000, 64), ("W5", 3000, 8), ("W1", 200, 4),
                                          ("W4", 6000, 16)])
def test_row_cache_parity(S, monkeypatch, name, n, slots):
    """Kernel-row LRU cache on the streaming path (X not resident): tiny
    caches force constant eviction; results stay identical to the oracle and to the
    uncached solve."""
    monkeypatch.setenv("SVMB200_NO_RESIDENT", "1")
    w = W.get(name)
    X, y = w.train(n)
    r_g, r_or = _run_pair(S, w, X, y, cache_rows=slots)
    _assert_exact(r_g, r_or)
    r_nc = S.svm_train_ex(X, y, w.C, w.kernel, w.gamma, w.tol, cache_rows=-1)
    np.testing.assert_array_equal(r_nc["alpha"], r_g["alpha"])


def test_row_cache_with_virtual_ranks(S, monkeypatch):
    monkeypatch.setenv("SVMB200_NO_RESIDENT", "1")
    w = W.get("W5")
    X, y = w.train(2500)
    r_g, r_or = _run_pair(S, w, X, y, cache_rows=32, virtual_ranks=3)
    _assert_exact(r_g, r_or)


def _mixed_data(rng, n, runs):
    """Columns in runs of continuous (Gaussian, some negative, some exact 0/1 values
    mixed in) and binary (exactly 0/1) features, in the given order."""
    cols = []
    for kind, k in runs:
        if kind == "c":
            c = rng.normal(0.3, 0.6, (n, k)).astype(np.float32)
            c[rng.random((n, k)) < 0.2] = 1.0             # 0/1 values inside a continuous column
            c[rng.random((n, k)) < 0.2] = 0.0
            cols.append(c)
        else:
            cols.append((rng.random((n, k)) < 0.15).astype(np.float32))
    X = np.ascontiguousarray(np.concatenate(cols, axis=1))
    s = X[:, :3].sum(1) - X[:, -3:].sum(1) + 0.4 * rng.normal(size=n)
    y = np.where(s > np.median(s), 1, -1).astype(np.int8)
    return X, y


@pytest.mark.parametrize("runs,kern,gamma", [
    ((("c", 10), ("b", 44)), O.RBF, 1 / 54),                       # covtype-like order
    ((("c", 5), ("b", 40), ("c", 3), ("b", 33)), O.RBF, 0.05),     # interleaved runs, words split
    ((("b", 70), ("c", 6)), O.RBF, 0.1),                            # binary first: integral sums
    ((("c", 7), ("b", 36), ("c", 2)), O.LINEAR, 0.0),               # linear, negative partial sums
])
def test_mixed_rows_parity(S, monkeypatch, runs, kern, gamma):
    """Mixed compact rows (binary columns as bits, the rest fp32) equal
    the oracle and the dense fp32 path bit for bit, for several RPT values, virtual
    ranks and the row cache."""
    rng = np.random.default_rng(sum(k for _, k in runs))
    n = 2311
    X, y = _mixed_data(rng, n, runs)
    d = X.shape[1]
    w = W.Workload("mix", "", n, d, kern, gamma, 2.0, 1e-3, 0, 0, 0, None)
    r_or = O.train(X, y, w.C, w.kernel, w.gamma, w.tol, trace_cap=100000)
    r_g = S.svm_train_ex(X, y, w.C, w.kernel, w.gamma, w.tol, want_f=True, trace_cap=100000, cluster=-1)
    assert S.last_plan()["mode"].startswith("mixed")
    _assert_exact(r_g, r_or)
    for rpt in ("1", "2"):
        monkeypatch.setenv("SVMB200_RPT", rpt)
        r2 = S.svm_train_ex(X, y, w.C, w.kernel, w.gamma, w.tol, want_f=True, cluster=-1, ctas=37)
        _assert_exact(r2, r_or)
    monkeypatch.delenv("SVMB200_RPT")
    r3 = S.svm_train_ex(X, y, w.C, w.kernel, w.gamma, w.tol, want_f=True, virtual_ranks=3)
    _assert_exact(r3, r_or)
    monkeypatch.setenv("SVMB200_NO_RESIDENT", "1")          # streamed stages, with / without cache
    r4 = S.svm_train_ex(X, y, w.C, w.kernel, w.gamma, w.tol, want_f=True, cache_rows=16, cluster=-1)
    assert S.last_plan()["mode"] == "mixed+row-cache"
    _assert_exact(r4, r_or)
    r6 = S.svm_train_ex(X, y, w.C, w.kernel, w.gamma, w.tol, want_f=True, cache_rows=-1, cluster=-1)
    assert S.last_plan()["mode"] == "mixed-streamed"
    _assert_exact(r6, r_or)
    monkeypatch.delenv("SVMB200_NO_RESIDENT")
    monkeypatch.setenv("SVMB200_NO_COMPACT_PIVOTS", "1")          # pivots gathered dense
    r7 = S.svm_train_ex(X, y, w.C, w.kernel, w.gamma, w.tol, want_f=True, cluster=-1)
    _assert_exact(r7, r_or)
    monkeypatch.delenv("SVMB200_NO_COMPACT_PIVOTS")
    monkeypatch.setenv("SVMB200_NO_MIXED", "1")
    r5 = S.svm_train_ex(X, y, w.C, w.kernel, w.gamma, w.tol, want_f=True, cluster=-1)
    assert not S.last_plan()["mode"].startswith("mixed")
    _assert_exact(r5, r_or)


@pytest.mark.parametrize("case", ["W3", "levels256", "linear_neg"])
def test_dict_rows_parity(S, monkeypatch, case):
    """Dictionary-coded rows (<= 256 distinct fp32 values stored as one-byte codes, e.g.
    uint8 pixels) equal the oracle bit for bit: streamed / resident / row
    cache, RPT 1/2/4, virtual ranks; 257 distinct values fall back to fp32 rows."""
    rng = np.random.default_rng(41)
    if case == "W3":
        w = W.get("W3")
        X, y = w.train(1700)
    else:
        n, d = 1900, 40
        levels = rng.normal(0.0, 1.0, 256).astype(np.float32)
        levels[0] = 0.0
        X = levels[rng.integers(0, 256, size=(n, d))]
        X[rng.random((n, d)) < 0.5] = 0.0
        X = np.ascontiguousarray(X)
        s = X[:, :5].sum(1) + 0.3 * rng.normal(size=n)
        y = np.where(s > np.median(s), 1, -1).astype(np.int8)
        kern, gamma = (O.RBF, 0.03) if case == "levels256" else (O.LINEAR, 0.0)
        w = W.Workload("lv", "", n, d, kern, gamma, 1.0, 1e-3, 0, 0, 0, None)
    r_or = O.train(X, y, w.C, w.kernel, w.gamma, w.tol, trace_cap=100000)
    r_g = S.svm_train_ex(X, y, w.C, w.kernel, w.gamma, w.tol, want_f=True, trace_cap=100000, cluster=-1)
    assert S.last_plan()["mode"].startswith("dict")
    _assert_exact(r_g, r_or)
    for rpt in ("1", "2", "4"):
        monkeypatch.setenv("SVMB200_RPT", rpt)
        r2 = S.svm_train_ex(X, y, w.C, w.kernel, w.gamma, w.tol, want_f=True, cluster=-1, ctas=23)
        _assert_exact(r2, r_or)
    monkeypatch.delenv("SVMB200_RPT")
    r3 = S.svm_train_ex(X, y, w.C, w.kernel, w.gamma, w.tol, want_f=True, virtual_ranks=3)
    _assert_exact(r3, r_or)
    monkeypatch.setenv("SVMB200_NO_RESIDENT", "1")
    r4 = S.svm_train_ex(X, y, w.C, w.kernel, w.gamma, w.tol, want_f=True, cache_rows=16, cluster=-1)
    assert S.last_plan()["mode"] == "dict+row-cache"
    _assert_exact(r4, r_or)
    r5 = S.svm_train_ex(X, y, w.C, w.kernel, w.gamma, w.tol, want_f=True, cache_rows=-1, cluster=-1)
    assert S.last_plan()["mode"] == "dict-streamed"
    _assert_exact(r5, r_or)
    monkeypatch.delenv("SVMB200_NO_RESIDENT")
    if case == "levels256":
        X2 = X.copy()
        X2[0, 0] = np.float32(0.123456)                       # a 257th value
        r_o2 = O.train(X2, y, w.C, w.kernel, w.gamma, w.tol)
        r6 = S.svm_train_ex(X2, y, w.C, w.kernel, w.gamma, w.tol, want_f=True, cluster=-1)
        assert not S.last_plan()["mode"].startswith("dict")
        np.testing.assert_array_equal(r6["alpha"], r_o2.alpha)


@pytest.mark.parametrize("nt", ["256", "512"])
def test_consumer_warp_counts(S, monkeypatch, nt):
    """smo_persistent with 8 and with 16 consumer warps (NTC = 256 / 512; 16 is the default
    for narrow rows without row cache) equals the oracle on dense, mixed and streamed data."""
    monkeypatch.setenv("SVMB200_NT", nt)
    for name, n in (("W4", 5000), ("W5", 2600), ("W1", 200)):
        w = W.get(name)
        X, y = w.train(n)
        r_g, r_or = _run_pair(S, w, X, y, cluster=-1, cache_rows=-1)
        _assert_exact(r_g, r_or)
        assert S.last_plan()["threads"] == int(nt) + 64


def test_l2_prefetch_switch_keeps_results(S, monkeypatch):
    """SVMB200_L2_PF (L2 prefetch of the stages beyond the ring, a tuning switch) and the L2
    keep window change only where bytes come from: the trajectory stays the oracle's."""
    monkeypatch.setenv("SVMB200_NO_RESIDENT", "1")
    w = W.get("W5")
    X, y = w.train(3000)
    for pf, keep in (("2", "48"), ("6", "0")):
        monkeypatch.setenv("SVMB200_L2_PF", pf)
        monkeypatch.setenv("SVMB200_L2_KEEP_MB", keep)
        r_g, r_or = _run_pair(S, w, X, y, cluster=-1, cache_rows=-1)
        _assert_exact(r_g, r_or)


@pytest.fixture(scope="module")
def w5_small_model():
    w = W.get("W5")
    X, y = w.train(3000)
    r = O.train(X, y, w.C, w.kernel, w.gamma, w.tol)
    sv = r.alpha > 1e-8
    Xt, _ = w.test(700)
    Xs, cf = np.ascontiguousarray(X[sv]), (r.alpha * y)[sv]
    return w, Xs, cf, r.b, Xt, O.decision(Xs, cf, r.b, w.kernel, w.gamma, Xt)


@pytest.mark.parametrize("bn", ["128", "256"])
@pytest.mark.parametrize("expv", ["0", "1", "2", "3", "4", "5"])
def test_predict_tensor_exp_variants(S, monkeypatch, w5_small_model, expv, bn):
    """The tensor-core epilogue's exp variants (SVMB200_PREDICT_EXP) and both tile widths
    (SVMB200_PREDICT_BN: 128 or 256 support vectors per accumulator tile; 700 test rows,
    a ragged last tile of SVs) all stay within BASELINE.json's 1e-4 of the oracle."""
    monkeypatch.setenv("SVMB200_PREDICT_EXP", expv)
    monkeypatch.setenv("SVMB200_PREDICT_BN", bn)
    w, Xs, cf, b, Xt, d_o = w5_small_model
    d_t = S.svm_predict(Xs, cf, b, w.kernel, w.gamma, Xt, mode=S.PREDICT_TENSOR)
    assert np.max(np.abs(d_t - d_o)) <= 1e-4


def test_predict_tensor_row_factor_fallback(S, monkeypatch, w5_small_model):
    """Epilogue variant 5 takes exp(-gamma |t|^2) out of every kernel value only for warps
    whose rows all have gamma |t|^2 <= 600 (so exp(x + gamma |t|^2) stays finite).  Test
    rows shifted far from the origin (gamma |t|^2 ~ 10^3; the kernel values are unchanged)
    take the fallback, which is variant 3's arithmetic: bit-identical results; unshifted
    rows take the factored form and agree with variant 3 to rounding."""
    w, Xs, cf, b, Xt, _ = w5_small_model
    shift = np.float32(np.sqrt(1000.0 / (w.gamma * Xs.shape[1])))
    res = {}
    for v in ("3", "5"):
        monkeypatch.setenv("SVMB200_PREDICT_EXP", v)
        res[v] = (S.svm_predict(Xs + shift, cf, b, w.kernel, w.gamma, Xt + shift, mode=S.PREDICT_TENSOR),
                  S.svm_predict(Xs, cf, b, w.kernel, w.gamma, Xt, mode=S.PREDICT_TENSOR))
    assert np.array_equal(res["3"][0], res["5"][0])
    assert np.max(np.abs(res["3"][1] - res["5"][1])) <= 1e-10


@pytest.mark.parametrize("name,n,vr,ctas", [("W5", 2500, 1, 0), ("W5", 2500, 4, 0), ("W4", 6000, 1, 0),
                                             ("W3", 1500, 2, 0), ("W5", 2500, 3, 17)])
def test_wide_poll_parity(S, monkeypatch, name, n, vr, ctas):
    """The wide record poll (every consumer thread polls a slice of the records; the
    automatic choice above 320 records, i.e. three or more GPUs) forced on one GPU: the same
    trajectory, alpha, f and b as the oracle, with virtual ranks and ragged CTA counts."""
    monkeypatch.setenv("SVMB200_WIDE_POLL", "1")
    w = W.get(name)
    X, y = w.train(n)
    r_g, r_or = _run_pair(S, w, X, y, virtual_ranks=vr, ctas=ctas, cluster=-1)
    assert S.last_plan()["cluster"] == 0 and S.last_plan()["poll"] == "wide"
    _assert_exact(r_g, r_or)


@pytest.mark.parametrize("name,n", [("W5", 2500), ("W4", 6000)])
def test_record_duplication_hook(S, monkeypatch, name, n):
    """SVMB200_XCH_DUP = 8 stores every record in 8 slots (one GPU then polls the 1,184
    records of an 8-GPU exchange, a timing aid): the wide poll is chosen automatically and
    the result still equals the oracle bit for bit; with the wide poll forced off, too."""
    monkeypatch.setenv("SVMB200_XCH_DUP", "8")
    w = W.get(name)
    X, y = w.train(n)
    r_g, r_or = _run_pair(S, w, X, y, cluster=-1)
    assert S.last_plan()["poll"] == "wide"
    _assert_exact(r_g, r_or)
    monkeypatch.setenv("SVMB200_WIDE_POLL", "0")
    r_g, r_or = _run_pair(S, w, X, y, cluster=-1)
    assert S.last_plan()["poll"] == "warp"
    _assert_exact(r_g, r_or)


@pytest.mark.parametrize("nt", ["448", "512"])
def test_mixed_rows_only_kernel(S, monkeypatch, nt):
    """The mixed-rows-only 16-warp instantiations (MIX; 512 consumer threads, or 448 so the
    16 warps get 128 registers each) equal the oracle on mixed compact rows, RBF and linear,
    with ragged tiles; SVMB200_NO_SPECIALISE gives the general kernel the same result."""
    monkeypatch.setenv("SVMB200_NT", nt)
    for name, n, kern in (("W4", 5000, None), ("W4", 3333, O.LINEAR)):
        w = W.get(name)
        if kern is not None:
            import dataclasses
            w = dataclasses.replace(w, kernel=kern)
        X, y = w.train(n)
        r_g, r_or = _run_pair(S, w, X, y, cluster=-1, cache_rows=-1)
        _assert_exact(r_g, r_or)
        plan = S.last_plan()
        assert plan["threads"] == int(nt) + 64 and plan["kernel"].endswith(",mix>"), plan


@pytest.mark.parametrize("spec", ["1", None])
def test_dense_only_kernel(S, monkeypatch, spec):
    """The dense-streamed-only 8-warp instantiation (SPEC 2, W5's kernel) and, with
    SVMB200_NO_SPECIALISE, the general one both equal the oracle on streamed fp32 rows
    (RBF, and linear with virtual ranks)."""
    if spec:
        monkeypatch.setenv("SVMB200_NO_SPECIALISE", spec)
    import dataclasses
    # (few CTAs, so each holds >= 2 rows per consumer thread: the instantiations with
    # RPT 2 and 4; alpha in shared memory (<= 2048 rows per CTA) and in HBM)
    for w, n, vr, ctas in ((W.get("W5"), 2600, 1, 4), (W.get("W5"), 5000, 1, 2),
                           (dataclasses.replace(W.get("W5"), kernel=O.LINEAR), 1800, 2, 4)):
        X, y = w.train(n)
        r_g, r_or = _run_pair(S, w, X, y, cluster=-1, cache_rows=-1, virtual_ranks=vr, ctas=ctas)
        _assert_exact(r_g, r_or)
        assert S.last_plan()["kernel"].endswith(",dense>") == (spec is None), S.last_plan()


@pytest.mark.parametrize("cache", [-1, 0])
def test_dict_only_kernel(S, monkeypatch, cache):
    """The dictionary-rows-only 8-warp instantiation (SPEC 3, W3's kernel), with and
    without the row cache, equals the oracle (W3 subset, few CTAs so each thread holds
    >= 2 rows); the general kernel (SVMB200_NO_SPECIALISE) gives the same result."""
    w = W.get("W3")
    X, y = w.train(2000)
    r_g, r_or = _run_pair(S, w, X, y, cluster=-1, cache_rows=cache, ctas=3)
    _assert_exact(r_g, r_or)
    assert S.last_plan()["kernel"].endswith(",dict>"), S.last_plan()
    monkeypatch.setenv("SVMB200_NO_SPECIALISE", "1")
    r_g2 = S.svm_train_ex(X, y, w.C, w.kernel, w.gamma, w.tol, cluster=-1, cache_rows=cache, ctas=3)
    assert not S.last_plan()["kernel"].endswith(",dict>")
    assert np.array_equal(r_g2["alpha"], r_g["alpha"]) and r_g2["b"] == r_g["b"]
