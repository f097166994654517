"""Pins of the projected-gradient dual trainer in the oracle (oracle_gd_train; SURVEY
§8(f) NEXT-3, the paper's TensorFlow path P:L174-179 read as full-batch projected
gradient ascent on W, R23-R26).  CPU only.

The pins come from outside the oracle's own formula: the first epoch from alpha = 0 in
closed form (the gradient at the origin is all ones), the two-point linear
dual maximised over the box by hand (alpha* = (C, (C + 1/3)/3), W* = 241/18 for C = 10),
and a brute-force active-set solution of the box-constrained QP on tiny RBF problems."""
import itertools

import numpy as np
import pytest

from oracle import oracle as O


def test_first_epoch_closed_form():
    """From alpha = 0 the gradient is 1 everywhere, so one epoch gives alpha = min(C, lr);
    with integer linear data g = lr K y is exact."""
    rng = np.random.default_rng(1)
    X = rng.integers(-3, 4, size=(7, 3)).astype(np.float32)
    y = np.array([1, -1, 1, 1, -1, -1, 1], np.int8)
    K = X.astype(np.int64) @ X.astype(np.int64).T
    r = O.gd_train(X, y, 10.0, O.LINEAR, 0.0, 0.25, 1)
    assert np.all(r.alpha == 0.25)
    np.testing.assert_array_equal(r.g, 0.25 * (K @ y.astype(np.int64)))
    r = O.gd_train(X, y, 0.1, O.LINEAR, 0.0, 0.25, 1)          # clipped at C
    assert np.all(r.alpha == 0.1)


def test_zero_epochs():
    X = np.array([[0.0], [1.0], [3.0]], np.float32)
    y = np.array([1, -1, 1], np.int8)
    r = O.gd_train(X, y, 1.0, O.RBF, 0.5, 0.01, 0)
    assert np.all(r.alpha == 0) and np.all(r.g == 0) and r.b == 0.0 and r.W == 0.0


def test_two_point_linear_box_optimum():
    """x = (1, 3), y = (+1, -1): W(a) = a1 + a2 - (a1 - 3 a2)^2 / 2.  Over [0, 10]^2 the
    maximum is at a1 = C, a1 - 3 a2 = -1/3 (grad_2 = 0), i.e. a* = (10, 31/9),
    W* = 241/18; there the free multiplier has y g = 1, so b = 0."""
    X = np.array([[1.0], [3.0]], np.float32)
    y = np.array([1, -1], np.int8)
    r = O.gd_train(X, y, 10.0, O.LINEAR, 0.0, 0.05, 4000)
    np.testing.assert_allclose(r.alpha, [10.0, 31.0 / 9.0], rtol=0, atol=1e-12)
    assert abs(r.W - 241.0 / 18.0) <= 1e-12
    assert abs(r.b) <= 1e-12


def _int_problem():
    """Integer linear data: K = X X^T and every g below are exact small integers times a
    power of two, so the expected biases are exact in fp64."""
    X = np.array([[2, 0], [1, 1], [0, 3], [-1, 2], [3, -1], [1, -2]], np.float32)
    y = np.array([1, 1, -1, -1, 1, -1], np.int8)
    K = X.astype(np.int64) @ X.astype(np.int64).T
    return X, y, K


def test_bias_interior_svs_after_one_epoch():
    """Bias with free multipliers away from the optimum (R25): one epoch from
    alpha = 0 gives alpha = lr < C everywhere (all interior), g = lr K y, and
    b = mean_i (y_i - g_i), written out here from the definition.  The data make that
    mean clearly non-zero, so a sign slip (g - y) or a wrong set fails."""
    X, y, K = _int_problem()
    lr = 0.125
    r = O.gd_train(X, y, 10.0, O.LINEAR, 0.0, lr, 1)
    assert np.all(r.alpha == lr)
    g = lr * (K @ y.astype(np.int64))
    np.testing.assert_array_equal(r.g, g)
    b_def = float(np.mean(y.astype(np.float64) - g))
    assert abs(b_def) > 0.1
    assert r.b == b_def


def test_bias_fallback_all_at_bound():
    """No interior multiplier: one epoch with lr > C puts every alpha at C, and the bias
    falls back to the midpoint -(max g + min g)/2 over the SVs (S:L307 fallback), with
    g = C K y."""
    X, y, K = _int_problem()
    C = 0.5
    r = O.gd_train(X, y, C, O.LINEAR, 0.0, 4.0, 1)
    assert np.all(r.alpha == C)
    g = C * (K @ y.astype(np.int64))
    b_mid = -(g.max() + g.min()) / 2.0
    assert b_mid != 0.0 and b_mid != -float(np.mean(y - g))
    assert r.b == b_mid


def test_bias_fallback_mixed_bounds():
    """Multipliers at 0 and at C but none interior: the fallback ranges over the SVs
    (alpha > 1e-8) only.  Two epochs with lr = 4, C = 1 on two well-separated pairs:
    epoch 1 sets alpha = C; epoch 2 gives y g >> 1 for the far pair (alpha -> 0) and
    y g < 1 for the overlapping pair (alpha stays at C)."""
    X = np.array([[0.0], [0.25], [5.0], [-5.0]], np.float32)
    y = np.array([1, -1, 1, -1], np.int8)
    r = O.gd_train(X, y, 1.0, O.LINEAR, 0.0, 4.0, 2)
    # hand computation: alpha1 = (1, 1, 1, 1); g1 = K y with K = x x^T:
    #   v = (1, -1, 1, -1); K v = x * (0 - 0.25 + 5 + 5) = 9.75 x
    #   grad = 1 - y * 9.75 x = (1, 1 + 2.4375, 1 - 48.75, 1 - 48.75) -> alpha2 = (1, 1, 0, 0)
    np.testing.assert_array_equal(r.alpha, [1.0, 1.0, 0.0, 0.0])
    # final g = K (alpha2 o y) = x * (0 - 0.25) = (0, -0.0625, -1.25, 1.25); SVs = {0, 1}
    np.testing.assert_array_equal(r.g, [0.0, -0.0625, -1.25, 1.25])
    assert r.b == -(0.0 + -0.0625) / 2.0          # over the SVs only (all-i midpoint would be 0)


def _box_qp_bruteforce(Q, C):
    """max 1'a - a'Qa/2 over [0, C]^n: every (0 / C / free) pattern whose free block
    solves Q_FF a_F = 1 - Q_FB a_B inside (0, C) with the bounded gradients pointing out."""
    n = Q.shape[0]
    best = None
    for pat in itertools.product((0, 1, 2), repeat=n):
        a = np.array([0.0 if p == 0 else C for p in pat])
        F = [i for i, p in enumerate(pat) if p == 2]
        if F:
            B = [i for i in range(n) if i not in F]
            rhs = 1.0 - Q[np.ix_(F, B)] @ a[B] if B else np.ones(len(F))
            try:
                a[F] = np.linalg.solve(Q[np.ix_(F, F)], rhs)
            except np.linalg.LinAlgError:
                continue
            if np.any(a[F] <= 0) or np.any(a[F] >= C):
                continue
        grad = 1.0 - Q @ a
        ok = all((p == 0 and grad[i] <= 1e-9) or (p == 1 and grad[i] >= -1e-9) or p == 2
                 for i, p in enumerate(pat))
        if ok:
            W = a.sum() - 0.5 * a @ Q @ a
            if best is None or W > best[1]:
                best = (a, W)
    return best


@pytest.mark.parametrize("seed", range(8))
def test_matches_bruteforce_box_qp(seed):
    """Tiny RBF problems: the GD iterate converges to the brute-force box-QP optimum
    (lr = 1 / lambda_max, contraction by 1 - lambda_min / lambda_max per epoch)."""
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(3, 7))
    X = rng.normal(size=(n, 2)).astype(np.float32)
    y = np.where(rng.random(n) < 0.5, 1, -1).astype(np.int8)
    y[0], y[1] = 1, -1
    C = float(rng.choice([0.3, 1.0, 5.0]))
    gamma = 0.7
    Xd = X.astype(np.float64)
    D = ((Xd[:, None, :] - Xd[None, :, :]) ** 2).sum(-1)
    K = np.exp(-gamma * D)
    Q = (y[:, None] * y[None, :]) * K
    ev = np.linalg.eigvalsh(Q)
    lr = 1.0 / ev[-1]
    epochs = int(min(400000, 60 * ev[-1] / ev[0]))
    a_star, W_star = _box_qp_bruteforce(Q, C)
    r = O.gd_train(X, y, C, O.RBF, gamma, lr, epochs)
    assert np.all(r.alpha >= 0) and np.all(r.alpha <= C)
    assert r.W <= W_star + 1e-12 * max(1.0, abs(W_star))      # a feasible point
    assert abs(r.W - W_star) <= 1e-9 * max(1.0, abs(W_star))
    np.testing.assert_allclose(r.alpha, a_star, atol=1e-6 * C)
    # g is K (alpha o y) of the returned alpha; W from g equals the quadratic form
    v = r.alpha * y
    np.testing.assert_allclose(r.g, K @ v, rtol=1e-13, atol=1e-13)


def test_smo_optimum_below_box_optimum():
    """The SMO solution satisfies the extra equality sum alpha y = 0, so its dual value
    is bounded by the box-only optimum the GD iterate approaches."""
    rng = np.random.default_rng(5)
    X = rng.normal(size=(40, 3)).astype(np.float32)
    y = np.where(X[:, 0] + 0.3 * rng.normal(size=40) > 0, 1, -1).astype(np.int8)
    r_smo = O.train(X, y, 1.0, O.RBF, 0.5, 1e-6)
    W_smo = O.dual_objective(X, y, r_smo.alpha, O.RBF, 0.5)
    r = O.gd_train(X, y, 1.0, O.RBF, 0.5, 0.05, 20000)
    assert W_smo <= r.W + 1e-9
