"""Pins of the CPU oracle against values fixed by the paper/SPEC and by mathematics
(closed forms, known margins, the exact exponential).  CPU only.

Each fixture under tests/golden/ carries its citation."""
import json
import math
import os

import numpy as np
import pytest

from oracle import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")
KIND = {"linear": O.LINEAR, "rbf": O.RBF}


def gold(name):
    with open(os.path.join(GOLD, name)) as fh:
        return json.load(fh)


# ----------------------------------------------------------------------------- exp
def _mp_exp(x):
    import mpmath
    mpmath.mp.prec = 256
    return float(mpmath.exp(mpmath.mpf(x)))  # round-to-nearest of a 256-bit value


def test_exp_correctly_rounded_vs_mpmath():
    """oracle_exp_cr is the exponential rounded once (reading R14); pinned to
    mpmath at 256 bits over the RBF argument range [-708, 0]."""
    rng = np.random.default_rng(11)
    xs = np.concatenate([
        -rng.uniform(0, 708, 4000),
        -np.exp(rng.uniform(-45, 1.5, 4000)),          # tiny |x|: exp(x) ~ 1 - |x|
        -np.arange(0, 60, 0.5),                         # Adult-like arguments -gamma*D
        -(np.arange(1, 2000) * 0.0125 / 255.0 ** 2),    # MNIST-like grid
        np.array([-708.0, -707.999999, -1e-300, -5e-324, -0.0]),
    ])
    before = O.exp_ambiguous_count()
    bad = [x for x in xs if O.exp_cr(x) != _mp_exp(x)]
    assert not bad, f"{len(bad)} mismatches, e.g. {bad[:3]}"
    assert O.exp_ambiguous_count() == before


def test_exp_special_values():
    assert O.exp_cr(0.0) == 1.0
    assert O.exp_cr(-0.0) == 1.0
    assert O.exp_cr(-1.0) == float.fromhex("0x1.78b56362cef38p-2")   # e^-1 rounded
    assert O.exp_cr(-708.5) == 0.0            # DESIGN.md reading R15: arguments < -708 -> 0
    assert O.exp_cr(-2.0) == pytest.approx(0.1353352832366127, abs=0)


# -------------------------------------------------------------------------- kernels
def test_kernel_examples():
    g = gold("kernel_examples.json")
    for e in g["eval"]:
        a = np.array(e["a"], np.float32); b = np.array(e["b"], np.float32)
        v = O.kernel(a, b, KIND[e["kernel"]], e.get("gamma", 0.0))
        assert v == e["value"], e["cite"]
    r = g["row"]
    row = O.kernel_row(np.array(r["X"], np.float32), r["i"], KIND[r["kernel"]])
    assert row.tolist() == r["value"]
    X = np.array(g["gram"]["X"], np.float32)
    G = np.stack([O.kernel_row(X, i, O.LINEAR) for i in range(2)])
    assert G.tolist() == g["gram"]["value"]


def test_kernel_symmetry_and_range():
    """K(x,y) == K(y,x) exactly; RBF in (0,1]; Gram PSD spot check."""
    rng = np.random.default_rng(3)
    X = rng.standard_normal((7, 5)).astype(np.float32)
    for kind, gamma in ((O.LINEAR, 0.0), (O.RBF, 0.3)):
        G = np.stack([O.kernel_row(X, i, kind, gamma) for i in range(7)])
        assert np.array_equal(G, G.T)
        assert np.linalg.eigvalsh(G).min() >= -1e-8
        if kind == O.RBF:
            assert np.all(G > 0) and np.all(G <= 1) and np.all(np.diag(G) == 1.0)


def test_rbf_against_independent_formula():
    """RBF value vs numpy's own exp of the direct distance (independent evaluation,
    agrees to rounding of the distance sum; exact equality is pinned by the mpmath test)."""
    rng = np.random.default_rng(5)
    X = rng.standard_normal((20, 9)).astype(np.float32)
    for i in range(20):
        row = O.kernel_row(X, i, O.RBF, 0.21)
        ref = np.exp(-0.21 * ((X.astype(np.float64) - X[i].astype(np.float64)) ** 2).sum(1))
        np.testing.assert_allclose(row, ref, rtol=1e-14, atol=0)


# ------------------------------------------------------------------ init / selection
def test_init_and_selection_forced_states():
    # y = [+1, -1] -> f = [-1, +1], b_up = -1, b_low = +1; S:L200 pair (1, 0)
    X = np.array([[0.0], [1.0]], np.float32)
    y = np.array([1, -1], np.int8)
    r = O.train(X, y, 1.0, O.LINEAR, max_iter=1, tol=1e-3, trace_cap=4)
    assert r.trace[0].tolist() == [0, 1]                  # (i_up, i_low)
    ok, iu, il, bu, bl = O.select(-y.astype(float), y, np.zeros(2), 1.0)
    assert (ok, iu, il, bu, bl) == (True, 0, 1, -1.0, 1.0)
    # y = [+1, +1, -1] -> i_up = 0 (lowest index)
    y3 = np.array([1, 1, -1], np.int8)
    ok, iu, il, _, _ = O.select(-y3.astype(float), y3, np.zeros(3), 1.0)
    assert iu == 0 and il == 2
    # f = [0.5, 0.5, -0.5], all alpha interior -> i_up = 2, i_low = 0
    ok, iu, il, bu, bl = O.select([0.5, 0.5, -0.5], [1, 1, 1], [0.5, 0.5, 0.5], 1.0)
    assert (iu, il) == (2, 0) and (bu, bl) == (-0.5, 0.5)


def test_single_class_rejected():
    # S:L193 all-positive labels -> error
    with pytest.raises(ValueError):
        O.train(np.zeros((3, 1), np.float32), np.ones(3, np.int8), 1.0, O.LINEAR)


def test_selection_against_exhaustive_scan():
    """S:L202 random n=20 states: the selection equals a double-loop scan."""
    rng = np.random.default_rng(7)
    for _ in range(50):
        n, C = 20, 1.0
        y = np.where(rng.random(n) < 0.5, 1, -1).astype(np.int8)
        alpha = rng.choice([0.0, C, 0.3, 0.7], size=n)
        f = rng.choice([-1.0, 0.0, 0.25, 0.5, 1.0], size=n)   # many exact ties
        ok, iu, il, bu, bl = O.select(f, y, alpha, C)
        up = [j for j in range(n) if (y[j] == 1 and alpha[j] < C) or (y[j] == -1 and alpha[j] > 0)]
        lo = [j for j in range(n) if (y[j] == 1 and alpha[j] > 0) or (y[j] == -1 and alpha[j] < C)]
        if not up or not lo:
            assert not ok
            continue
        eu = min(up, key=lambda j: (f[j], j))
        el = min(lo, key=lambda j: (-f[j], j))
        assert (iu, il) == (eu, el)


# ---------------------------------------------------------------------- closed forms
def _coef_decision(X, y, r, kind, gamma, pts):
    sv = r.alpha > 1e-8
    return O.decision(X[sv], (r.alpha * y)[sv], r.b, kind, gamma, np.array(pts, np.float32))


@pytest.mark.parametrize("name", ["two_point_linear.json", "three_point_linear.json"])
def test_linear_closed_forms(name):
    g = gold(name)
    X = np.array(g["X"], np.float32); y = np.array(g["y"], np.int8)
    r = O.train(X, y, g["C"], O.LINEAR, tol=g["tol"])
    assert r.converged and r.iterations == g["iterations"]
    np.testing.assert_allclose(r.alpha, g["alpha"], rtol=0, atol=1e-15)
    assert r.b == pytest.approx(g["b"], abs=1e-15)
    assert O.dual_objective(X, y, r.alpha, O.LINEAR) == pytest.approx(g["W"], abs=1e-15)
    dec = _coef_decision(X, y, r, O.LINEAR, 0.0, g["decision"]["x"])
    np.testing.assert_allclose(dec, g["decision"]["value"], atol=1e-14)


def test_clipped_two_point():
    g = gold("two_point_clipped.json")
    X = np.array(g["X"], np.float32); y = np.array(g["y"], np.int8)
    r = O.train(X, y, g["C"], O.LINEAR, tol=g["tol"])
    assert r.iterations == 1 and r.converged
    assert r.alpha.tolist() == g["alpha"]          # snapped exactly onto C
    assert (r.b_up, r.b_low, r.b) == (g["b_up"], g["b_low"], g["b"])
    assert O.dual_objective(X, y, r.alpha, O.LINEAR) == g["W"]


def test_rbf_two_point():
    g = gold("rbf_two_point.json")
    X = np.array(g["X"], np.float32); y = np.array(g["y"], np.int8)
    for c in g["cases"]:
        r = O.train(X, y, c["C"], O.RBF, g["gamma"], tol=1e-12)
        np.testing.assert_allclose(r.alpha, c["alpha"], rtol=1e-14)
        assert O.dual_objective(X, y, r.alpha, O.RBF, g["gamma"]) == pytest.approx(c["W"], rel=1e-14)
        assert abs(r.b - c["b"]) < 1e-12


def test_eta_zero_duplicates():
    g = gold("eta_zero_duplicates.json")
    X = np.array(g["X"], np.float32); y = np.array(g["y"], np.int8)
    r = O.train(X, y, g["C"], O.RBF, g["gamma"], tol=g["tol"], trace_cap=16)
    # first step pairs the duplicates (0, 1): eta = 0, the step runs to the bound
    assert r.trace[0].tolist() == [0, 1]
    np.testing.assert_allclose(r.alpha, g["alpha"], atol=1e-12)
    assert O.dual_objective(X, y, r.alpha, O.RBF, g["gamma"]) == pytest.approx(g["W"], abs=1e-12)
    assert r.b == pytest.approx(g["b"], abs=1e-3)


def test_separable_toy_known_margin():
    g = gold("separable_toy.json")
    X = np.array(g["X"], np.float32); y = np.array(g["y"], np.int8)
    r = O.train(X, y, g["C"], O.LINEAR, tol=g["tol"])
    assert r.converged
    w = ((r.alpha * y)[:, None] * X.astype(np.float64)).sum(0)
    np.testing.assert_allclose(w, g["w"], atol=1e-5)
    assert abs(r.b - g["b"]) < 1e-5
    assert 2.0 / np.linalg.norm(w) == pytest.approx(g["margin"], rel=1e-5)
    assert O.dual_objective(X, y, r.alpha, O.LINEAR) == pytest.approx(g["W"], rel=1e-5)
    # every training point on or outside the margin
    assert np.all(y * (X.astype(np.float64) @ w + r.b) >= 1 - 1e-5)


def test_decision_empty_support_is_bias():
    # empty support set -> b
    dec = O.decision(np.zeros((0, 3), np.float32), np.zeros(0), 0.75, O.RBF, 0.1,
                     np.ones((4, 3), np.float32))
    assert dec.tolist() == [0.75] * 4


def test_dual_objective_examples():
    # W(0) = 0, two-point W(0.5, 0.5) = 0.5; f-form identity
    X = np.array([[1.0], [3.0]], np.float32); y = np.array([1, -1], np.int8)
    assert O.dual_objective(X, y, np.zeros(2), O.LINEAR) == 0.0
    assert O.dual_objective(X, y, np.array([0.5, 0.5]), O.LINEAR) == 0.5
    rng = np.random.default_rng(9)
    X = rng.standard_normal((30, 4)).astype(np.float32)
    y = np.where(rng.random(30) < 0.5, 1, -1).astype(np.int8)
    r = O.train(X, y, 2.0, O.RBF, 0.4)
    W = O.dual_objective(X, y, r.alpha, O.RBF, 0.4)
    assert O.dual_objective_from_f(r.alpha, y, r.f) == pytest.approx(W, rel=1e-12)
