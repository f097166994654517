"""GPU parity of the projected-gradient dual trainer (svm_train_gd_dev; SURVEY §8(f)
NEXT-3, R23-R26) against the oracle (oracle_gd_train) on the same seeded
inputs.  Both sides sum g_i = sum_j K_ij v_j in ascending j with one fma per term over
the same correctly rounded kernel values, so alpha, b and W are compared bit for bit."""
import numpy as np
import pytest

from gen import workloads as W
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S():
    import paper_2311_14908_b200 as S
    S.lib()
    return S


def _gpu(S, X, y, C, kern, gamma, lr, epochs):
    import torch
    r = S.svm_train_gd_dev(torch.from_numpy(np.ascontiguousarray(X)).cuda(), torch.from_numpy(y).cuda(),
                           C, kern, gamma, lr, epochs)
    return r["alpha"].cpu().numpy(), r["b"], r["info"]


@pytest.mark.parametrize("name,n,lr,epochs", [
    ("W1", 200, 0.01, 50), ("W2", 1500, 1e-3, 7), ("W3", 777, 0.02, 5), ("W5", 1031, 0.05, 12),
    ("W4", 2049, 0.01, 1), ("W2", 600, 1e-3, 0)])
def test_gd_bit_identical_to_oracle(S, name, n, lr, epochs):
    w = W.get(name)
    X, y = w.train(n)
    a, b, info = _gpu(S, X, y, w.C, w.kernel, w.gamma, lr, epochs)
    r = O.gd_train(X, y, w.C, w.kernel, w.gamma, lr, epochs)
    np.testing.assert_array_equal(a, r.alpha)
    assert b == r.b
    assert info["objective"] == r.W
    assert info["epochs"] == epochs
    assert S.last_plan()["kernel"] == "k_gd_epoch"


def test_gd_two_point_box_optimum(S):
    """x = (1, 3), y = (+1, -1), C = 10: alpha* = (10, 31/9), W* = 241/18, b = 0."""
    X = np.array([[1.0], [3.0]], np.float32)
    y = np.array([1, -1], np.int8)
    a, b, info = _gpu(S, X, y, 10.0, S.LINEAR, 0.0, 0.05, 4000)
    np.testing.assert_allclose(a, [10.0, 31.0 / 9.0], rtol=0, atol=1e-12)
    assert abs(info["objective"] - 241.0 / 18.0) <= 1e-12 and abs(b) <= 1e-12


def test_gd_errors(S):
    import torch
    X = torch.zeros((4, 2), dtype=torch.float32, device="cuda")
    y = torch.tensor([1, -1, 1, -1], dtype=torch.int8, device="cuda")
    for lr, ep in ((0.0, 5), (-1.0, 5), (float("nan"), 5), (0.1, -1)):
        with pytest.raises(S.SvmError):
            S.svm_train_gd_dev(X, y, 1.0, S.RBF, 0.5, lr, ep)
    with pytest.raises(S.SvmError):
        S.svm_train_gd_dev(X, torch.ones(4, dtype=torch.int8, device="cuda"), 1.0, S.RBF, 0.5, 0.1, 3)


def test_gd_full_size_w2_sampled(S):
    """Full-size W2 (the bench configuration): after two epochs alpha_i =
    clamp(lr + lr (1 - y_i lr sum_j K_ij y_j)) -- checked on 48 sampled rows against the
    oracle's kernel rows (different summation order: 1e-12 relative)."""
    w = W.get("W2")
    X, y = w.train()
    lr = 1e-4
    a, b, info = _gpu(S, X, y, w.C, w.kernel, w.gamma, lr, 2)
    rng = np.random.default_rng(3)
    for i in rng.choice(len(y), 48, replace=False):
        k = O.kernel_row(X, int(i), w.kernel, w.gamma)
        g = lr * float(np.dot(k, y.astype(np.float64)))
        exp = min(w.C, max(0.0, lr + lr * (1.0 - y[i] * g)))
        assert abs(a[i] - exp) <= 1e-12 * abs(exp)
    n = len(y)
    assert 8 * n * n <= info["gram_bytes"] < 8 * n * (n + 256)
