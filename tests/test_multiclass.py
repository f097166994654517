"""One-against-one multiclass (Fig. 4; SPEC.md
L335-413).  Host logic on CPU; the batched GPU solves against the oracle on the GPU."""
import numpy as np
import pytest

from gen import workloads as W
from oracle import oracle as O


def test_enumerate_pairs_spec_examples():
    from paper_2311_14908_b200.multiclass import enumerate_pairs
    assert enumerate_pairs(3) == [(0, 1), (0, 2), (1, 2)]
    assert enumerate_pairs(2) == [(0, 1)]
    assert len(enumerate_pairs(9)) == 36                            # S:L359 (Table 4 "/9")
    with pytest.raises(ValueError):
        enumerate_pairs(1)


def test_binary_problem_convention():
    from paper_2311_14908_b200.multiclass import binary_problem
    labels = np.array([2, 0, 1, 0, 2, 1])
    idx, y = binary_problem(labels, (0, 2))
    assert idx.tolist() == [0, 1, 3, 4]                             # original order
    assert y.tolist() == [-1, 1, 1, -1]                             # +1 for the lower id
    with pytest.raises(ValueError):
        binary_problem(np.array([0, 0, 1]), (0, 2))


def test_vote_spec_examples():
    from paper_2311_14908_b200.multiclass import vote
    # m = 3, decisions giving votes (2, 1, 0) -> class 0
    d = {(0, 1): np.array([1.0]), (0, 2): np.array([1.0]), (1, 2): np.array([1.0])}
    assert vote(d, 3).tolist() == [0]
    # cyclic tie (1, 1, 1) -> class 0: 0 beats 1, 2 beats 0, 1 beats 2
    d = {(0, 1): np.array([1.0]), (0, 2): np.array([-1.0]), (1, 2): np.array([1.0])}
    assert vote(d, 3).tolist() == [0]
    # m = 2 reduces to the sign of the decision value; 0 votes for the lower class
    d = {(0, 1): np.array([0.5, -0.5, 0.0])}
    assert vote(d, 2).tolist() == [0, 1, 0]


def _oracle_ovo(X, labels, m, w):
    """Independent OvO on the oracle: plain loops, SPEC conventions."""
    models = {}
    for a in range(m):
        for b in range(a + 1, m):
            idx = [i for i in range(len(labels)) if labels[i] in (a, b)]
            y = np.array([1 if labels[i] == a else -1 for i in idx], np.int8)
            r = O.train(X[idx], y, w.C, w.kernel, w.gamma, w.tol)
            models[(a, b)] = (np.array(idx), y, r)
    return models


def _oracle_predict(models, X, m, w, Xt):
    votes = np.zeros((len(Xt), m), dtype=int)
    for (a, b), (idx, y, r) in models.items():
        sv = r.alpha > 1e-8
        dec = O.decision(X[idx][sv], (r.alpha * y)[sv], r.b, w.kernel, w.gamma, Xt)
        for i, v in enumerate(dec):
            votes[i, a if v >= 0 else b] += 1
    out = []
    for row in votes:
        best = 0
        for c in range(1, m):
            if row[c] > row[best]:
                best = c
        out.append(best)
    return np.array(out)


@pytest.mark.gpu
@pytest.mark.parametrize("batch", [1, 8])
def test_ovo_matches_oracle(batch):
    """Pavia-like (Table 1: 9 classes, 102 bands) at 40 samples per class: every
    one of the 36 binary models equals the oracle's bit for bit, whatever the batching
    (pool equivalence), and the voted predictions are identical."""
    import paper_2311_14908_b200 as S
    from paper_2311_14908_b200.multiclass import predict_ovo, train_ovo
    m = 9
    X, labels = W.pavia_like(40, seed=7)
    Xt, _ = W.pavia_like(20, seed=8)
    w = W.Workload("pavia", "", len(labels), 102, O.RBF, 1.0 / 102, 10.0, 1e-3, 0, 0, 0, None)
    model = train_ovo(X, labels, m, w.C, w.kernel, w.gamma, w.tol, batch=batch)
    ref = _oracle_ovo(X, labels, m, w)
    for pair, (idx, y, r) in ref.items():
        got = model.models[pair]
        assert got["info"]["iterations"] == r.iterations, pair
        np.testing.assert_array_equal(got["alpha"], r.alpha)
        assert got["b"] == r.b
    pred = predict_ovo(model, X, Xt, mode=S.PREDICT_EXACT)
    np.testing.assert_array_equal(pred, _oracle_predict(ref, X, m, w, Xt))


@pytest.mark.gpu
def test_batch_with_fewer_ctas_than_problems_is_an_error():
    """ctas < problems per launch is rejected with SVM_EINVAL (it used to divide by zero
    in the planner)."""
    import torch
    import paper_2311_14908_b200 as S
    X, labels = W.pavia_like(10, seed=3)
    probs = []
    for c in range(4):
        sel = (labels == c) | (labels == c + 1)
        yy = np.where(labels[sel] == c, 1, -1).astype(np.int8)
        probs.append((torch.from_numpy(np.ascontiguousarray(X[sel])).cuda(), torch.from_numpy(yy).cuda()))
    with pytest.raises(S.SvmError, match="EINVAL"):
        S.svm_train_batch_dev(probs, 1.0, S.RBF, 0.01, ctas=2)
    out = S.svm_train_batch_dev(probs, 1.0, S.RBF, 0.01, ctas=4)      # one CTA each: fine
    assert len(out) == 4 and all(o["info"]["converged"] for o in out)
