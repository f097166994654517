"""One-against-one multiclass training and voting.

PAPER.md L134 (§3.1): "For m classes, there are m(m-1)/2 independent binary
classification problems"; L144 (§3.2, Fig. 4): "running multiple parallel binary SMOs
to implement a parallel multi-class SMO.  We distribute the number of parallel binary
SMOs among the MPI working nodes"; L412 (§4.2): MPI only transfers the input at the
beginning and the results at the end.  Conventions from SPEC.md L350-399: pairs (a, b),
a < b, in lexicographic order; +1 for the lower class id; a model votes for a when its
decision value is >= 0, else for b; ties in the vote count go to the lowest class id.

The B200 form: the binary problems of a batch run concurrently inside ONE persistent
launch (svm_train_batch_dev: the SMs are split into CTA groups, one per problem, each
with its own SMO loop and exchange).  With several GPUs, batches are dealt round-robin
to ranks and the models are gathered at the end -- no communication while training.
This module only orchestrates; every solve and every decision value runs in the CUDA
library.
"""
from __future__ import annotations

from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import (PREDICT_EXACT, PREDICT_TENSOR, svm_predict_dev, svm_train_batch_dev)

Pair = Tuple[int, int]


def enumerate_pairs(m: int) -> List[Pair]:
    """[(0,1), (0,2), ..., (m-2, m-1)], m(m-1)/2 of them."""
    if m < 2:
        raise ValueError("m >= 2 required")
    return [(a, b) for a in range(m) for b in range(a + 1, m)]


def binary_problem(labels: np.ndarray, pair: Pair):
    """the samples of the two classes in their original order, +1 for
    the lower class id."""
    a, b = pair
    idx = np.flatnonzero((labels == a) | (labels == b))
    if not (np.any(labels[idx] == a) and np.any(labels[idx] == b)):
        raise ValueError(f"pair {pair}: a class is missing")
    y = np.where(labels[idx] == a, 1, -1).astype(np.int8)
    return idx, y


class OvOModel:
    def __init__(self, m: int, kernel: int, gamma: float):
        self.m, self.kernel, self.gamma = m, kernel, gamma
        self.models: Dict[Pair, dict] = {}   # pair -> dict(sv_idx, coef, b, info)


def train_ovo(X, labels, m: int, C: float, kernel: int, gamma: float = 0.0, tol: float = 1e-3,
              batch: int = 8, rank: int = 0, world: int = 1, device=None, **params) -> OvOModel:
    """Train all m(m-1)/2 binary SVMs.  X: host float32 [n, d]; labels: host ints in [0, m).
    With world > 1 this rank trains batches k with k % world == rank (static round-robin,
    Fig. 4's node assignment) and the caller gathers the models (see gather_models)."""
    import torch
    device = device or torch.device("cuda", torch.cuda.current_device())
    labels = np.asarray(labels)
    pairs = enumerate_pairs(m)
    Xd = torch.from_numpy(np.ascontiguousarray(X, dtype=np.float32)).to(device)
    model = OvOModel(m, kernel, gamma)
    batches = [pairs[i:i + batch] for i in range(0, len(pairs), batch)]
    for k, bp in enumerate(batches):
        if k % world != rank:
            continue
        probs, idxs = [], []
        for pair in bp:
            idx, y = binary_problem(labels, pair)
            it = torch.from_numpy(idx).to(device)
            probs.append((Xd.index_select(0, it).contiguous(), torch.from_numpy(y).to(device)))
            idxs.append((idx, y))
        res = svm_train_batch_dev(probs, C, kernel, gamma, tol, **params)
        for pair, (idx, y), r in zip(bp, idxs, res):
            alpha = r["alpha"].cpu().numpy()
            sv = alpha > 1e-8
            model.models[pair] = dict(sv_idx=idx[sv], coef=(alpha * y)[sv], b=r["b"], info=r["info"],
                                      alpha=alpha)
    return model


def gather_models(model: OvOModel) -> OvOModel:
    """Collect every rank's models on every rank (torch.distributed, gloo or NCCL)."""
    import torch.distributed as dist
    parts: List[Optional[dict]] = [None] * dist.get_world_size()
    dist.all_gather_object(parts, model.models)
    for p in parts:
        model.models.update(p)
    return model


def decision_values(model: OvOModel, X, X_test, mode: int = PREDICT_EXACT, device=None) -> Dict[Pair, np.ndarray]:
    import torch
    device = device or torch.device("cuda", torch.cuda.current_device())
    Xd = torch.from_numpy(np.ascontiguousarray(X, dtype=np.float32)).to(device)
    Td = torch.from_numpy(np.ascontiguousarray(X_test, dtype=np.float32)).to(device)
    out = {}
    for pair in enumerate_pairs(model.m):
        mdl = model.models[pair]
        sv = torch.from_numpy(mdl["sv_idx"]).to(device)
        Xsv = Xd.index_select(0, sv).contiguous()
        coef = torch.from_numpy(np.ascontiguousarray(mdl["coef"])).to(device)
        out[pair] = svm_predict_dev(Xsv, coef, mdl["b"], model.kernel, model.gamma, Td, mode=mode).cpu().numpy()
    return out


def vote(decisions: Dict[Pair, np.ndarray], m: int) -> np.ndarray:
    """vote for a if dec >= 0 else b; argmax of counts, ties -> lowest id."""
    pairs = enumerate_pairs(m)
    n = len(next(iter(decisions.values())))
    votes = np.zeros((n, m), dtype=np.int64)
    for a, b in pairs:
        d = decisions[(a, b)]
        votes[np.arange(n), np.where(d >= 0, a, b)] += 1
    return np.argmax(votes, axis=1)   # argmax returns the first (lowest) maximal index


def predict_ovo(model: OvOModel, X, X_test, mode: int = PREDICT_EXACT) -> np.ndarray:
    return vote(decision_values(model, X, X_test, mode), model.m)
