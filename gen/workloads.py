"""Seeded synthetic workloads W1-W5, shared by the oracle side and
the CUDA side.

This module holds NO arithmetic of the method (no kernel values, no SMO steps): it
only draws feature matrices X (float32, row-major n x d) and labels y (int8 in
{+1, -1}) with numpy's PCG64 generator.  Both the oracle (`oracle/`) and the CUDA
path (`paper_2311_14908_b200/`) read the identical bytes it returns.

The paper trains on Pavia Centre / Iris / Breast Cancer (Table 1)
which are not available offline; BASELINE.json `configs` name five synthetic
stand-ins, whose recipes are stated in DESIGN.md ("Input recipe"):

  W1  2-D two-Gaussian, n=200           linear, C=1,   tol=1e-3   (configs[0])
  W2  Adult-like, n=32,561, d=123        RBF g=0.5,  C=100          (configs[1])
  W3  MNIST-like even/odd, n=60,000 d=784 RBF g=0.0125, C=10        (configs[2])
  W4  covtype-like, n=581,012, d=54      RBF g=1/54, C=1            (configs[3])
  W5  scaling, n=1,000,000, d=256        RBF g=1/256, C=1           (configs[4])

Every generator takes `n` so tests can draw small instances of the same law.
"""
from __future__ import annotations

import dataclasses
from typing import Callable, Dict, Optional, Tuple

import numpy as np

LINEAR = 0
RBF = 1


@dataclasses.dataclass(frozen=True)
class Workload:
    name: str
    config: str          # the BASELINE.json configs[] entry it stands for
    n: int
    d: int
    kernel: int
    gamma: float
    C: float
    tol: float
    seed_train: int
    seed_test: int
    n_test: int
    make: Callable[[int, int], Tuple[np.ndarray, np.ndarray]]  # (n, seed) -> X, y

    def train(self, n: Optional[int] = None) -> Tuple[np.ndarray, np.ndarray]:
        return self.make(self.n if n is None else n, self.seed_train)

    def test(self, m: Optional[int] = None) -> Tuple[np.ndarray, np.ndarray]:
        return self.make(self.n_test if m is None else m, self.seed_test)

    def params(self) -> dict:
        return dict(kernel=self.kernel, gamma=self.gamma, C=self.C, tol=self.tol)


def _rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def _finish(X: np.ndarray, y: np.ndarray) -> Tuple[np.ndarray, np.ndarray]:
    X = np.ascontiguousarray(X, dtype=np.float32)
    y = np.ascontiguousarray(y, dtype=np.int8)
    assert X.ndim == 2 and y.shape == (X.shape[0],)
    assert np.all(np.isfinite(X))
    return X, y


# --------------------------------------------------------------------------- W1
def gaussian_blobs(n: int, seed: int, d: int = 2, m: int = 2,
                   separation: float = 3.0) -> Tuple[np.ndarray, np.ndarray]:
    """SPEC.md L75-83 `generate_synthetic`: unit-variance Gaussian blobs whose centers
    are at pairwise distance >= separation (seeded random directions, rejection).
    Class 0 -> +1, every other class -> -1 (binary use).  Rows are shuffled.
    Returns class ids in y when m > 2 (int8 in [0, m))."""
    rng = _rng(seed)
    # the class centers are part of the law (shared by train and test draws), so they
    # come from a generator fixed by (m, d, separation), not by the sample seed
    law = _rng(9000 + 97 * m + d + int(1000 * separation))
    while True:
        centers = law.standard_normal((m, d)) * separation
        if m == 2:
            u = law.standard_normal(d)
            u /= np.linalg.norm(u)
            centers = np.stack([0.5 * separation * u, -0.5 * separation * u])
        dist = np.linalg.norm(centers[:, None, :] - centers[None, :, :], axis=-1)
        if np.all(dist[np.triu_indices(m, 1)] >= separation * (1 - 1e-12)):
            break
    cls = np.arange(n) % m
    rng.shuffle(cls)
    X = centers[cls] + rng.standard_normal((n, d))
    if m == 2:
        y = np.where(cls == 0, 1, -1)
    else:
        y = cls
    return _finish(X, y)


# --------------------------------------------------------------------------- W2
ADULT_GROUPS = (5, 8, 5, 16, 5, 7, 14, 6, 5, 2, 2, 2, 5, 41)  # sums to 123 (a9a layout)


def adult_like(n: int, seed: int) -> Tuple[np.ndarray, np.ndarray]:
    """Adult-like (a9a-style) binary one-hot data: 14 categorical groups, exactly one
    active column per group (so every row has 14 ones, d = 123, values exactly 0/1).
    Skewed per-group categoricals (Dirichlet(0.6)); label from a latent logistic
    score, thresholded to ~24% positives."""
    rng = _rng(seed)
    # the law (probabilities and label weights) is fixed by a constant seed so that
    # train and test sets of different seeds share it
    law = _rng(12345)
    probs = [law.dirichlet(np.full(g, 0.6)) for g in ADULT_GROUPS]
    weights = [law.standard_normal(g) * 1.2 for g in ADULT_GROUPS]
    d = sum(ADULT_GROUPS)
    X = np.zeros((n, d), dtype=np.float32)
    score = np.zeros(n)
    off = 0
    for g, p, w in zip(ADULT_GROUPS, probs, weights):
        c = rng.choice(g, size=n, p=p)
        X[np.arange(n), off + c] = 1.0
        score += w[c]
        off += g
    score += rng.logistic(size=n)
    thr = _law_quantile(lambda k: _adult_score_sample(probs, weights, k), 0.76)
    y = np.where(score > thr, 1, -1)
    return _finish(X, y)


def _adult_score_sample(probs, weights, k):
    r = _rng(999)
    s = np.zeros(k)
    for g, p, w in zip(ADULT_GROUPS, probs, weights):
        s += w[r.choice(g, size=k, p=p)]
    return s + r.logistic(size=k)


_QCACHE: Dict[str, float] = {}


def _law_quantile(sampler, q: float) -> float:
    key = f"{sampler.__code__.co_name}:{q}"
    if key not in _QCACHE:
        _QCACHE[key] = float(np.quantile(sampler(200_000), q))
    return _QCACHE[key]


# --------------------------------------------------------------------------- W3
def _digit_prototypes() -> np.ndarray:
    """10 smooth 28x28 stroke images (sums of Gaussian blobs along random polylines)."""
    law = _rng(2718)
    yy, xx = np.mgrid[0:28, 0:28].astype(np.float64)
    protos = np.zeros((10, 28, 28))
    for c in range(10):
        pts = law.uniform(6, 22, size=(5, 2))
        img = np.zeros((28, 28))
        for a, b in zip(pts[:-1], pts[1:]):
            for t in np.linspace(0, 1, 12):
                cy, cx = a * (1 - t) + b * t
                img += np.exp(-((yy - cy) ** 2 + (xx - cx) ** 2) / (2 * 1.3 ** 2))
        protos[c] = np.clip(img / img.max() * 2.0, 0, 1)
    return protos


def mnist_like(n: int, seed: int) -> Tuple[np.ndarray, np.ndarray]:
    """MNIST-like even-vs-odd: a random prototype digit per sample, shifted by up to
    +-2 pixels, intensity-jittered, plus noise; clipped to [0,1], small values zeroed,
    quantised to k/255 and stored as float32 (d = 784).  Even digit -> +1."""
    rng = _rng(seed)
    protos = _digit_prototypes()
    cls = rng.integers(0, 10, size=n)
    X = np.empty((n, 784), dtype=np.float32)
    chunk = 8192
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        k = e - s
        img = protos[cls[s:e]]
        sh = rng.integers(-2, 3, size=(k, 2))
        out = np.empty_like(img)
        for dy in range(-2, 3):
            for dx in range(-2, 3):
                sel = (sh[:, 0] == dy) & (sh[:, 1] == dx)
                if sel.any():
                    out[sel] = np.roll(np.roll(img[sel], dy, axis=1), dx, axis=2)
        out *= rng.uniform(0.7, 1.0, size=(k, 1, 1))
        out += rng.normal(0.0, 0.12, size=out.shape)
        out = np.clip(out, 0.0, 1.0)
        out[out < 0.2] = 0.0
        X[s:e] = (np.round(out.reshape(k, 784) * 255.0) / 255.0).astype(np.float32)
    y = np.where(cls % 2 == 0, 1, -1)
    return _finish(X, y)


# --------------------------------------------------------------------------- W4
def covtype_like(n: int, seed: int) -> Tuple[np.ndarray, np.ndarray]:
    """covtype-like: 10 continuous features in [0,1] (correlated Beta-ish), a 4-way
    one-hot (wilderness area) and a 40-way one-hot (soil type, skewed), d = 54.
    Label: a nonlinear score plus noise thresholded at ~48.8% positives."""
    rng = _rng(seed)
    law = _rng(31415)
    mix = law.standard_normal((10, 10)) * 0.4 + np.eye(10)
    p_w = law.dirichlet(np.full(4, 2.0))
    p_s = law.dirichlet(np.full(40, 0.4))
    eff_w = law.standard_normal(4)
    eff_s = law.standard_normal(40) * 0.8
    freq = law.uniform(1.0, 4.0, size=10)
    wts = law.standard_normal(10)

    def draw(r, k):
        z = r.standard_normal((k, 10)) @ mix.T
        cont = 1.0 / (1.0 + np.exp(-z))
        w = r.choice(4, size=k, p=p_w)
        s = r.choice(40, size=k, p=p_s)
        score = (np.sin(cont * freq) @ wts + 1.5 * cont[:, 0] * cont[:, 1]
                 - cont[:, 2] ** 2 + eff_w[w] + eff_s[s] + 0.5 * r.standard_normal(k))
        return cont, w, s, score

    cont, w, s, score = draw(rng, n)
    thr = _law_quantile(lambda k: draw(_rng(777), k)[3], 1.0 - 0.488)
    X = np.zeros((n, 54), dtype=np.float32)
    X[:, :10] = cont
    X[np.arange(n), 10 + w] = 1.0
    X[np.arange(n), 14 + s] = 1.0
    y = np.where(score > thr, 1, -1)
    return _finish(X, y)


# --------------------------------------------------------------------------- W5
def two_gaussians_256(n: int, seed: int, d: int = 256,
                      delta: float = 2.563) -> Tuple[np.ndarray, np.ndarray]:
    """Scaling law: x ~ N(+-(delta/2) u, I_d), random unit u (fixed law), balanced
    labels; delta = 2.563 gives a 10% Bayes error."""
    rng = _rng(seed)
    u = _rng(4242).standard_normal(d)
    u /= np.linalg.norm(u)
    y = np.where(rng.random(n) < 0.5, 1, -1).astype(np.int8)
    X = np.empty((n, d), dtype=np.float32)
    chunk = 1 << 16
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        X[s:e] = (rng.standard_normal((e - s, d), dtype=np.float32)
                  + (0.5 * delta * u)[None, :].astype(np.float32) * y[s:e, None])
    return _finish(X, y)


def pavia_like(k_per_class: int, seed: int, m: int = 9, d: int = 102,
               separation: float = 4.0) -> Tuple[np.ndarray, np.ndarray]:
    """Pavia-Centre stand-in (Table 1: 9 classes, 102 bands):
    multiclass blobs, class ids 0..m-1 in y."""
    return gaussian_blobs(k_per_class * m, seed, d=d, m=m, separation=separation)


WORKLOADS: Dict[str, Workload] = {
    "W1": Workload("W1", "2-D two-Gaussian synthetic, n=200, linear kernel, C=1, tol=1e-3",
                   200, 2, LINEAR, 0.0, 1.0, 1e-3, 0, 100, 200,
                   lambda n, s: gaussian_blobs(n, s, d=2, m=2, separation=3.0)),
    "W2": Workload("W2", "Adult-like binary: n=32,561, d=123 sparse-binary densified, RBF gamma=0.5, C=100",
                   32561, 123, RBF, 0.5, 100.0, 1e-3, 1, 101, 16281, adult_like),
    "W3": Workload("W3", "MNIST-like even-vs-odd: n=60,000, d=784, RBF gamma=0.0125, C=10",
                   60000, 784, RBF, 0.0125, 10.0, 1e-3, 2, 102, 10000, mnist_like),
    "W4": Workload("W4", "covtype-like binary: n=581,012, d=54, RBF gamma=1/54, C=1",
                   581012, 54, RBF, 1.0 / 54.0, 1.0, 1e-3, 3, 103, 10000, covtype_like),
    "W5": Workload("W5", "scaling sweep: synthetic n=1M, d=256, RBF, C=1",
                   1_000_000, 256, RBF, 1.0 / 256.0, 1.0, 1e-3, 4, 5, 1_000_000,
                   two_gaussians_256),
}


def get(name: str) -> Workload:
    return WORKLOADS[name]
