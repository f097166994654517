"""ctypes wrapper of the fp64 CPU oracle (oracle/smo_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference leg.  The product package never imports this module.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "smo_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

LINEAR = 0
RBF = 1


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (plain C, OpenMP, no fast-math, no contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fopenmp", "-fno-fast-math",
               "-ffp-contract=off", "-fno-builtin", "-o", _LIB + ".tmp", _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB)
            P = ctypes.c_void_p
            i64, f64, i32 = ctypes.c_int64, ctypes.c_double, ctypes.c_int
            L.oracle_exp_cr.argtypes = [f64]
            L.oracle_exp_cr.restype = f64
            L.oracle_exp_ambiguous_count.restype = ctypes.c_long
            L.oracle_kernel.argtypes = [i32, f64, P, P, i64, i32]
            L.oracle_kernel.restype = f64
            L.oracle_kernel_row.argtypes = [i32, f64, P, i64, i64, i64, P]
            L.oracle_select.argtypes = [P, P, P, f64, i64, P, P, P, P]
            L.oracle_select.restype = i32
            L.oracle_svm_train.argtypes = [P, P, i64, i64, f64, i32, f64, f64, i64, P, P,
                                           P, P, P, P, P, P, P, P, i64]
            L.oracle_svm_train.restype = i32
            L.oracle_svm_train_wss.argtypes = L.oracle_svm_train.argtypes + [i32]
            L.oracle_svm_train_wss.restype = i32
            L.oracle_svm_train_full.argtypes = L.oracle_svm_train.argtypes + [i32, i64]
            L.oracle_svm_train_full.restype = i32
            L.oracle_select_second_order.argtypes = [P, P, P, P, f64, i64, i64, i32, f64, i64]
            L.oracle_select_second_order.restype = i64
            L.oracle_decision.argtypes = [P, P, i64, i64, f64, i32, f64, P, i64, P]
            L.oracle_dual_objective.argtypes = [P, P, P, i64, i64, i32, f64]
            L.oracle_dual_objective.restype = f64
            L.oracle_num_threads.restype = i32
            L.oracle_gd_train.argtypes = [P, P, i64, i64, f64, i32, f64, f64, i64, P, P, P, P]
            L.oracle_gd_train.restype = i32
            _lib = L
    return _lib


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _f32(X):
    return np.ascontiguousarray(X, dtype=np.float32)


def exp_cr(x: float) -> float:
    return lib().oracle_exp_cr(float(x))


def exp_ambiguous_count() -> int:
    return lib().oracle_exp_ambiguous_count()


def num_threads() -> int:
    return lib().oracle_num_threads()


def kernel(a, b, kernel: int, gamma: float = 0.0, same: bool = False) -> float:
    a = _f32(np.atleast_1d(a)); b = _f32(np.atleast_1d(b))
    assert a.shape == b.shape
    return lib().oracle_kernel(kernel, gamma, _p(a), _p(b), a.size, int(same))


def kernel_row(X, i: int, kernel: int, gamma: float = 0.0) -> np.ndarray:
    X = _f32(X)
    out = np.empty(X.shape[0])
    lib().oracle_kernel_row(kernel, gamma, _p(X), X.shape[0], X.shape[1], i, _p(out))
    return out


def select(f, y, alpha, C):
    f = np.ascontiguousarray(f, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.int8)
    alpha = np.ascontiguousarray(alpha, dtype=np.float64)
    iu, il = ctypes.c_int64(), ctypes.c_int64()
    bu, bl = ctypes.c_double(), ctypes.c_double()
    ok = lib().oracle_select(_p(f), _p(y), _p(alpha), C, f.size, ctypes.byref(iu),
                             ctypes.byref(il), ctypes.byref(bu), ctypes.byref(bl))
    return bool(ok), iu.value, il.value, bu.value, bl.value


class TrainResult(dict):
    __getattr__ = dict.__getitem__


def train(X, y, C: float, kernel: int, gamma: float = 0.0, tol: float = 1e-3,
          max_iter: int = 0, alpha0=None, f0=None, trace_cap: int = 0, wss: int = 1,
          shrink: int = 0) -> TrainResult:
    """The oracle SMO solve (smo_oracle.c).  wss: 1 maximal violating pair (reading R1,
    default), 2 second-order selection of the second index (Fan et al.).
    shrink: window length H of window shrinking (reading R29), 0 = off."""
    X = _f32(X)
    y = np.ascontiguousarray(y, dtype=np.int8)
    n, d = X.shape
    alpha = np.empty(n)
    f = np.empty(n)
    a0 = None if alpha0 is None else np.ascontiguousarray(alpha0, dtype=np.float64)
    g0 = None if f0 is None else np.ascontiguousarray(f0, dtype=np.float64)
    trace = np.full((max(trace_cap, 0), 2), -1, dtype=np.int64) if trace_cap > 0 else None
    b, it = ctypes.c_double(), ctypes.c_int64()
    conv = ctypes.c_int()
    bu, bl = ctypes.c_double(), ctypes.c_double()
    rc = lib().oracle_svm_train_full(_p(X), _p(y), n, d, float(C), int(kernel), float(gamma),
                                     float(tol), int(max_iter), _p(a0), _p(g0), _p(alpha), _p(f),
                                     ctypes.byref(b), ctypes.byref(it), ctypes.byref(conv),
                                     ctypes.byref(bu), ctypes.byref(bl), _p(trace),
                                     trace_cap if trace_cap > 0 else 0, int(wss), int(shrink))
    if rc != 0:
        raise ValueError(f"oracle_svm_train failed with status {rc}")
    res = TrainResult(alpha=alpha, f=f, b=b.value, iterations=it.value,
                      converged=bool(conv.value), b_up=bu.value, b_low=bl.value)
    if trace is not None:
        res["trace"] = trace[:min(it.value, trace_cap)]
    return res


def decision(X_sv, coef, b: float, kernel: int, gamma: float, X_test) -> np.ndarray:
    X_sv = _f32(X_sv).reshape(-1, np.shape(X_test)[1]) if np.size(X_sv) else \
        np.zeros((0, np.shape(X_test)[1]), dtype=np.float32)
    X_test = _f32(X_test)
    coef = np.ascontiguousarray(coef, dtype=np.float64)
    out = np.empty(X_test.shape[0])
    lib().oracle_decision(_p(X_sv), _p(coef), coef.size, X_test.shape[1], float(b), kernel,
                          float(gamma), _p(X_test), X_test.shape[0], _p(out))
    return out


def dual_objective(X, y, alpha, kernel: int, gamma: float = 0.0) -> float:
    X = _f32(X)
    y = np.ascontiguousarray(y, dtype=np.int8)
    alpha = np.ascontiguousarray(alpha, dtype=np.float64)
    return lib().oracle_dual_objective(_p(X), _p(y), _p(alpha), X.shape[0], X.shape[1],
                                       kernel, float(gamma))


def dual_objective_from_f(alpha, y, f) -> float:
    """W = 1/2 sum_i alpha_i (1 - y_i f_i)  (identity from the f definition)."""
    return 0.5 * float(np.sum(np.asarray(alpha) * (1.0 - np.asarray(y, dtype=np.float64) * np.asarray(f))))


class GdResult:
    def __init__(self, alpha, g, b, W):
        self.alpha, self.g, self.b, self.W = alpha, g, b, W


def gd_train(X, y, C: float, kernel: int, gamma: float, lr: float, epochs: int) -> GdResult:
    """Projected-gradient dual trainer (oracle_gd_train): alpha after `epochs` epochs,
    g = K (alpha o y) of the final alpha, bias b (R25) and W(alpha)."""
    X = _f32(X)
    y = np.ascontiguousarray(y, dtype=np.int8)
    n, d = X.shape
    alpha = np.zeros(n)
    g = np.zeros(n)
    b = ctypes.c_double()
    W = ctypes.c_double()
    rc = lib().oracle_gd_train(_p(X), _p(y), n, d, float(C), int(kernel), float(gamma), float(lr),
                               int(epochs), _p(alpha), _p(g), ctypes.byref(b), ctypes.byref(W))
    if rc:
        raise MemoryError("oracle_gd_train: allocation failed")
    return GdResult(alpha, g, b.value, W.value)

