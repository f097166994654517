"""paper_2311_14908_b200 -- B200-native SMO SVM solver (arXiv 2311.14908 hot path).

Thin ctypes binding of libsvmb200.so (C ABI: include/svmb200.h).  Argument marshalling
only: every step of the solve and of prediction runs in the library's sm_100a kernels.
There is no CPU fallback: importing the binding without the built library raises.

Names follow the C ABI: svm_train, svm_train_ex, svm_train_dev, svm_predict,
svm_predict_dev, svm_comm_unique_id, svm_comm_init, svm_train_shard, svm_comm_destroy.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

__all__ = ["LINEAR", "RBF", "PREDICT_EXACT", "PREDICT_TENSOR", "SvmError", "lib", "svm_train", "svm_train_ex", "svm_train_dev",
           "svm_predict", "svm_predict_dev", "svm_train_batch_dev", "svm_comm_unique_id", "svm_comm_init",
           "svm_train_shard", "svm_comm_destroy", "svm_train_gd_dev", "Params", "Info", "version"]

LINEAR = 0
RBF = 1
_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libsvmb200.so")

STATUS = {0: "SVM_OK", -1: "SVM_EINVAL", -2: "SVM_ELABEL", -3: "SVM_ESINGLECLASS",
          -4: "SVM_ENONFINITE", -5: "SVM_ENOMEM", -6: "SVM_ECUDA", -7: "SVM_ENCCL",
          -8: "SVM_ETIMEOUT"}


class SvmError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


class Params(ctypes.Structure):
    _fields_ = [("C", ctypes.c_double), ("gamma", ctypes.c_double), ("tol", ctypes.c_double),
                ("max_iter", ctypes.c_int64), ("check_interval", ctypes.c_int32),
                ("kernel", ctypes.c_int32), ("sv_epsilon", ctypes.c_double),
                ("virtual_ranks", ctypes.c_int32), ("ctas", ctypes.c_int32),
                ("iters_per_launch", ctypes.c_int64), ("gram", ctypes.c_int32), ("cache_rows", ctypes.c_int32),
                ("cluster", ctypes.c_int32), ("reserved0", ctypes.c_int32)]


class Info(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int64), ("converged", ctypes.c_int32),
                ("n_sv", ctypes.c_int32), ("gap", ctypes.c_double), ("b_up", ctypes.c_double),
                ("b_low", ctypes.c_double), ("dual_objective", ctypes.c_double),
                ("seconds_solve", ctypes.c_double), ("seconds_total", ctypes.c_double),
                ("launches", ctypes.c_int64)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


class Debug(ctypes.Structure):
    _fields_ = [("alpha0", ctypes.c_void_p), ("f0", ctypes.c_void_p), ("f_out", ctypes.c_void_p),
                ("pair_trace", ctypes.c_void_p), ("pair_trace_cap", ctypes.c_int64)]


_lib = None


def lib():
    """Load libsvmb200.so; fails loudly if it was not built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(LIB_PATH)
        P, i64, f64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_int
        L.svm_train.argtypes = [P, P, i64, i64, f64, i32, f64, f64, P, P]
        L.svm_train_ex.argtypes = [P, P, i64, i64, P, P, P, P, P]
        L.svm_train_dev.argtypes = [P, P, i64, i64, P, P, P, P, P, P]
        L.svm_predict.argtypes = [P, P, i64, i64, f64, i32, f64, P, i64, P]
        L.svm_predict_dev.argtypes = [P, P, i64, i64, f64, i32, f64, P, i64, P, P]
        L.svm_predict_ex.argtypes = [P, P, i64, i64, f64, i32, f64, P, i64, P, i32]
        L.svm_predict_dev_ex.argtypes = [P, P, i64, i64, f64, i32, f64, P, i64, P, i32, P]
        L.svm_train_batch_dev.argtypes = [i32, P, P, P, i64, P, P, P, P, P]
        L.svm_comm_unique_id.argtypes = [P]
        L.svm_comm_init.argtypes = [ctypes.POINTER(ctypes.c_void_p), i32, i32, P, i32]
        L.svm_train_shard.argtypes = [P, P, P, i64, i64, i64, i64, P, P, P, P, P]
        L.svm_train_gd_dev.argtypes = [P, P, i64, i64, f64, i32, f64, f64, i64, P, P, P, P]
        L.svm_comm_destroy.argtypes = [P]
        L.svm_comm_destroy.restype = None
        L.svm_last_error.restype = ctypes.c_char_p
        L.svm_kernel_launches.restype = ctypes.c_int64
        L.svm_last_plan.restype = ctypes.c_char_p
        L.svm_version.restype = ctypes.c_char_p
        for name in ("svm_train", "svm_train_ex", "svm_train_dev", "svm_predict", "svm_predict_dev",
                     "svm_predict_ex", "svm_predict_dev_ex", "svm_train_batch_dev",
                     "svm_comm_unique_id", "svm_comm_init", "svm_train_shard", "svm_train_gd_dev"):
            getattr(L, name).restype = ctypes.c_int
        _lib = L
    return _lib


def kernel_launches() -> int:
    """CUDA kernels the library launched from this thread so far."""
    return int(lib().svm_kernel_launches())


def last_plan() -> dict:
    """How the last solve on this thread ran (kernel, CTAs, cluster, mode) -- svm_last_plan."""
    import json
    txt = lib().svm_last_plan().decode()
    return json.loads(txt) if txt else {}


def version() -> str:
    return lib().svm_version().decode()


def _check(rc: int):
    if rc != 0:
        raise SvmError(rc, lib().svm_last_error().decode())


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def make_params(C: float, kernel: int, gamma: float = 0.0, tol: float = 1e-3, **kw) -> Params:
    p = Params()
    p.C, p.kernel, p.gamma, p.tol = float(C), int(kernel), float(gamma), float(tol)
    for k, v in kw.items():
        setattr(p, k, v)
    return p


def svm_train(X, y, C: float, kernel: int, gamma: float = 0.0, tol: float = 1e-3):
    """Host arrays -> (alpha [n] fp64, b)."""
    X = np.ascontiguousarray(X, dtype=np.float32)
    y = np.ascontiguousarray(y, dtype=np.int8)
    n, d = X.shape
    alpha = np.empty(n)
    b = ctypes.c_double()
    _check(lib().svm_train(_ptr(X), _ptr(y), n, d, float(C), int(kernel), float(gamma), float(tol),
                           _ptr(alpha), ctypes.byref(b)))
    return alpha, b.value


def svm_train_ex(X, y, C: float, kernel: int, gamma: float = 0.0, tol: float = 1e-3,
                 alpha0=None, f0=None, want_f: bool = False, trace_cap: int = 0, **params):
    """Host arrays with full controls.  Returns dict(alpha, b, info, [f], [trace])."""
    X = np.ascontiguousarray(X, dtype=np.float32)
    y = np.ascontiguousarray(y, dtype=np.int8)
    n, d = X.shape
    p = make_params(C, kernel, gamma, tol, **params)
    alpha = np.empty(n)
    b = ctypes.c_double()
    info = Info()
    dbg = Debug()
    keep = []
    if alpha0 is not None:
        a0 = np.ascontiguousarray(alpha0, dtype=np.float64); g0 = np.ascontiguousarray(f0, dtype=np.float64)
        keep += [a0, g0]
        dbg.alpha0, dbg.f0 = a0.ctypes.data, g0.ctypes.data
    f = np.empty(n) if want_f else None
    if f is not None:
        dbg.f_out = f.ctypes.data
    trace = np.full((trace_cap, 2), -1, dtype=np.int64) if trace_cap > 0 else None
    if trace is not None:
        dbg.pair_trace, dbg.pair_trace_cap = trace.ctypes.data, trace_cap
    _check(lib().svm_train_ex(_ptr(X), _ptr(y), n, d, ctypes.byref(p), _ptr(alpha), ctypes.byref(b),
                              ctypes.byref(info), ctypes.byref(dbg)))
    out = dict(alpha=alpha, b=b.value, info=info.as_dict())
    if f is not None:
        out["f"] = f
    if trace is not None:
        out["trace"] = trace[:min(info.iterations, trace_cap)]
    return out


def _stream_ptr(stream):
    if stream is None:
        import torch
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def svm_train_dev(X, y, C: float, kernel: int, gamma: float = 0.0, tol: float = 1e-3,
                  stream=None, trace_cap: int = 0, want_f: bool = False, **params):
    """torch CUDA tensors (X float32 [n, d] contiguous, y int8 [n]) -> dict(alpha tensor, b, info)."""
    import torch
    assert X.is_cuda and X.dtype == torch.float32 and X.is_contiguous()
    assert y.is_cuda and y.dtype == torch.int8 and y.is_contiguous()
    n, d = X.shape
    alpha = torch.empty(n, dtype=torch.float64, device=X.device)
    p = make_params(C, kernel, gamma, tol, **params)
    b = ctypes.c_double()
    info = Info()
    dbg = Debug()
    trace = np.full((trace_cap, 2), -1, dtype=np.int64) if trace_cap > 0 else None
    if trace is not None:
        dbg.pair_trace, dbg.pair_trace_cap = trace.ctypes.data, trace_cap
    f = np.empty(n) if want_f else None
    if f is not None:
        dbg.f_out = f.ctypes.data
    _check(lib().svm_train_dev(ctypes.c_void_p(X.data_ptr()), ctypes.c_void_p(y.data_ptr()), n, d,
                               ctypes.byref(p), ctypes.c_void_p(alpha.data_ptr()), ctypes.byref(b),
                               ctypes.byref(info), ctypes.byref(dbg), _stream_ptr(stream)))
    out = dict(alpha=alpha, b=b.value, info=info.as_dict())
    if trace is not None:
        out["trace"] = trace[:min(info.iterations, trace_cap)]
    if f is not None:
        out["f"] = f
    return out


class GdInfo(ctypes.Structure):
    _fields_ = [("objective", ctypes.c_double), ("seconds_gram", ctypes.c_double),
                ("seconds_epochs", ctypes.c_double), ("epochs", ctypes.c_int64),
                ("gram_bytes", ctypes.c_int64)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


def svm_train_gd_dev(X, y, C: float, kernel: int, gamma: float, lr: float, epochs: int, stream=None):
    """Projected-gradient dual trainer (C ABI svm_train_gd_dev): torch CUDA tensors
    (X float32 [n, d] contiguous, y int8 [n]) -> dict(alpha tensor, b, info)."""
    import torch
    assert X.is_cuda and X.dtype == torch.float32 and X.is_contiguous()
    assert y.is_cuda and y.dtype == torch.int8 and y.is_contiguous()
    n, d = X.shape
    alpha = torch.empty(n, dtype=torch.float64, device=X.device)
    b = ctypes.c_double()
    info = GdInfo()
    _check(lib().svm_train_gd_dev(ctypes.c_void_p(X.data_ptr()), ctypes.c_void_p(y.data_ptr()), n, d,
                                  float(C), int(kernel), float(gamma), float(lr), int(epochs),
                                  ctypes.c_void_p(alpha.data_ptr()), ctypes.byref(b), ctypes.byref(info),
                                  _stream_ptr(stream)))
    return dict(alpha=alpha, b=b.value, info=info.as_dict())


PREDICT_EXACT = 0
PREDICT_TENSOR = 1


def svm_predict(X_sv, coef, b: float, kernel: int, gamma: float, X_test,
                mode: int = PREDICT_EXACT) -> np.ndarray:
    """Host arrays -> decision values [m] fp64 (dec = K(X_test, SV) coef + b).
    mode PREDICT_EXACT (fp64 SIMT, bit-exact) or PREDICT_TENSOR (tcgen05 3xTF32)."""
    X_test = np.ascontiguousarray(X_test, dtype=np.float32)
    m, d = X_test.shape
    X_sv = np.ascontiguousarray(X_sv, dtype=np.float32).reshape(-1, d)
    coef = np.ascontiguousarray(coef, dtype=np.float64)
    assert coef.shape[0] == X_sv.shape[0]
    dec = np.empty(m)
    _check(lib().svm_predict_ex(_ptr(X_sv), _ptr(coef), coef.shape[0], d, float(b), int(kernel),
                                float(gamma), _ptr(X_test), m, _ptr(dec), int(mode)))
    return dec


def svm_predict_dev(X_sv, coef, b: float, kernel: int, gamma: float, X_test, stream=None,
                    mode: int = PREDICT_EXACT):
    """torch CUDA tensors -> decision values tensor [m] fp64."""
    import torch
    m, d = X_test.shape
    dec = torch.empty(m, dtype=torch.float64, device=X_test.device)
    _check(lib().svm_predict_dev_ex(ctypes.c_void_p(X_sv.data_ptr()), ctypes.c_void_p(coef.data_ptr()),
                                    coef.shape[0], d, float(b), int(kernel), float(gamma),
                                    ctypes.c_void_p(X_test.data_ptr()), m,
                                    ctypes.c_void_p(dec.data_ptr()), int(mode), _stream_ptr(stream)))
    return dec


def svm_train_batch_dev(problems, C: float, kernel: int, gamma: float = 0.0, tol: float = 1e-3,
                        stream=None, **params):
    """Independent binary problems solved concurrently (CTA groups of one persistent launch).
    problems: list of (X [n_k, d] float32 CUDA tensor, y [n_k] int8 CUDA tensor).
    Returns a list of dict(alpha tensor, b, info)."""
    import torch
    B = len(problems)
    d = problems[0][0].shape[1]
    alphas = [torch.empty(X.shape[0], dtype=torch.float64, device=X.device) for X, _ in problems]
    Xp = (ctypes.c_void_p * B)(*[X.data_ptr() for X, _ in problems])
    yp = (ctypes.c_void_p * B)(*[y.data_ptr() for _, y in problems])
    ap = (ctypes.c_void_p * B)(*[a.data_ptr() for a in alphas])
    ns = (ctypes.c_int64 * B)(*[X.shape[0] for X, _ in problems])
    bs = (ctypes.c_double * B)()
    infos = (Info * B)()
    p = make_params(C, kernel, gamma, tol, **params)
    for X, y in problems:
        assert X.is_cuda and X.dtype == torch.float32 and X.is_contiguous() and X.shape[1] == d
        assert y.is_cuda and y.dtype == torch.int8 and y.is_contiguous()
    _check(lib().svm_train_batch_dev(B, Xp, yp, ns, d, ctypes.byref(p), ap, bs, infos, _stream_ptr(stream)))
    return [dict(alpha=alphas[k], b=bs[k], info=infos[k].as_dict()) for k in range(B)]


def svm_comm_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    _check(lib().svm_comm_unique_id(buf))
    return bytes(buf)


def svm_comm_init(rank: int, world: int, uid: bytes, device: int):
    buf = (ctypes.c_uint8 * 128).from_buffer_copy(uid)
    h = ctypes.c_void_p()
    _check(lib().svm_comm_init(ctypes.byref(h), rank, world, buf, device))
    return h


def svm_comm_destroy(comm) -> None:
    lib().svm_comm_destroy(comm)


def svm_train_shard(comm, X_local, y_local, row_offset: int, n_global: int, C: float, kernel: int,
                    gamma: float = 0.0, tol: float = 1e-3, stream=None, **params):
    """Row-sharded solve, one process per GPU.  X_local/y_local: this rank's torch CUDA
    rows.  Returns dict(alpha tensor [n_local], b, info)."""
    import torch
    n_local, d = X_local.shape
    alpha = torch.empty(max(n_local, 1), dtype=torch.float64, device=X_local.device)[:n_local]
    p = make_params(C, kernel, gamma, tol, **params)
    b = ctypes.c_double()
    info = Info()
    _check(lib().svm_train_shard(comm, ctypes.c_void_p(X_local.data_ptr()),
                                 ctypes.c_void_p(y_local.data_ptr()), n_local, row_offset, n_global,
                                 d, ctypes.byref(p), ctypes.c_void_p(alpha.data_ptr()),
                                 ctypes.byref(b), ctypes.byref(info), _stream_ptr(stream)))
    return dict(alpha=alpha, b=b.value, info=info.as_dict())


def shard_rows(n: int, world: int):
    """Contiguous row blocks: rank r owns [r*ceil(n/P), min(n, (r+1)*ceil(n/P)))."""
    per = -(-n // world)
    return [(min(n, r * per), min(n, (r + 1) * per)) for r in range(world)]
