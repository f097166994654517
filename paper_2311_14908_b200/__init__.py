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
           "svm_comm_init_host", "svm_train_shard", "svm_comm_destroy", "svm_train_gd_dev",
           "svm_support_vectors_dev", "Params", "Info", "version"]

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
                ("cluster", ctypes.c_int32), ("wss", ctypes.c_int32),
                ("shrink_window", ctypes.c_int32), ("reserved1", ctypes.c_int32)]


class Info(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int64), ("converged", ctypes.c_int32),
                ("n_sv", ctypes.c_int32), ("gap", ctypes.c_double), ("b_up", ctypes.c_double),
                ("b_low", ctypes.c_double), ("dual_objective", ctypes.c_double),
                ("seconds_solve", ctypes.c_double), ("seconds_total", ctypes.c_double),
                ("launches", ctypes.c_int64), ("cache_hits", ctypes.c_int64),
                ("cache_misses", ctypes.c_int64), ("seconds_h2d", ctypes.c_double)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


class Debug(ctypes.Structure):
    _fields_ = [("alpha0", ctypes.c_void_p), ("f0", ctypes.c_void_p), ("f_out", ctypes.c_void_p),
                ("pair_trace", ctypes.c_void_p), ("pair_trace_cap", ctypes.c_int64)]


_ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64)


class HostColl(ctypes.Structure):
    _fields_ = [("ctx", ctypes.c_void_p), ("allgather", _ALLGATHER_FN)]


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
        L.svm_train_shard.argtypes = [P, P, P, i64, i64, i64, i64, P, P, P, P, P, P]
        L.svm_comm_init_host.argtypes = [ctypes.POINTER(ctypes.c_void_p), i32, i32, i32, P]
        L.svm_support_vectors_dev.argtypes = [P, P, P, i64, i64, f64, P, P, P, P, P]
        L.svm_train_gd_dev.argtypes = [P, P, i64, i64, f64, i32, f64, f64, i64, P, P, P, P]
        L.svm_comm_destroy.argtypes = [P]
        L.svm_comm_destroy.restype = None
        L.svm_last_error.restype = ctypes.c_char_p
        L.svm_kernel_launches.restype = ctypes.c_int64
        L.svm_last_plan.restype = ctypes.c_char_p
        L.svm_version.restype = ctypes.c_char_p
        for name in ("svm_train", "svm_train_ex", "svm_train_dev", "svm_predict", "svm_predict_dev",
                     "svm_predict_ex", "svm_predict_dev_ex", "svm_train_batch_dev",
                     "svm_comm_unique_id", "svm_comm_init", "svm_comm_init_host", "svm_train_shard",
                     "svm_train_gd_dev", "svm_support_vectors_dev"):
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


def _gamma(gamma, kernel: int, d: int) -> float:
    """RBF width: the caller's, else 1/d (the C ABI has no default)."""
    if gamma is None:
        return 1.0 / d if int(kernel) == RBF else 0.0
    return float(gamma)


def make_params(C: float, kernel: int, gamma: float = 0.0, tol: float = 1e-3, **kw) -> Params:
    p = Params()
    p.C, p.kernel, p.gamma, p.tol = float(C), int(kernel), float(gamma), float(tol)
    for k, v in kw.items():
        setattr(p, k, v)
    return p


def svm_train(X, y, C: float, kernel: int, gamma: Optional[float] = None, tol: float = 1e-3):
    """Host arrays -> (alpha [n] fp64, b).  gamma None -> 1/d for RBF."""
    X = np.ascontiguousarray(X, dtype=np.float32)
    y = np.ascontiguousarray(y, dtype=np.int8)
    n, d = X.shape
    alpha = np.empty(n)
    b = ctypes.c_double()
    _check(lib().svm_train(_ptr(X), _ptr(y), n, d, float(C), int(kernel), _gamma(gamma, kernel, d), float(tol),
                           _ptr(alpha), ctypes.byref(b)))
    return alpha, b.value


def _warm(alpha0, f0, n: int):
    if (alpha0 is None) != (f0 is None):
        raise ValueError("a warm start needs both alpha0 and f0")
    if alpha0 is not None and (tuple(np.shape(alpha0)) != (n,) or tuple(np.shape(f0)) != (n,)):
        raise ValueError(f"alpha0 and f0 must have shape ({n},)")


def svm_train_ex(X, y, C: float, kernel: int, gamma: Optional[float] = None, tol: float = 1e-3,
                 alpha0=None, f0=None, want_f: bool = False, trace_cap: int = 0, **params):
    """Host arrays with full controls.  Returns dict(alpha, b, info, [f], [trace])."""
    X = np.ascontiguousarray(X, dtype=np.float32)
    y = np.ascontiguousarray(y, dtype=np.int8)
    n, d = X.shape
    if y.shape != (n,):
        raise ValueError("y must have shape (n,)")
    _warm(alpha0, f0, n)
    p = make_params(C, kernel, _gamma(gamma, kernel, d), tol, **params)
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


def _stream_ptr(stream, device=None):
    if stream is None:
        import torch
        stream = torch.cuda.current_stream(device)
    return ctypes.c_void_p(stream.cuda_stream)


def _dev(t, dtype, name: str, shape=None, device=None):
    """Check a torch tensor argument of a device entry point (dtype, CUDA, contiguity, shape)."""
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} must have shape {tuple(shape)}, got {tuple(t.shape)}")
    if device is not None and t.device != device:
        raise ValueError(f"{name} is on {t.device}, expected {device}")
    return ctypes.c_void_p(t.data_ptr())


def _dev_debug(n: int, device, alpha0, f0, want_f: bool, trace_cap: int):
    """svm_debug of a device entry point: alpha0 / f0 / f_out device tensors, trace host."""
    import torch
    _warm(alpha0, f0, n)
    dbg = Debug()
    keep = {}
    if alpha0 is not None:
        dbg.alpha0 = _dev(alpha0, torch.float64, "alpha0", (n,), device).value
        dbg.f0 = _dev(f0, torch.float64, "f0", (n,), device).value
    if want_f:
        keep["f"] = torch.empty(max(n, 1), dtype=torch.float64, device=device)[:n]
        dbg.f_out = keep["f"].data_ptr()
    if trace_cap > 0:
        keep["trace"] = np.full((trace_cap, 2), -1, dtype=np.int64)
        dbg.pair_trace, dbg.pair_trace_cap = keep["trace"].ctypes.data, trace_cap
    return dbg, keep


def svm_train_dev(X, y, C: float, kernel: int, gamma: Optional[float] = None, tol: float = 1e-3,
                  stream=None, trace_cap: int = 0, want_f: bool = False, alpha0=None, f0=None, **params):
    """torch CUDA tensors (X float32 [n, d] contiguous, y int8 [n]) -> dict(alpha tensor, b, info,
    [f tensor], [trace]).  alpha0 / f0: optional warm start (float64 CUDA tensors [n])."""
    import torch
    n, d = X.shape
    xp = _dev(X, torch.float32, "X")
    yp = _dev(y, torch.int8, "y", (n,), X.device)
    alpha = torch.empty(n, dtype=torch.float64, device=X.device)
    p = make_params(C, kernel, _gamma(gamma, kernel, d), tol, **params)
    b = ctypes.c_double()
    info = Info()
    dbg, keep = _dev_debug(n, X.device, alpha0, f0, want_f, trace_cap)
    _check(lib().svm_train_dev(xp, yp, n, d, ctypes.byref(p), ctypes.c_void_p(alpha.data_ptr()), ctypes.byref(b),
                               ctypes.byref(info), ctypes.byref(dbg), _stream_ptr(stream, X.device)))
    out = dict(alpha=alpha, b=b.value, info=info.as_dict())
    if "trace" in keep:
        out["trace"] = keep["trace"][:min(info.iterations, trace_cap)]
    if "f" in keep:
        out["f"] = keep["f"]
    return out


def svm_support_vectors_dev(X, y, alpha, sv_epsilon: float = 1e-8, stream=None, want_index: bool = False):
    """The support set {i : alpha_i > sv_epsilon} in ascending i, compacted on the device
    (C ABI svm_support_vectors_dev): returns (X_sv float32 [n_sv, d], coef = alpha * y
    float64 [n_sv], index int64 [n_sv] or None)."""
    import torch
    n, d = X.shape
    xp = _dev(X, torch.float32, "X")
    yp = _dev(y, torch.int8, "y", (n,), X.device)
    ap = _dev(alpha, torch.float64, "alpha", (n,), X.device)
    st = _stream_ptr(stream, X.device)
    nsv = ctypes.c_int64()
    _check(lib().svm_support_vectors_dev(xp, yp, ap, n, d, float(sv_epsilon), None, None, None, ctypes.byref(nsv), st))
    k = nsv.value
    Xsv = torch.empty((max(k, 1), d), dtype=torch.float32, device=X.device)[:k]
    coef = torch.empty(max(k, 1), dtype=torch.float64, device=X.device)[:k]
    idx = torch.empty(max(k, 1), dtype=torch.int64, device=X.device)[:k] if want_index else None
    _check(lib().svm_support_vectors_dev(xp, yp, ap, n, d, float(sv_epsilon), ctypes.c_void_p(Xsv.data_ptr()),
                                         ctypes.c_void_p(coef.data_ptr()),
                                         ctypes.c_void_p(idx.data_ptr()) if idx is not None else None,
                                         ctypes.byref(nsv), st))
    assert nsv.value == k
    return Xsv, coef, idx


class GdInfo(ctypes.Structure):
    _fields_ = [("objective", ctypes.c_double), ("seconds_gram", ctypes.c_double),
                ("seconds_epochs", ctypes.c_double), ("epochs", ctypes.c_int64),
                ("gram_bytes", ctypes.c_int64)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


def svm_train_gd_dev(X, y, C: float, kernel: int, gamma: Optional[float], lr: float, epochs: int, stream=None):
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
                                  float(C), int(kernel), _gamma(gamma, kernel, d), float(lr), int(epochs),
                                  ctypes.c_void_p(alpha.data_ptr()), ctypes.byref(b), ctypes.byref(info),
                                  _stream_ptr(stream)))
    return dict(alpha=alpha, b=b.value, info=info.as_dict())


PREDICT_EXACT = 0
PREDICT_TENSOR = 1


def svm_predict(X_sv, coef, b: float, kernel: int, gamma: Optional[float], X_test,
                mode: int = PREDICT_EXACT) -> np.ndarray:
    """Host arrays -> decision values [m] fp64 (dec = K(X_test, SV) coef + b).
    mode PREDICT_EXACT (fp64 SIMT, bit-exact) or PREDICT_TENSOR (tcgen05 3xTF32).
    X_sv [n_sv, d] must match X_test's d (dimension mismatch is an error)."""
    X_test = np.ascontiguousarray(X_test, dtype=np.float32)
    if X_test.ndim != 2:
        raise ValueError("X_test must be 2-D")
    m, d = X_test.shape
    X_sv = np.ascontiguousarray(X_sv, dtype=np.float32)
    if X_sv.size == 0:
        X_sv = X_sv.reshape(0, d)
    if X_sv.ndim != 2 or X_sv.shape[1] != d:
        raise ValueError(f"X_sv must have shape (n_sv, {d}), got {X_sv.shape}")
    coef = np.ascontiguousarray(coef, dtype=np.float64)
    if coef.shape != (X_sv.shape[0],):
        raise ValueError("coef must have one entry per support vector")
    dec = np.empty(m)
    _check(lib().svm_predict_ex(_ptr(X_sv), _ptr(coef), coef.shape[0], d, float(b), int(kernel),
                                _gamma(gamma, kernel, d), _ptr(X_test), m, _ptr(dec), int(mode)))
    return dec


def svm_predict_dev(X_sv, coef, b: float, kernel: int, gamma: Optional[float], X_test, stream=None,
                    mode: int = PREDICT_EXACT):
    """torch CUDA tensors (X_sv float32 [n_sv, d], coef float64 [n_sv], X_test float32
    [m, d], one device) -> decision values tensor [m] fp64."""
    import torch
    if X_test.dim() != 2 or X_sv.dim() != 2:
        raise ValueError("X_sv and X_test must be 2-D")
    m, d = X_test.shape
    dv = X_test.device
    tp = _dev(X_test, torch.float32, "X_test")
    sp = _dev(X_sv, torch.float32, "X_sv", (X_sv.shape[0], d), dv)
    cp = _dev(coef, torch.float64, "coef", (X_sv.shape[0],), dv)
    dec = torch.empty(m, dtype=torch.float64, device=dv)
    _check(lib().svm_predict_dev_ex(sp, cp, coef.shape[0], d, float(b), int(kernel), _gamma(gamma, kernel, d),
                                    tp, m, ctypes.c_void_p(dec.data_ptr()), int(mode), _stream_ptr(stream, dv)))
    return dec


def svm_train_batch_dev(problems, C: float, kernel: int, gamma: Optional[float] = None, tol: float = 1e-3,
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
    p = make_params(C, kernel, _gamma(gamma, kernel, d), tol, **params)
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


class HostComm:
    """A communicator bootstrapped through a host all-gather over a torch.distributed
    process group (e.g. gloo) -- svm_comm_init_host.  Keeps the callback alive."""

    def __init__(self, rank: int, world: int, device: int, group=None):
        import torch
        import torch.distributed as dist

        def allgather(ctx, send, recv, nbytes):
            try:
                src = torch.frombuffer(bytearray(ctypes.string_at(send, nbytes)), dtype=torch.uint8) \
                    if nbytes > 0 else torch.zeros(0, dtype=torch.uint8)
                out = [torch.empty(nbytes, dtype=torch.uint8) for _ in range(world)]
                dist.all_gather(out, src, group=group)
                flat = torch.cat(out).numpy().tobytes()
                ctypes.memmove(recv, flat, len(flat))
                return 0
            except Exception:                                    # reported as SVM_ENCCL
                return 1

        self._fn = _ALLGATHER_FN(allgather)
        self._coll = HostColl(None, self._fn)
        self.handle = ctypes.c_void_p()
        _check(lib().svm_comm_init_host(ctypes.byref(self.handle), rank, world, device, ctypes.byref(self._coll)))

    @property
    def _as_parameter_(self):
        return self.handle


def svm_comm_init_host(rank: int, world: int, device: int, group=None) -> HostComm:
    return HostComm(rank, world, device, group)


def svm_comm_destroy(comm) -> None:
    lib().svm_comm_destroy(comm.handle if isinstance(comm, HostComm) else comm)


def svm_train_shard(comm, X_local, y_local, row_offset: int, n_global: int, C: float, kernel: int,
                    gamma: Optional[float] = None, tol: float = 1e-3, stream=None, trace_cap: int = 0,
                    want_f: bool = False, alpha0=None, f0=None, **params):
    """Row-sharded solve, one process per GPU.  X_local/y_local: this rank's torch CUDA
    rows.  Returns dict(alpha tensor [n_local], b, info, [f tensor [n_local]], [trace
    (rank 0)]).  alpha0 / f0: optional warm start of the rank's rows (CUDA float64)."""
    import torch
    n_local, d = X_local.shape
    xp = _dev(X_local, torch.float32, "X_local")
    yp = _dev(y_local, torch.int8, "y_local", (n_local,), X_local.device)
    alpha = torch.empty(max(n_local, 1), dtype=torch.float64, device=X_local.device)[:n_local]
    p = make_params(C, kernel, _gamma(gamma, kernel, d), tol, **params)
    b = ctypes.c_double()
    info = Info()
    dbg, keep = _dev_debug(n_local, X_local.device, alpha0, f0, want_f, trace_cap)
    h = comm.handle if isinstance(comm, HostComm) else comm
    _check(lib().svm_train_shard(h, xp, yp, n_local, row_offset, n_global, d, ctypes.byref(p),
                                 ctypes.c_void_p(alpha.data_ptr()), ctypes.byref(b), ctypes.byref(info),
                                 ctypes.byref(dbg), _stream_ptr(stream, X_local.device)))
    out = dict(alpha=alpha, b=b.value, info=info.as_dict())
    if "trace" in keep:
        out["trace"] = keep["trace"][:min(info.iterations, trace_cap)]
    if "f" in keep:
        out["f"] = keep["f"]
    return out


def shard_rows(n: int, world: int):
    """Contiguous row blocks: rank r owns [r*ceil(n/P), min(n, (r+1)*ceil(n/P)))."""
    per = -(-n // world)
    return [(min(n, r * per), min(n, (r + 1) * per)) for r in range(world)]
