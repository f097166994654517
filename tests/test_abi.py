"""CPU-side checks of the CUDA path's boundary and host logic (no GPU needed):
the C-ABI library loads and exports every symbol include/svmb200.h declares, argument
validation answers before any device work, the binding's struct layouts match the
header, and the CUDA path's exp (compiled for the host from the same header) is
correctly rounded."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "svmb200.h")


@pytest.fixture(scope="module")
def S():
    from paper_2311_14908_b200 import _build
    _build.build()
    import paper_2311_14908_b200 as S
    return S


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(svm_[a-z_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for n in ("svm_train", "svm_train_ex", "svm_train_dev", "svm_predict", "svm_predict_dev",
              "svm_comm_unique_id", "svm_comm_init", "svm_comm_init_host", "svm_train_shard",
              "svm_comm_destroy", "svm_support_vectors_dev", "svm_last_error", "svm_version"):
        assert n in names


def test_library_exports_every_declared_symbol(S):
    L = S.lib()
    for n in declared_functions():
        assert hasattr(L, n), n
    out = subprocess.check_output(["nm", "-D", "--defined-only", S.LIB_PATH]).decode()
    exported = set(re.findall(r" T (svm_\w+)", out))
    assert set(declared_functions()) <= exported


def test_library_is_sm100a(S):
    out = subprocess.check_output(["cuobjdump", "--list-elf", S.LIB_PATH]).decode()
    assert "sm_100a" in out


def test_struct_layouts_match_header(S):
    # svm_params: 3 doubles, int64, int32, int32, double, int32, int32, int64, 6 x int32 = 88 bytes
    assert ctypes.sizeof(S.Params) == 88
    # svm_info: int64, 2 x int32, 4 doubles, 2 doubles, int64, 2 x int64, double = 96 bytes
    assert ctypes.sizeof(S.Info) == 96
    assert ctypes.sizeof(S.Debug) == 40
    assert S.version().startswith("svmb200")


@pytest.mark.parametrize("kw,msg", [
    (dict(n=1), "n < 2"), (dict(d=0), "d < 1"), (dict(C=0.0), "C must"),
    (dict(C=float("inf")), "C must"), (dict(kernel=7), "unknown kernel"),
    (dict(kernel=1, gamma=0.0), "gamma"), (dict(kernel=1, gamma=-1.0), "gamma"),
])
def test_argument_validation_before_device_work(S, kw, msg):
    n, d = kw.pop("n", 4), kw.pop("d", 2)
    p = S.make_params(kw.pop("C", 1.0), kw.pop("kernel", 0), kw.pop("gamma", 0.0))
    X = np.zeros((max(n, 1), max(d, 1)), np.float32)
    y = np.ones(max(n, 1), np.int8)
    alpha = np.empty(max(n, 1))
    b = ctypes.c_double()
    rc = S.lib().svm_train_ex(X.ctypes.data, y.ctypes.data, n, d, ctypes.byref(p), alpha.ctypes.data,
                              ctypes.byref(b), None, None)
    assert rc == -1
    assert msg in S.lib().svm_last_error().decode()


def test_last_plan_before_any_solve(S):
    assert isinstance(S.last_plan(), dict)


def test_null_pointers_rejected(S):
    b = ctypes.c_double()
    assert S.lib().svm_train(None, None, 4, 2, 1.0, 0, 0.0, 1e-3, None, ctypes.byref(b)) == -1
    assert S.lib().svm_predict(None, None, 0, 2, 0.0, 0, 0.0, None, 3, None) == -1


def test_shard_rows_partition():
    from paper_2311_14908_b200 import shard_rows
    for n in (2, 7, 200, 581012, 1_000_000):
        for P in (1, 2, 3, 4, 8):
            blocks = shard_rows(n, P)
            assert blocks[0][0] == 0 and blocks[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(blocks, blocks[1:]))


@pytest.fixture(scope="module")
def exp_host(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("exp") / "exp_host.so")
    subprocess.check_call(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-fPIC", "-shared",
                           "-o", out, os.path.join(ROOT, "tests", "helpers", "exp_host.cpp")])
    L = ctypes.CDLL(out)
    L.svm_exp_host.restype = ctypes.c_double
    L.svm_exp_host.argtypes = [ctypes.c_double]
    L.svm_exp_host_batch.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_long]
    return L


def test_cuda_path_exp_correctly_rounded(exp_host):
    """The CUDA path's exp (svm_exp.cuh, built for the host) agrees with mpmath's
    correctly rounded exponential; independent of oracle/."""
    import mpmath
    mpmath.mp.prec = 256
    rng = np.random.default_rng(21)
    xs = np.concatenate([-rng.uniform(0, 708, 3000), -np.exp(rng.uniform(-45, 1.5, 3000)),
                         -np.arange(0, 60, 0.5), [-708.0, -1e-300, -0.0, 0.0]])
    for x in xs:
        assert exp_host.svm_exp_host(float(x)) == float(mpmath.exp(mpmath.mpf(float(x)))), x
    assert exp_host.svm_exp_host(-708.5) == 0.0


def test_cuda_path_exp_matches_oracle_exp_bulk(exp_host):
    """Two independent correctly rounded exps (oracle: series-built double-double with
    argument halving; CUDA path: table-driven two-phase) agree on 10^6 arguments."""
    from oracle import oracle as O
    rng = np.random.default_rng(22)
    xs = np.concatenate([-rng.uniform(0, 30, 400000), -rng.uniform(0, 708, 300000),
                         -np.exp(rng.uniform(-40, 2, 300000))])
    out = np.empty_like(xs)
    exp_host.svm_exp_host_batch(xs.ctypes.data, out.ctypes.data, xs.size)
    ref = np.array([O.exp_cr(x) for x in xs[:200000]])
    np.testing.assert_array_equal(out[:200000], ref)


def test_binding_validates_before_the_library(S):
    """Host-side argument checks of the binding: a warm start needs both
    alpha0 and f0 of shape (n,); a support-vector / test dimension mismatch raises
     instead of being reshaped."""
    X = np.zeros((4, 2), np.float32)
    y = np.array([1, -1, 1, -1], np.int8)
    with pytest.raises(ValueError, match="both"):
        S.svm_train_ex(X, y, 1.0, S.LINEAR, alpha0=np.zeros(4))
    with pytest.raises(ValueError, match="shape"):
        S.svm_train_ex(X, y, 1.0, S.LINEAR, alpha0=np.zeros(3), f0=np.zeros(3))
    with pytest.raises(ValueError, match="X_sv"):
        S.svm_predict(np.zeros((3, 3), np.float32), np.ones(3), 0.0, S.LINEAR, 0.0, X)
    with pytest.raises(ValueError, match="coef"):
        S.svm_predict(np.zeros((3, 2), np.float32), np.ones(2), 0.0, S.LINEAR, 0.0, X)


def test_gamma_defaults_to_one_over_d(S):
    """the RBF width defaults to 1/d in the Python layer (the C ABI has none)."""
    from paper_2311_14908_b200 import _gamma
    assert _gamma(None, S.RBF, 256) == 1.0 / 256
    assert _gamma(None, S.LINEAR, 256) == 0.0
    assert _gamma(0.5, S.RBF, 256) == 0.5


def test_support_vector_call_validates(S):
    n = ctypes.c_int64()
    assert S.lib().svm_support_vectors_dev(None, None, None, 4, 2, 0.0, None, None, None, ctypes.byref(n), None) == -1
    a = np.zeros(4)
    # coef requested without y
    assert S.lib().svm_support_vectors_dev(None, None, a.ctypes.data, 4, 2, 0.0, None, a.ctypes.data, None,
                                           ctypes.byref(n), None) == -1
