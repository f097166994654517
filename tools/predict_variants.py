"""Tensor-core prediction at the bench shape (10^6 held-out W5 rows x 284,028 SVs, d = 256)
for each epilogue exp variant (SVMB200_PREDICT_EXP), timed with CUDA events; max |diff|
against the exact fp64 path (bit-identical to the oracle) on 2,048 sampled rows.  Also the
cuBLAS TF32 and BF16 GEMM rates (8192^3) as the tensor-pipe peaks of this box.
  python tools/predict_variants.py [variants, e.g. 0,3,4 or 3:128,3:256 (exp variant:BN)]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2311_14908_b200 as S  # noqa: E402
from gen import workloads as W  # noqa: E402


def timed(fn, reps=1):
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        out = fn()
    e1.record(st)
    torch.cuda.synchronize()
    return out, e0.elapsed_time(e1) * 1e-3 / reps


variants = (sys.argv[1] if len(sys.argv) > 1 else "0,3,4").split(",")
peaks = "--no-peaks" not in sys.argv
# tensor-pipe peaks (cuBLAS)
n = 8192 if peaks else 256
a = torch.randn(n, n, device="cuda")
bm = torch.randn(n, n, device="cuda")
torch.backends.cuda.matmul.allow_tf32 = True
for _ in range(3):
    a @ bm
_, t = timed(lambda: a @ bm, 10)
print(json.dumps({"probe": "cublas_tf32", "n": n, "tflops": 2 * n ** 3 / t / 1e12}), flush=True)
ah, bh = a.bfloat16(), bm.bfloat16()
for _ in range(3):
    ah @ bh
_, t = timed(lambda: ah @ bh, 10)
print(json.dumps({"probe": "cublas_bf16", "n": n, "tflops": 2 * n ** 3 / t / 1e12}), flush=True)
del a, bm, ah, bh
torch.cuda.empty_cache()

w = W.get("W5")
nsv = 284_028
X, _ = w.train(nsv)
Xsv = torch.from_numpy(X).cuda()
coef = torch.from_numpy(np.random.default_rng(5).uniform(-1, 1, nsv)).cuda()
Xt, _ = w.test()
Xt = torch.from_numpy(Xt).cuda()
rows = torch.from_numpy(np.random.default_rng(6).choice(Xt.shape[0], 2048, replace=False)).cuda()
ref = S.svm_predict_dev(Xsv, coef, 0.1, w.kernel, w.gamma, Xt[rows].contiguous(), mode=S.PREDICT_EXACT)
for spec in variants:
    v, _, bn = spec.partition(":")
    os.environ["SVMB200_PREDICT_EXP"] = v
    os.environ["SVMB200_PREDICT_BN"] = bn or "128"
    S.svm_predict_dev(Xsv, coef, 0.1, w.kernel, w.gamma, Xt, mode=S.PREDICT_TENSOR)     # warm, full shape
    dec, t = timed(lambda: S.svm_predict_dev(Xsv, coef, 0.1, w.kernel, w.gamma, Xt, mode=S.PREDICT_TENSOR))
    err = float((dec[rows] - ref).abs().max())
    print(json.dumps({"probe": "predict", "exp_variant": int(v), "bn": int(bn or 128), "rows": Xt.shape[0], "n_sv": nsv, "seconds": t,
                      "tflops_algorithmic": 2.0 * Xt.shape[0] * nsv * 256 / t / 1e12,
                      "tf32_issued_tflops": 6.0 * Xt.shape[0] * nsv * 256 / t / 1e12,
                      "max_err_vs_exact": err}), flush=True)
