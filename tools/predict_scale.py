"""Batched prediction at the W5 scale (BASELINE.json configs[4]: "batched predict on 1M test
rows"): m test rows against n_sv support vectors (rows of the W5 training law with random
coefficients -- timing only), d = 256, RBF gamma = 1/256, tcgen05 3xTF32 path.
  python tools/predict_scale.py [m] [n_sv]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2311_14908_b200 as S  # noqa: E402
from gen import workloads as W  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
nsv = int(sys.argv[2]) if len(sys.argv) > 2 else 400_000
w = W.get("W5")
Xs, _ = w.train(nsv)
Xt, _ = w.test(m)
rng = np.random.default_rng(0)
coef = rng.uniform(-1.0, 1.0, nsv) * w.C
Xs_d, Xt_d = torch.from_numpy(Xs).cuda(), torch.from_numpy(Xt).cuda()
cf_d = torch.from_numpy(coef).cuda()
st = torch.cuda.current_stream()
S.svm_predict_dev(Xs_d, cf_d, 0.0, w.kernel, w.gamma, Xt_d[:4096].contiguous(), stream=st, mode=S.PREDICT_TENSOR)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
dec = S.svm_predict_dev(Xs_d, cf_d, 0.0, w.kernel, w.gamma, Xt_d, stream=st, mode=S.PREDICT_TENSOR)
e1.record(st)
torch.cuda.synchronize()
t = e0.elapsed_time(e1) * 1e-3
flop = 2.0 * m * nsv * w.d
print(json.dumps({"m": m, "n_sv": nsv, "d": w.d, "seconds": t, "algorithmic_tflops": flop / t / 1e12,
                  "tf32_mma_tflops_issued": 3 * flop / t / 1e12, "gexp_per_s": m * nsv / t / 1e9,
                  "dec_finite": bool(torch.isfinite(dec).all().item())}), flush=True)
