"""One tensor-core prediction at the W5 shape (profiling aid: run under ncu).
  python tools/predict_one.py [m] [n_sv] [exp_variant]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2311_14908_b200 as S  # noqa: E402
from gen import workloads as W  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 37888
nsv = int(sys.argv[2]) if len(sys.argv) > 2 else 284028
if len(sys.argv) > 3:
    os.environ["SVMB200_PREDICT_EXP"] = sys.argv[3]
w = W.get("W5")
X, _ = w.train(nsv)
Xt, _ = w.test(m)
coef = torch.from_numpy(np.random.default_rng(5).uniform(-1, 1, nsv)).cuda()
dec = S.svm_predict_dev(torch.from_numpy(X).cuda(), coef, 0.1, w.kernel, w.gamma, torch.from_numpy(Xt).cuda(), mode=1)
torch.cuda.synchronize()
print("predict", m, nsv, float(dec[:4].sum()))
