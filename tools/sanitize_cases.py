"""Small solves / predictions for compute-sanitizer (memcheck, racecheck, synccheck):
  compute-sanitizer --tool racecheck python tools/sanitize_cases.py <case>
cases: bincl (smo_bincl, W2 rows in a cluster), cluster (smo_persistent cluster mode, W1),
global (smo_persistent, 8 CTAs, global mailboxes, streamed stages), cache (row cache),
wss2 (second-order gain pass), predict_tc (k_predict_tc), predict_exact, gd (k_gd_epoch)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2311_14908_b200 as S  # noqa: E402
from gen import workloads as W  # noqa: E402

case = sys.argv[1]
it = int(sys.argv[2]) if len(sys.argv) > 2 else 30
if case == "bincl":
    w = W.get("W2"); X, y = w.train(600)
    r = S.svm_train_ex(X, y, w.C, w.kernel, w.gamma, w.tol, max_iter=it, cluster=2)
elif case == "cluster":
    w = W.get("W1"); X, y = w.train(200)
    r = S.svm_train_ex(X, y, w.C, w.kernel, w.gamma, w.tol, max_iter=it, cluster=2)
elif case == "global":
    os.environ["SVMB200_NO_RESIDENT"] = "1"
    w = W.get("W5"); X, y = w.train(3000)
    r = S.svm_train_ex(X, y, w.C, w.kernel, w.gamma, w.tol, max_iter=it, ctas=8, cluster=-1, cache_rows=-1)
elif case == "cache":
    os.environ["SVMB200_NO_RESIDENT"] = "1"
    w = W.get("W3"); X, y = w.train(1500)
    r = S.svm_train_ex(X, y, w.C, w.kernel, w.gamma, w.tol, max_iter=it, ctas=8, cluster=-1, cache_rows=8)
elif case == "wss2":
    w = W.get("W4"); X, y = w.train(2000)
    r = S.svm_train_ex(X, y, w.C, w.kernel, w.gamma, w.tol, max_iter=it, ctas=8, wss=2)
elif case in ("predict_tc", "predict_exact"):
    w = W.get("W5"); X, y = w.train(300)
    Xt, _ = w.test(200)
    coef = np.random.default_rng(0).uniform(-1, 1, 300)
    d = S.svm_predict(X, coef, 0.1, w.kernel, w.gamma, Xt, mode=1 if case == "predict_tc" else 0)
elif case == "gd":
    w = W.get("W2"); X, y = w.train(500)
    S.svm_train_gd_dev(torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda(), w.C, w.kernel, w.gamma, 1e-3, 3)
torch.cuda.synchronize()
print(case, "ok", S.last_plan())
