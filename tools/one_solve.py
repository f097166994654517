"""One solve of a workload on cuda:0 (profiling aid: run under ncu).
  python tools/one_solve.py W2 [max_iter] [key=value ...]   (extra svm_params fields)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2311_14908_b200 as S  # noqa: E402
from gen import workloads as W  # noqa: E402

w = W.get(sys.argv[1])
mi = int(sys.argv[2]) if len(sys.argv) > 2 else 0
kw = dict(a.split("=") for a in sys.argv[3:])
kw = {k: int(v) for k, v in kw.items()}
X, y = w.train()
Xd, yd = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
r = S.svm_train_dev(Xd, yd, w.C, w.kernel, w.gamma, w.tol, max_iter=mi, **kw)
torch.cuda.synchronize()
print(sys.argv[1], r["info"]["iterations"], r["info"]["seconds_solve"])
