"""One GD training run on the full W2 (profiling aid: run under ncu).
  python tools/gd_one.py [epochs]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2311_14908_b200 as S  # noqa: E402
from gen import workloads as W  # noqa: E402

w = W.get("W2")
X, y = w.train()
ep = int(sys.argv[1]) if len(sys.argv) > 1 else 3
r = S.svm_train_gd_dev(torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda(), w.C, w.kernel, w.gamma, 1e-4, ep)
torch.cuda.synchronize()
print("gd", ep, r["info"])
