"""Per-GPU shard sizes of a multi-GPU run on one GPU: W5 rows n (e.g. 125,000 = 1/8 of W5)
with and without the L2 evict_last window (SVMB200_L2_KEEP_MB), profiling aid.
  python tools/l2_probe.py n iters"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2311_14908_b200 as S  # noqa: E402
from gen import workloads as W  # noqa: E402

n, k = int(sys.argv[1]), int(sys.argv[2])
w = W.get("W5")
X, y = w.train(n)
Xd, yd = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
for rep in range(2):
    r = S.svm_train_dev(Xd, yd, w.C, w.kernel, w.gamma, w.tol, max_iter=k, cache_rows=-1)
us = 1e6 * r["info"]["seconds_solve"] / r["info"]["iterations"]
print(f"n={n} keep={os.environ.get('SVMB200_L2_KEEP_MB', '0')} MB: {us:.2f} us/iter, "
      f"{n * 1049 / us / 1e3:.0f} GB/s, plan {S.last_plan()['mode']}", flush=True)
