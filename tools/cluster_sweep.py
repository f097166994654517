"""W2 solve time for forced cluster sizes (profiling aid)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import paper_2311_14908_b200 as S
from gen import workloads as W
w = W.get("W2"); X, y = w.train()
Xd, yd = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
for cl in (16, 8, 4):
    for rep in range(2):
        r = S.svm_train_dev(Xd, yd, w.C, w.kernel, w.gamma, w.tol, cluster=cl)
    torch.cuda.synchronize()
    print("cluster", cl, r["info"]["iterations"], "%.4f s" % r["info"]["seconds_solve"], "%.2f us/iter" % (1e6 * r["info"]["seconds_solve"] / r["info"]["iterations"]), S.last_plan())
