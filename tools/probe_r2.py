"""Round-2 perf probe (one GPU): per-iteration times of the streamed configs, the tensor-core
predict epilogue variants at the W5 scale, and window shrinking on the full solves.
  python tools/probe_r2.py [what ...]   what: iters predict shrink5 shrink4"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2311_14908_b200 as S  # noqa: E402
from gen import workloads as W  # noqa: E402

what = sys.argv[1:] or ["iters", "predict", "shrink5"]


def dev(name, n=None):
    w = W.get(name)
    X, y = w.train(n)
    return w, torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()


def timed(fn):
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); r = fn(); e1.record(); torch.cuda.synchronize()
    return r, e0.elapsed_time(e1) * 1e-3


if "iters" in what:
    for name, k in (("W3", 0), ("W4", 6000), ("W5", 1500)):
        w, Xd, yd = dev(name)
        kw = dict(max_iter=k) if k else {}
        S.svm_train_dev(Xd, yd, w.C, w.kernel, w.gamma, w.tol, **kw)
        r, t = timed(lambda: S.svm_train_dev(Xd, yd, w.C, w.kernel, w.gamma, w.tol, **kw))
        print(json.dumps({"probe": "iters", "workload": name, "iterations": r["info"]["iterations"],
                          "us_per_iter": 1e6 * r["info"]["seconds_solve"] / r["info"]["iterations"],
                          "plan": S.last_plan()}), flush=True)
        del Xd, yd
        torch.cuda.empty_cache()

if "predict" in what:
    w, Xd, yd = dev("W5")
    nsv = 284_028
    rng = np.random.default_rng(5)
    coef = torch.from_numpy(rng.uniform(-1, 1, nsv)).cuda()
    Xsv = Xd[:nsv].contiguous()
    Xt, _ = w.test()
    Xt = torch.from_numpy(Xt).cuda()
    for v in ("0", "1", "2"):
        os.environ["SVMB200_PREDICT_EXP"] = v
        S.svm_predict_dev(Xsv, coef, 0.1, w.kernel, w.gamma, Xt[:4096], mode=1)
        dec, t = timed(lambda: S.svm_predict_dev(Xsv, coef, 0.1, w.kernel, w.gamma, Xt, mode=1))
        if v == "0":
            ref = dec.clone()
        print(json.dumps({"probe": "predict", "exp_variant": int(v), "rows": Xt.shape[0], "n_sv": nsv, "seconds": t,
                          "tflops_algorithmic": 2.0 * Xt.shape[0] * nsv * 256 / t / 1e12,
                          "max_diff_vs_variant0": float((dec - ref).abs().max())}), flush=True)
    os.environ.pop("SVMB200_PREDICT_EXP")
    del Xd, yd, Xt, Xsv
    torch.cuda.empty_cache()

for tag, name in (("shrink5", "W5"), ("shrink4", "W4")):
    if tag not in what:
        continue
    w, Xd, yd = dev(name)
    for H in (0, 1000):
        r, t = timed(lambda: S.svm_train_dev(Xd, yd, w.C, w.kernel, w.gamma, w.tol, shrink_window=H))
        print(json.dumps({"probe": "shrink", "workload": name, "H": H, "time_to_converge_s": t,
                          "iterations": r["info"]["iterations"], "converged": r["info"]["converged"],
                          "b": r["b"], "n_sv": r["info"]["n_sv"], "W": r["info"]["dual_objective"],
                          "launches": r["info"]["launches"]}), flush=True)
    del Xd, yd
    torch.cuda.empty_cache()

if "wss5" in what:
    # the second-order rule on W5 (report both rules on the bench config)
    w, Xd, yd = dev("W5")
    for wss in (1, 2):
        r, t = timed(lambda: S.svm_train_dev(Xd, yd, w.C, w.kernel, w.gamma, w.tol, wss=wss))
        print(json.dumps({"probe": "wss", "workload": "W5", "wss": wss, "time_to_converge_s": t,
                          "iterations": r["info"]["iterations"], "us_per_iter": 1e6 * t / r["info"]["iterations"],
                          "b": r["b"], "n_sv": r["info"]["n_sv"], "W": r["info"]["dual_objective"]}), flush=True)
    del Xd, yd
    torch.cuda.empty_cache()

if "cache4" in what:
    # the kernel-row cache on W4 (auto-off for n > 200k: replayed LRU hit rate ~11%)
    w, Xd, yd = dev("W4")
    for slots in (-1, 2048):
        r, t = timed(lambda: S.svm_train_dev(Xd, yd, w.C, w.kernel, w.gamma, w.tol, cache_rows=slots))
        print(json.dumps({"probe": "cache", "workload": "W4", "cache_rows": slots, "time_to_converge_s": t,
                          "iterations": r["info"]["iterations"], "cache_hits": r["info"]["cache_hits"],
                          "cache_misses": r["info"]["cache_misses"], "plan": S.last_plan()}), flush=True)
    del Xd, yd
    torch.cuda.empty_cache()

if "pf5" in what:
    # L2 prefetch beyond the ring x L2 keep window, W5 prefix (SVMB200_L2_PF / _L2_KEEP_MB)
    w, Xd, yd = dev("W5")
    for pf, keep in (("0", "48"), ("2", "48"), ("4", "48"), ("4", "16"), ("6", "0"), ("8", "0"), ("0", "48")):
        os.environ["SVMB200_L2_PF"] = pf
        os.environ["SVMB200_L2_KEEP_MB"] = keep
        S.svm_train_dev(Xd, yd, w.C, w.kernel, w.gamma, w.tol, max_iter=200)
        ts = []
        for rep in range(2):
            r, t = timed(lambda: S.svm_train_dev(Xd, yd, w.C, w.kernel, w.gamma, w.tol, max_iter=2000))
            ts.append(1e6 * r["info"]["seconds_solve"] / r["info"]["iterations"])
        print(json.dumps({"probe": "l2pf", "workload": "W5", "pf": int(pf), "keep_mb": int(keep), "us_per_iter": ts}), flush=True)
    os.environ.pop("SVMB200_L2_PF"); os.environ.pop("SVMB200_L2_KEEP_MB")
    del Xd, yd
    torch.cuda.empty_cache()

if "shards" in what:
    # the per-GPU work of a P-way W5 shard, on one GPU (rows 1M / P, the launch configuration
    # of a rank: row cache off as for n_global = 1M)
    w = W.get("W5")
    for n in (125_000, 250_000, 500_000, 1_000_000):
        X, y = w.train(n)
        Xd, yd = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
        S.svm_train_dev(Xd, yd, w.C, w.kernel, w.gamma, w.tol, max_iter=300, cache_rows=-1)
        r, t = timed(lambda: S.svm_train_dev(Xd, yd, w.C, w.kernel, w.gamma, w.tol, max_iter=3000, cache_rows=-1))
        print(json.dumps({"probe": "shard", "workload": "W5", "rows": n, "P_equiv": 1_000_000 // n,
                          "us_per_iter": 1e6 * r["info"]["seconds_solve"] / r["info"]["iterations"],
                          "plan": S.last_plan()}), flush=True)
        del Xd, yd
        torch.cuda.empty_cache()

if "keep" in what:
    # L2 evict_last window size for W5 shards (the per-GPU work of a P-way run)
    w = W.get("W5")
    for n in (125_000, 250_000):
        X, y = w.train(n)
        Xd, yd = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
        for keep in ("0", "48", "64", "80", "96", "112"):
            os.environ["SVMB200_L2_KEEP_MB"] = keep
            S.svm_train_dev(Xd, yd, w.C, w.kernel, w.gamma, w.tol, max_iter=300, cache_rows=-1)
            r, t = timed(lambda: S.svm_train_dev(Xd, yd, w.C, w.kernel, w.gamma, w.tol, max_iter=3000, cache_rows=-1))
            print(json.dumps({"probe": "keep", "rows": n, "keep_mb": int(keep),
                              "us_per_iter": 1e6 * r["info"]["seconds_solve"] / r["info"]["iterations"]}), flush=True)
        os.environ.pop("SVMB200_L2_KEEP_MB")
        del Xd, yd
        torch.cuda.empty_cache()

if "persist" in what:
    # persisting-L2 carve-out x evict_last window (SVMB200_L2_PERSIST_MB, SVMB200_L2_KEEP_MB)
    w = W.get("W5")
    for n, its in ((125_000, 3000), (1_000_000, 1500)):
        X, y = w.train(n)
        Xd, yd = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
        for persist, keep in (("", "48"), ("79", "48"), ("79", "64"), ("79", "76"), ("79", "96"), ("40", "40")):
            if persist:
                os.environ["SVMB200_L2_PERSIST_MB"] = persist
            else:
                os.environ.pop("SVMB200_L2_PERSIST_MB", None)
            os.environ["SVMB200_L2_KEEP_MB"] = keep
            S.svm_train_dev(Xd, yd, w.C, w.kernel, w.gamma, w.tol, max_iter=200, cache_rows=-1)
            r, t = timed(lambda: S.svm_train_dev(Xd, yd, w.C, w.kernel, w.gamma, w.tol, max_iter=its, cache_rows=-1))
            print(json.dumps({"probe": "persist", "rows": n, "persist_mb": persist or "default", "keep_mb": int(keep),
                              "us_per_iter": 1e6 * r["info"]["seconds_solve"] / r["info"]["iterations"]}), flush=True)
        os.environ.pop("SVMB200_L2_KEEP_MB"); os.environ.pop("SVMB200_L2_PERSIST_MB", None)
        del Xd, yd
        torch.cuda.empty_cache()
