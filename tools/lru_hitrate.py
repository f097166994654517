"""Evidence for SURVEY §8 row a8 (HBM kernel-row LRU cache): replay the exact pair
trajectory of a solve (the GPU's pair trace) through an LRU cache of kernel rows and
report the hit rate for capacities that fit in HBM.
  python tools/lru_hitrate.py W4 W5:100000"""
import collections
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2311_14908_b200 as S  # noqa: E402
from gen import workloads as W  # noqa: E402


def lru_hits(trace, cap):
    cache = collections.OrderedDict()
    hits = 0
    for u, l in trace:
        for i in (int(u), int(l)):
            if i in cache:
                hits += 1
                cache.move_to_end(i)
            else:
                cache[i] = True
                if len(cache) > cap:
                    cache.popitem(last=False)
    return hits / (2 * len(trace))


for spec in sys.argv[1:]:
    name, _, mi = spec.partition(":")
    w = W.get(name)
    X, y = w.train()
    kw = dict(max_iter=int(mi)) if mi else {}
    r = S.svm_train_dev(torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda(), w.C, w.kernel, w.gamma, w.tol,
                        trace_cap=int(mi) if mi else 10 * len(y), gram=-1, **kw)
    tr = r["trace"]
    row_bytes = 8 * len(y)
    out = {"workload": name, "n": len(y), "iterations": len(tr), "row_bytes": row_bytes}
    for frac in (0.005, 0.01, 0.02, 0.05, 0.10):
        cap = max(1, int(frac * len(y)))
        out[f"hit@{frac:g}n ({cap * row_bytes / 1e9:.1f} GB)"] = round(lru_hits(tr, cap), 4)
    print(json.dumps(out), flush=True)
