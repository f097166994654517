"""OvO multiclass training time on the Pavia-like stand-in (Table 4 sizes:
9 classes, 102 bands, 200/400/600/800 samples per class, 36 binary SMOs).  Context for
the paper's MPI-CUDA column (GTX 950M, 8.49-10.69 s); prints one JSON line per size.
  python tools/ovo_bench.py [--per-class 200 400 600 800] [--batch 8]"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2311_14908_b200 as S  # noqa: E402
from gen import workloads as W  # noqa: E402
from paper_2311_14908_b200.multiclass import predict_ovo, train_ovo  # noqa: E402

PAPER = {200: 8.4855, 400: 9.13105, 600: 9.6268, 800: 10.688}   # PAPER.md L346-352 (Table 4)

ap = argparse.ArgumentParser()
ap.add_argument("--per-class", type=int, nargs="*", default=[200, 400, 600, 800])
ap.add_argument("--batch", type=int, default=8)
ap.add_argument("--repeats", type=int, default=3)
args = ap.parse_args()
S.lib()
for k in args.per_class:
    X, labels = W.pavia_like(k, seed=11)
    Xt, lt = W.pavia_like(100, seed=12)
    gamma, C = 1.0 / 102, 10.0
    train_ovo(X, labels, 9, C, S.RBF, gamma, 1e-3, batch=args.batch)    # warm-up
    ts = []
    for _ in range(args.repeats):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        model = train_ovo(X, labels, 9, C, S.RBF, gamma, 1e-3, batch=args.batch)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    pred = predict_ovo(model, X, Xt, mode=S.PREDICT_TENSOR)
    iters = sum(m["info"]["iterations"] for m in model.models.values())
    print(json.dumps({"workload": f"Pavia-like 9 classes x {k}/class, d=102, RBF gamma=1/102, C=10",
                      "ovo_train_s": float(np.median(ts)), "pairs": 36, "batch": args.batch,
                      "smo_iterations_total": int(iters), "test_accuracy": float((pred == lt).mean()),
                      "paper_mpi_cuda_s_gtx950m": PAPER.get(k)}), flush=True)
