"""Per-phase cycle breakdown of the persistent SMO kernel (profiling aid).

  SVMB200_PHASE_TIMERS=1 python tools/phase_probe.py W2 W3:0 W4:20000 W5:3000 W5@125000:3000
(workload[:max_iter]; 0 = run to convergence)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if os.environ.get("SVMB200_PHASE_TIMERS", "1") != "0":
    os.environ["SVMB200_PHASE_TIMERS"] = "1"
else:
    del os.environ["SVMB200_PHASE_TIMERS"]

import torch  # noqa: E402

import paper_2311_14908_b200 as S  # noqa: E402
from gen import workloads as W  # noqa: E402

for spec in sys.argv[1:]:
    name, _, rest = spec.partition(":")
    name, _, nrows = name.partition("@")          # W5@125000:3000 -> the first 125,000 rows (a P = 8 shard)
    mi, _, kern = rest.partition(":")          # W4:20000:lin -> the linear kernel on W4's data
    w = W.get(name)
    if kern == "lin":
        import dataclasses
        w = dataclasses.replace(w, kernel=0)
    extra_kw = {"cache_rows": -1} if kern == "nocache" else {}
    X, y = w.train(int(nrows) if nrows else None)
    Xd, yd = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
    kw = dict(max_iter=int(mi)) if mi and int(mi) > 0 else {}
    for extra in (extra_kw,):
        S.svm_train_dev(Xd, yd, w.C, w.kernel, w.gamma, w.tol, **kw, **extra)   # warm
        torch.cuda.synchronize()
        t0 = time.time()
        r = S.svm_train_dev(Xd, yd, w.C, w.kernel, w.gamma, w.tol, **kw, **extra)
        torch.cuda.synchronize()
        it = r["info"]["iterations"]
        print(f"{name} {extra} iters={it} solve={r['info']['seconds_solve']:.4f}s "
              f"us/iter={1e6 * r['info']['seconds_solve'] / it:.2f} GB/s={X.nbytes * it / r['info']['seconds_solve'] / 1e9:.0f}",
              flush=True)
