"""Write oracle-computed reference results for full-size parity tests.

Calls only oracle/ (and the seeded generators in gen/).  Output: tests/golden/
<workload>_oracle.npz with alpha, f, b, b_up, b_low, iterations, converged and the
SHA-256 of the (i_up, i_low) pair trace.

  python oracle/tools/make_golden.py W2          # ~5 min on 8 cores
  python oracle/tools/make_golden.py W3 0 2      # second-order working set (wss = 2)
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from gen import workloads as W  # noqa: E402
from oracle import oracle as O  # noqa: E402


def main(name: str, n: int = 0, wss: int = 1):
    w = W.get(name)
    X, y = w.train(n or None)
    t0 = time.time()
    r = O.train(X, y, w.C, w.kernel, w.gamma, w.tol, trace_cap=10 * len(y) + 10000, wss=wss)
    dt = time.time() - t0
    trace_sha = hashlib.sha256(np.ascontiguousarray(r.trace, dtype=np.int64).tobytes()).hexdigest()
    W_obj = O.dual_objective_from_f(r.alpha, y, r.f)
    tag = (name if not n else f"{name}_n{n}") + ("" if wss == 1 else f"_wss{wss}")
    out = os.path.join(ROOT, "tests", "golden", f"{tag}_oracle.npz")
    np.savez_compressed(out, alpha=r.alpha, f=r.f, b=r.b, b_up=r.b_up, b_low=r.b_low,
                        iterations=r.iterations, converged=r.converged, trace_sha=trace_sha,
                        dual_objective=W_obj, n=len(y), seconds=dt, threads=O.num_threads(), wss=wss)
    print(json.dumps(dict(workload=tag, iterations=r.iterations, converged=r.converged,
                          n_sv=int((r.alpha > 1e-8).sum()), b=r.b, W=W_obj, seconds=dt,
                          threads=O.num_threads(), out=out)))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0, int(sys.argv[3]) if len(sys.argv) > 3 else 1)
