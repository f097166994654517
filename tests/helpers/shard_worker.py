"""Worker of tests/test_two_process.py: one rank of a row-sharded solve, launched by
torchrun (several processes on ONE GPU; bootstrap through gloo and svm_comm_init_host,
since NCCL refuses two ranks on one device).  Writes each case's result to out_dir.

  python -m torch.distributed.run --nproc-per-node 2 ... shard_worker.py out_dir cases.json
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main(out_dir, cases_json):
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo")
    torch.cuda.set_device(0)
    import paper_2311_14908_b200 as S
    from gen import workloads as W
    comm = S.svm_comm_init_host(rank, world, 0)
    try:
        for k, case in enumerate(json.load(open(cases_json))):
            w = W.get(case["workload"])
            X, y = w.train(case["n"])
            n = len(y)
            lo, hi = S.shard_rows(n, world)[rank]
            Xl = torch.from_numpy(X[lo:hi]).cuda().contiguous()
            yl = torch.from_numpy(y[lo:hi]).cuda().contiguous()
            kw = dict(case.get("params", {}))
            warm = case.get("warm")
            if warm:
                z = np.load(warm)
                kw["alpha0"] = torch.from_numpy(z["alpha"][lo:hi]).cuda().contiguous()
                kw["f0"] = torch.from_numpy(z["f"][lo:hi]).cuda().contiguous()
            r = S.svm_train_shard(comm, Xl, yl, lo, n, w.C, w.kernel, w.gamma, w.tol,
                                  trace_cap=10 * n + 10000, want_f=True, **kw)
            np.savez(os.path.join(out_dir, f"case{k}_rank{rank}.npz"), alpha=r["alpha"].cpu().numpy(),
                     f=r["f"].cpu().numpy(), trace=r.get("trace", np.zeros((0, 2), np.int64)), b=r["b"],
                     iterations=r["info"]["iterations"], launches=r["info"]["launches"],
                     n_sv=r["info"]["n_sv"], W=r["info"]["dual_objective"], lo=lo, hi=hi)
    finally:
        S.svm_comm_destroy(comm)
        dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
