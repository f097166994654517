"""The real cross-process row-sharded path on one B200: two processes (torchrun, gloo
bootstrap through svm_comm_init_host) each own half the rows; every iteration every CTA
stores its record into both processes' mailboxes through CUDA IPC mappings with
system-scope stores, exactly the code path of one process per GPU (only the link
differs: HBM instead of NVLink).  The two processes' persistent kernels are time-sliced
on the GPU.  Results must equal the oracle bit for bit (S:L197 partition independence,
reading R21).  Marked `gpu`."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from gen import workloads as W
from oracle import oracle as O

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_two_processes_one_gpu(tmp_path):
    w5, w1 = W.get("W5"), W.get("W1")
    X5, y5 = w5.train(1200)
    ref5 = O.train(X5, y5, w5.C, w5.kernel, w5.gamma, w5.tol, trace_cap=100000)
    k = ref5.iterations // 2
    part = O.train(X5, y5, w5.C, w5.kernel, w5.gamma, w5.tol, max_iter=k)
    warm = str(tmp_path / "warm.npz")
    np.savez(warm, alpha=part.alpha, f=part.f)
    cases = [
        {"workload": "W5", "n": 1200},
        {"workload": "W1", "n": 200},
        {"workload": "W5", "n": 1200, "params": {"iters_per_launch": 97}},
        {"workload": "W5", "n": 1200, "warm": warm},
        {"workload": "W3", "n": 900, "params": {"wss": 2}},
    ]
    cj = str(tmp_path / "cases.json")
    json.dump(cases, open(cj, "w"))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "tests", "helpers", "shard_worker.py"), str(tmp_path), cj]
    p = subprocess.run(cmd, cwd=ROOT, timeout=600, capture_output=True, text=True)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    X1, y1 = w1.train(200)
    ref1 = O.train(X1, y1, w1.C, w1.kernel, w1.gamma, w1.tol, trace_cap=100000)
    w3 = W.get("W3")
    X3, y3 = w3.train(900)
    ref3 = O.train(X3, y3, w3.C, w3.kernel, w3.gamma, w3.tol, trace_cap=100000, wss=2)
    expect = [(ref5, 0), (ref1, 0), (ref5, 0), (ref5, k), (ref3, 0)]
    for c, (ref, k0) in enumerate(expect):
        parts = [np.load(tmp_path / f"case{c}_rank{r}.npz") for r in range(2)]
        alpha = np.concatenate([q["alpha"] for q in parts])
        f = np.concatenate([q["f"] for q in parts])
        assert int(parts[0]["iterations"]) == ref.iterations - k0 == int(parts[1]["iterations"])
        np.testing.assert_array_equal(parts[0]["trace"], ref.trace[k0:])
        np.testing.assert_array_equal(alpha, ref.alpha)
        np.testing.assert_array_equal(f, ref.f)
        assert float(parts[0]["b"]) == ref.b == float(parts[1]["b"])
        assert int(parts[0]["n_sv"]) == int(np.sum(ref.alpha > 1e-8))
        if c == 2:
            assert int(parts[0]["launches"]) > 1
