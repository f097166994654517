"""bench.py's N > 1 path (torchrun, one rank per process, row-sharded solve in K windows,
max over ranks, gathered model, sharded prediction) run with two processes on one B200:
the test hook SVMB200_BENCH_HOSTCOMM=1 bootstraps over gloo + svm_comm_init_host, since
NCCL refuses two ranks on one device.  Marked `gpu`."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_bench_two_ranks_one_gpu():
    env = dict(os.environ, SVMB200_BENCH_HOSTCOMM="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--workload", "W1", "--windowed", "--steps", "3", "--warmup", "1",
           "--no-cpu-baseline", "--no-others", "--no-gd"]
    p = subprocess.run(cmd, cwd=ROOT, env=env, timeout=900, capture_output=True, text=True)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["iterations"] == 150 and d["converged"] == 1
    assert d["launches"] == 3 and d["value"] > 0 and d["gpu_launches"] > 0
    assert d["predict"]["rows"] > 0 and d["e2e"]["value"] > 0
    assert d["config"]["parallelism"] == "rows sharded over 2 GPU(s)"
