"""Build libsvmb200.so in-tree with nvcc for sm_100a (no torch extension machinery).

  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -c ... (one process
  per source, in parallel), then nvcc -shared ...

--fmad=false keeps every product and sum the source writes as a separate rounding;
the kernels request fused multiply-adds explicitly with fma() where the arithmetic
contract has one.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libsvmb200.so")
# (the solver's instantiations are spread over the four smo_*.cu units; every unit compiles
# in its own nvcc process, in parallel, then one link)
SOURCES = ["smo_gen_rbf.cu", "smo_gen_lin.cu", "smo_spec_rbf.cu", "smo_spec_lin.cu", "svmb200.cu", "predict.cu",
           "comm.cu", "gram.cu", "gd.cu", "finalize.cu", "shrink.cu"]
HEADERS = ["smo_kernel.cuh", "smo_pick.cuh", "smo_bincl.cuh", "svm_exp.cuh", "exp_table.inc", "svm_internal.h",
           "predict_tc.cuh"]


def _nccl_paths():
    try:
        import nvidia.nccl as _n  # the torch-bundled NCCL 2.28 (headers + libnccl.so.2)
        base = os.path.dirname(_n.__file__) if _n.__file__ else list(_n.__path__)[0]
    except Exception:
        base = "/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl"
    return os.path.join(base, "include"), os.path.join(base, "lib")


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "svmb200.h")]
    return any(os.path.exists(p) and os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    import tempfile
    from concurrent.futures import ThreadPoolExecutor
    inc, lib = _nccl_paths()
    srcs = [os.path.join(CSRC, f) for f in SOURCES if os.path.exists(os.path.join(CSRC, f))]
    common = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo",
              "--fmad=false", "-std=c++17", "-Xcompiler", "-fPIC",
              "-Xptxas", "-v" if verbose else "-O3",
              "-I", inc, "-I", os.path.join(ROOT, "include")]
    with tempfile.TemporaryDirectory(prefix="svmb200_build_") as tmp:
        objs = [os.path.join(tmp, os.path.basename(f) + ".o") for f in srcs]

        def compile_one(k):
            subprocess.check_call(common + ["-c", srcs[k], "-o", objs[k]])

        workers = max(1, min(len(srcs), os.cpu_count() or 1))
        with ThreadPoolExecutor(max_workers=workers) as ex:
            list(ex.map(compile_one, range(len(srcs))))       # re-raises the first failure
        link = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC",
                "-o", LIB + ".tmp"] + objs + [
               "-L", lib, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + lib, "-lcudart"]
        subprocess.check_call(link)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
