mkdir -p gpurun_out/r2g
timeout 600 python -m pytest tests/test_shrink_gpu.py -q -x > gpurun_out/r2g/pytest_shrink.log 2>&1; echo rc=$? >> gpurun_out/r2g/pytest_shrink.log
timeout 300 python tools/probe_r2.py iters > gpurun_out/r2g/probe_iters.jsonl 2> gpurun_out/r2g/probe_iters.err
SVMB200_SHRINK_LOG=1 timeout 600 python tools/probe_r2.py shrink5 shrink4 > gpurun_out/r2g/probe_shrink.jsonl 2> gpurun_out/r2g/shrink.log
