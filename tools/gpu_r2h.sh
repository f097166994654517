mkdir -p gpurun_out/r2h
timeout 300 python tools/probe_r2.py predict > gpurun_out/r2h/probe_predict.jsonl 2> gpurun_out/r2h/probe_predict.err
timeout 1800 python -m pytest tests -m gpu -q --durations=20 > gpurun_out/r2h/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/r2h/pytest_gpu.log
