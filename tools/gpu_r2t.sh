mkdir -p gpurun_out/r2t
timeout 300 python tools/probe_r2.py iters > gpurun_out/r2t/probe_iters.jsonl 2> gpurun_out/r2t/probe_iters.err
SVMB200_PHASE_TIMERS=1 timeout 300 python tools/phase_probe.py W4:20000 W3:0 > gpurun_out/r2t/phase.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_boundary.py tests/test_wss2_gpu.py -q -x -k "cache or mixed or W3 or wss2" > gpurun_out/r2t/pytest.log 2>&1; echo rc=$? >> gpurun_out/r2t/pytest.log
