mkdir -p gpurun_out/r2r
timeout 300 python tools/probe_r2.py iters > gpurun_out/r2r/probe_iters.jsonl 2> gpurun_out/r2r/probe_iters.err
SVMB200_PHASE_TIMERS=1 timeout 300 python tools/phase_probe.py W4:20000 W5:2000 > gpurun_out/r2r/phase.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_shrink_gpu.py tests/test_wss2_gpu.py tests/test_gpu_fullsize.py -q -x > gpurun_out/r2r/pytest.log 2>&1; echo rc=$? >> gpurun_out/r2r/pytest.log
