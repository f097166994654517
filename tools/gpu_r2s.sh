mkdir -p gpurun_out/r2s
timeout 300 python tools/probe_r2.py iters > gpurun_out/r2s/probe_iters.jsonl 2> gpurun_out/r2s/probe_iters.err
SVMB200_PHASE_TIMERS=1 timeout 300 python tools/phase_probe.py W4:20000 > gpurun_out/r2s/phase.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_wss2_gpu.py tests/test_shrink_gpu.py -q -x -k "mixed or W4 or wss2 or shrink or partition or trajectory" > gpurun_out/r2s/pytest.log 2>&1; echo rc=$? >> gpurun_out/r2s/pytest.log
