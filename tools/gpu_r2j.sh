mkdir -p gpurun_out/r2j
timeout 300 python tools/probe_r2.py predict > gpurun_out/r2j/probe_predict.jsonl 2> gpurun_out/r2j/probe_predict.err
SVMB200_PHASE_TIMERS=1 timeout 600 python tools/phase_probe.py W4:20000 W5:2000 W5@125000:4000 W5@250000:3000 W3:0 > gpurun_out/r2j/phase.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -k predict > gpurun_out/r2j/pytest_predict.log 2>&1; echo rc=$? >> gpurun_out/r2j/pytest_predict.log
