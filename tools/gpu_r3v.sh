# the solver instantiations split over four translation units: smoke, all GPU tests, timings
OUT=gpurun_out/r3v
mkdir -p $OUT
timeout 300 python __graft_entry__.py smoke > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 2400 python -m pytest tests -m gpu -q --durations=10 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
SVMB200_PHASE_TIMERS=0 timeout 300 python tools/phase_probe.py W4:20000 W5@125000:5000:nocache W3:0 W5:1500 > $OUT/t.txt 2>&1
