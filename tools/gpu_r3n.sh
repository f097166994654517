# phase timers in shared memory (fewer spills): timings, tests
OUT=gpurun_out/r3n
mkdir -p $OUT
for rep in 1 2; do
  SVMB200_PHASE_TIMERS=0 timeout 300 python tools/phase_probe.py W4:20000 W5@125000:5000 W3:0 W5:1500 >> $OUT/t.txt 2>&1
done
SVMB200_PHASE_TIMERS=1 timeout 300 python tools/phase_probe.py W4:20000 >> $OUT/phase.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
