# wide record poll (forced on one GPU) parity + timing; full GPU suite; bench with predict last
OUT=gpurun_out/r3i
mkdir -p $OUT
timeout 2400 python -m pytest tests -m gpu -q -x --durations=10 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
for wp in 0 1 0 1; do
  echo "== wide_poll=$wp" >> $OUT/wide.txt
  SVMB200_WIDE_POLL=$wp SVMB200_PHASE_TIMERS=0 timeout 300 python tools/phase_probe.py W4:20000 W5@125000:5000 W5:1500 W3:0 >> $OUT/wide.txt 2>&1
done
timeout 1500 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
