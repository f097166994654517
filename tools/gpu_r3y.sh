# W4: alpha in shared memory (mixed rows, when three stages still fit) vs in HBM
OUT=gpurun_out/r3y
mkdir -p $OUT
for rep in 1 2; do
  echo "== alpha in smem (default)" >> $OUT/t.txt
  SVMB200_PHASE_TIMERS=0 timeout 300 python tools/phase_probe.py W4:20000 >> $OUT/t.txt 2>&1
  echo "== alpha in HBM" >> $OUT/t.txt
  SVMB200_ALPHA_HBM=1 SVMB200_PHASE_TIMERS=0 timeout 300 python tools/phase_probe.py W4:20000 >> $OUT/t.txt 2>&1
done
SVMB200_PHASE_TIMERS=1 timeout 300 python tools/phase_probe.py W4:20000 >> $OUT/phase.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "mixed or W4" > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
