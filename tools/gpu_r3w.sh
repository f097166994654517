# W4: 448 consumer threads with 4 rows each (8 exp chains per thread, 128 registers)
OUT=gpurun_out/r3w
mkdir -p $OUT
for rep in 1 2; do
  echo "== default (512 x RPT 2)" >> $OUT/t.txt
  SVMB200_PHASE_TIMERS=0 timeout 300 python tools/phase_probe.py W4:20000 >> $OUT/t.txt 2>&1
  echo "== 448 x RPT 4" >> $OUT/t.txt
  SVMB200_NT=448 SVMB200_RPT=4 SVMB200_PHASE_TIMERS=0 timeout 300 python tools/phase_probe.py W4:20000 >> $OUT/t.txt 2>&1
done
SVMB200_NT=448 SVMB200_RPT=4 SVMB200_PHASE_TIMERS=1 timeout 300 python tools/phase_probe.py W4:20000 >> $OUT/phase.txt 2>&1
SVMB200_NT=448 SVMB200_RPT=4 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "mixed_rows_parity or mixed_rows_only" > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
