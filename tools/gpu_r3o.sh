# W4: mixed-rows-only instantiation, 512 vs 448 consumer threads (96 vs 128 registers)
OUT=gpurun_out/r3o
mkdir -p $OUT
for rep in 1 2; do
  for nt in 512 448; do
    echo "== NT=$nt" >> $OUT/t.txt
    SVMB200_NT=$nt SVMB200_PHASE_TIMERS=0 timeout 300 python tools/phase_probe.py W4:20000 >> $OUT/t.txt 2>&1
  done
  echo "== general kernel" >> $OUT/t.txt
  SVMB200_NO_SPECIALISE=1 SVMB200_PHASE_TIMERS=0 timeout 300 python tools/phase_probe.py W4:20000 >> $OUT/t.txt 2>&1
done
SVMB200_NT=448 SVMB200_PHASE_TIMERS=1 timeout 300 python tools/phase_probe.py W4:20000 >> $OUT/phase448.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "mixed or W4 or consumer_warp" > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
