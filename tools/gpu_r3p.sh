# dense-streamed-only instantiation (W5 and its shards) vs the general kernel
OUT=gpurun_out/r3p
mkdir -p $OUT
for rep in 1 2; do
  echo "== dense-only (default)" >> $OUT/t.txt
  SVMB200_PHASE_TIMERS=0 timeout 300 python tools/phase_probe.py W5@125000:5000:nocache W5:1500 W4:20000 >> $OUT/t.txt 2>&1
  echo "== general kernel" >> $OUT/t.txt
  SVMB200_NO_SPECIALISE=1 SVMB200_PHASE_TIMERS=0 timeout 300 python tools/phase_probe.py W5@125000:5000:nocache W5:1500 W4:20000 >> $OUT/t.txt 2>&1
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "W5 or partition or consumer or mixed_rows_only or wide or dup" > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
