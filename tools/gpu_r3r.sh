# dense-only instantiation with alpha in shared memory (the P = 8 shard's plan): test, timings
OUT=gpurun_out/r3r
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "dense_only or partition or trajectory or W5" > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
for rep in 1 2; do
  echo "== dense-only (default)" >> $OUT/t.txt
  SVMB200_PHASE_TIMERS=0 timeout 300 python tools/phase_probe.py W5@125000:5000:nocache W5@250000:3000:nocache >> $OUT/t.txt 2>&1
  echo "== general kernel" >> $OUT/t.txt
  SVMB200_NO_SPECIALISE=1 SVMB200_PHASE_TIMERS=0 timeout 300 python tools/phase_probe.py W5@125000:5000:nocache W5@250000:3000:nocache >> $OUT/t.txt 2>&1
  for wp in 0 1; do
    echo "== dup=8 wide_poll=$wp (nocache shard)" >> $OUT/t.txt
    SVMB200_XCH_DUP=8 SVMB200_WIDE_POLL=$wp SVMB200_PHASE_TIMERS=0 timeout 300 python tools/phase_probe.py W5@125000:5000:nocache >> $OUT/t.txt 2>&1
  done
done
