# wide poll as a noinline function: single-GPU timings (auto = off at 148 records) and at 8x records
OUT=gpurun_out/r3k
mkdir -p $OUT
for rep in 1 2; do
  echo "== default" >> $OUT/xch.txt
  SVMB200_PHASE_TIMERS=0 timeout 300 python tools/phase_probe.py W4:20000 W5@125000:5000 W5:1500 W3:0 >> $OUT/xch.txt 2>&1
  for wp in 0 1; do
    echo "== dup=8 wide_poll=$wp" >> $OUT/xch.txt
    SVMB200_XCH_DUP=8 SVMB200_WIDE_POLL=$wp SVMB200_PHASE_TIMERS=0 timeout 300 python tools/phase_probe.py W5@125000:5000 W4:10000 >> $OUT/xch.txt 2>&1
  done
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "wide_poll or partition" > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
