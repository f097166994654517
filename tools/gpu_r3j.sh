# exchange at multi-GPU record counts, simulated on one GPU (SVMB200_XCH_DUP = k: every record
# in k slots): one warp polling vs all consumer warps polling
OUT=gpurun_out/r3j
mkdir -p $OUT
for dup in 1 2 4 8; do
  for wp in 0 1; do
    echo "== dup=$dup wide_poll=$wp" >> $OUT/xchdup.txt
    SVMB200_XCH_DUP=$dup SVMB200_WIDE_POLL=$wp SVMB200_PHASE_TIMERS=1 timeout 300 python tools/phase_probe.py W5@125000:5000 W4:10000 >> $OUT/xchdup.txt 2>&1
  done
done
SVMB200_XCH_DUP=8 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "wide_poll or partition or trajectory" > $OUT/pytest_dup8.log 2>&1; echo rc=$? >> $OUT/pytest_dup8.log
