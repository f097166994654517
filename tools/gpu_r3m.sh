# 16-warp kernels without the binary-resident / row-cache paths (fewer spills): timings, tests
OUT=gpurun_out/r3m
mkdir -p $OUT
for rep in 1 2; do
  SVMB200_PHASE_TIMERS=0 timeout 300 python tools/phase_probe.py W4:20000 W5@125000:5000 W3:0 >> $OUT/t.txt 2>&1
done
SVMB200_PHASE_TIMERS=1 timeout 300 python tools/phase_probe.py W4:20000 >> $OUT/phase.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_boundary.py tests/test_wss2_gpu.py tests/test_shrink_gpu.py -q -x > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
