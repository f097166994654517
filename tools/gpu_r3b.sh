# predict epilogue variants (+ cuBLAS TF32/BF16 peaks), W4 with barrier B after the exps, parity subset
OUT=gpurun_out/r3b
mkdir -p $OUT
timeout 600 python tools/predict_variants.py 0,3,4 > $OUT/predict_variants.jsonl 2> $OUT/predict_variants.err
SVMB200_PHASE_TIMERS=1 timeout 300 python tools/phase_probe.py W4:20000 W3:0 W5:2000 > $OUT/phase.txt 2>&1
SVMB200_PHASE_TIMERS=0 timeout 300 python tools/phase_probe.py W4:20000 W3:0 > $OUT/noph.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_boundary.py tests/test_wss2_gpu.py tests/test_shrink_gpu.py -q -x > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
