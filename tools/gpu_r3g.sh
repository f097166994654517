# predict: row-factor variant (5) and BN 128 with 4 accumulators
OUT=gpurun_out/r3g
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -x -k "predict" > $OUT/pytest_predict.log 2>&1; echo rc=$? >> $OUT/pytest_predict.log
SVMB200_PREDICT_EXP=5 timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "predict" > $OUT/pytest_predict_v5.log 2>&1; echo rc=$? >> $OUT/pytest_predict_v5.log
timeout 900 python tools/predict_variants.py 3:256,5:256,3:128,5:128,3:256,5:256,3:128,5:128 --no-peaks > $OUT/predict_variants.jsonl 2> $OUT/predict_variants.err
