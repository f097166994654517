# predict defaults (split exp, BN 256): tests, repeated timing of both tile widths
OUT=gpurun_out/r3e
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -x -k "predict" > $OUT/pytest_predict.log 2>&1; echo rc=$? >> $OUT/pytest_predict.log
timeout 900 python tools/predict_variants.py 3:256,3:128,3:256,3:128,0:256 > $OUT/predict_variants.jsonl 2> $OUT/predict_variants.err
