# predict: accumulator handed back after the last TMEM load of a tile (before its compute)
OUT=gpurun_out/r3u
mkdir -p $OUT
timeout 900 python tools/predict_variants.py 5:256,5:128,5:256,5:128 > $OUT/predict_variants.jsonl 2> $OUT/predict_variants.err
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -x -k "predict" > $OUT/pytest_predict.log 2>&1; echo rc=$? >> $OUT/pytest_predict.log
