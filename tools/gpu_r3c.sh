# predict: exp variant x tile width; ncu of the predict kernel (v3) and of W4's solver (source hotspots)
OUT=gpurun_out/r3c
mkdir -p $OUT
timeout 600 python tools/predict_variants.py 3:128,3:256,0:256,3:256,3:128 --no-peaks > $OUT/predict_variants.jsonl 2> $OUT/predict_variants.err
timeout 600 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -x -k "predict" > $OUT/pytest_predict.log 2>&1; echo rc=$? >> $OUT/pytest_predict.log
SVMB200_PREDICT_BN=256 timeout 600 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -x -k "predict" > $OUT/pytest_predict_bn256.log 2>&1; echo rc=$? >> $OUT/pytest_predict_bn256.log
for bn in 128 256; do
SVMB200_PREDICT_BN=$bn timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_predict_tc -c 1 \
    -o $OUT/prof_predict_v3_bn$bn python tools/predict_one.py 37888 284028 3 > $OUT/ncu_predict_bn$bn.log 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:smo_ -c 1 \
    -o $OUT/prof_smo_W4 python tools/one_solve.py W4 3000 > $OUT/ncu_w4.log 2>&1
