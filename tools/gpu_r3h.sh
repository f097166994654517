# predict default = variant 5 (row factor): tests; the default bench line
OUT=gpurun_out/r3h
mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -x -k "predict" > $OUT/pytest_predict.log 2>&1; echo rc=$? >> $OUT/pytest_predict.log
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > $OUT/gpu.txt 2>&1
timeout 1500 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
