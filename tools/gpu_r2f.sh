mkdir -p gpurun_out/r2f
timeout 600 python -m pytest tests/test_shrink_gpu.py -q -x > gpurun_out/r2f/pytest_shrink.log 2>&1; echo rc=$? >> gpurun_out/r2f/pytest_shrink.log
SVMB200_SHRINK_LOG=1 timeout 600 python tools/probe_r2.py shrink5 > gpurun_out/r2f/probe_shrink5.jsonl 2> gpurun_out/r2f/shrink5.log
timeout 300 python tools/probe_r2.py iters > gpurun_out/r2f/probe_iters.jsonl 2> gpurun_out/r2f/probe_iters.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_predict_tc -c 1 -o gpurun_out/r2f/prof_predict_W5 python tools/predict_one.py 37888 284028 > gpurun_out/r2f/ncu_predict.log 2>&1
