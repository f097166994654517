mkdir -p gpurun_out/r2l
timeout 900 python -m pytest tests/test_bench_multirank.py tests/test_two_process.py -q > gpurun_out/r2l/pytest_multirank.log 2>&1; echo rc=$? >> gpurun_out/r2l/pytest_multirank.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:smo_ -c 1 -o gpurun_out/r2l/prof_smo_W4 python tools/one_solve.py W4 3000 > gpurun_out/r2l/ncu_w4.log 2>&1
ncu -i gpurun_out/r2l/prof_smo_W4.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r2l/w4_src.csv 2>/dev/null
