# session-3 evidence: smoke, all GPU tests, bench (+ reference arm), ncu launch list of the bench,
# DRAM traffic of the W5 solver, full captures of the W5 and W4 solvers
OUT=gpurun_out/r3q
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $OUT/gpu.txt 2>&1
timeout 300 python __graft_entry__.py smoke > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 2400 python -m pytest tests -m gpu -q --durations=15 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 1500 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
timeout 600 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:smo_ -c 1 --csv --log-file $OUT/traffic_W5.csv python tools/one_solve.py W5 3000 > $OUT/ncu_traffic.log 2>&1
python tools/traffic_json.py $OUT/traffic_W5.csv W5 $OUT/traffic_W5.json 3000 > /dev/null 2>&1
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-others --no-gd > $OUT/ncu_launch.log 2>&1
# (full captures in a separate call: two reports exceed gpurun's 64 MiB return limit)
