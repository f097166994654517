mkdir -p gpurun_out/r2k
timeout 300 python __graft_entry__.py smoke > gpurun_out/r2k/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2k/smoke.log
timeout 2400 python -m pytest tests -m gpu -q --durations=25 > gpurun_out/r2k/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2k/pytest_gpu.log
timeout 1200 python bench.py > gpurun_out/r2k/bench.json 2> gpurun_out/r2k/bench.err; echo "bench rc=$?" >> gpurun_out/r2k/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/r2k/bench_ref.json 2> gpurun_out/r2k/bench_ref.err
timeout 300 python tools/probe_r2.py shards > gpurun_out/r2k/probe_shards.jsonl 2> gpurun_out/r2k/probe_shards.err
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:smo_ -c 1 --csv --log-file gpurun_out/r2k/traffic_W5.csv python tools/one_solve.py W5 3000 > gpurun_out/r2k/ncu_traffic.log 2>&1
python tools/traffic_json.py gpurun_out/r2k/traffic_W5.csv W5 gpurun_out/r2k/traffic_W5.json 3000 > /dev/null 2>&1
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2k/launches.csv \
    python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-others --no-gd > gpurun_out/r2k/ncu_launch.log 2>&1
