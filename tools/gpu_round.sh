#!/bin/bash
# One GPU session: tests, bench, launch list, DRAM traffic and full ncu captures of the
# solver and predict kernels.   Usage (under gpurun): bash tools/gpu_round.sh <tag>
TAG=${1:-r1}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 300 python __graft_entry__.py smoke > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-streamed --no-gd > $OUT/ncu_launch.log 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:smo_ -c 1 --csv --log-file $OUT/traffic_W2.csv python tools/one_solve.py W2 > $OUT/ncu_traffic.log 2>&1
python tools/traffic_json.py $OUT/traffic_W2.csv W2 $OUT/traffic_W2.json > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:smo_ -c 1 \
    -o $OUT/prof_smo python tools/one_solve.py W2 8000 > $OUT/ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:predict -c 1 \
    -o $OUT/prof_predict python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-streamed --no-gd > $OUT/ncu_predict.log 2>&1
