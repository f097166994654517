#!/bin/bash
# One GPU session (round 2): smoke, GPU tests, the W5 headline bench, the ncu launch list
# of the bench, DRAM traffic and a full ncu capture of the W5 streamed solver.
#   bash tools/gpu_round2.sh <tag> [what...]   what: smoke tests bench launches traffic full
TAG=${1:-r2}
shift
WHAT=${@:-smoke tests bench traffic full}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/smi.txt 2>&1
for w in $WHAT; do
case $w in
smoke) timeout 300 python __graft_entry__.py smoke > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log ;;
tests) timeout 2400 python -m pytest tests -m gpu -q --durations=25 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log ;;
testsq) timeout 1200 python -m pytest tests -m gpu -q -x --durations=10 --deselect tests/test_gpu_fullsize.py > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log ;;
bench) timeout 1200 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err ;;
benchref) timeout 600 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err ;;
launches) timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-others --no-gd > $OUT/ncu_launch.log 2>&1 ;;
traffic) timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:smo_ -c 1 --csv --log-file $OUT/traffic_W5.csv python tools/one_solve.py W5 3000 > $OUT/ncu_traffic.log 2>&1
    python tools/traffic_json.py $OUT/traffic_W5.csv W5 $OUT/traffic_W5.json 3000 > /dev/null 2>&1 ;;
full) timeout 900 ncu --set full --clock-control none --import-source on -k regex:smo_ -c 1 \
    -o $OUT/prof_smo_W5 python tools/one_solve.py W5 300 > $OUT/ncu_full.log 2>&1 ;;
esac
done
for w in $WHAT; do
if [ "$w" = "sanitize" ]; then
  mkdir -p $OUT/sanitizer
  for c in bincl cluster global cache wss2 predict_tc predict_exact gd; do
    for tool in memcheck racecheck synccheck; do
      timeout 600 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_cases.py $c 20 \
        > $OUT/sanitizer/${c}_${tool}.log 2>&1
      echo "rc=$?" >> $OUT/sanitizer/${c}_${tool}.log
    done
  done
fi
done
