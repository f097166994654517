# round-2 final evidence: smoke, GPU tests, bench (+ reference arm), ncu launch list of the bench,
# DRAM traffic and a full capture of the W5 solver, sanitizer on the shrink / replay kernels
OUT=gpurun_out/r2q
mkdir -p $OUT
timeout 300 python __graft_entry__.py smoke > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 2400 python -m pytest tests -m gpu -q --durations=25 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 1200 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
timeout 600 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
    -k regex:smo_ -c 1 --csv --log-file $OUT/traffic_W5.csv python tools/one_solve.py W5 3000 > $OUT/ncu_traffic.log 2>&1
python tools/traffic_json.py $OUT/traffic_W5.csv W5 $OUT/traffic_W5.json 3000 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:smo_ -c 1 \
    -o $OUT/prof_smo_W5 python tools/one_solve.py W5 300 > $OUT/ncu_full.log 2>&1
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-others --no-gd > $OUT/ncu_launch.log 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 600 compute-sanitizer --tool $tool --print-limit 20 python -c "
import sys; sys.path.insert(0, '.')
import numpy as np, paper_2311_14908_b200 as S
from oracle import oracle as O
from tests.test_oracle_qp import _rand_problem
X, y, C, k = _rand_problem(1)
S.svm_train_ex(X, y, C, k, 0.5, 1e-3, shrink_window=3)
from gen import workloads as W
w = W.get('W5'); X, y = w.train(1500)
part = O.train(X, y, w.C, w.kernel, w.gamma, w.tol, max_iter=800)
S.svm_train_ex(X, y, w.C, w.kernel, w.gamma, w.tol, shrink_window=20, alpha0=part.alpha, f0=part.f, max_iter=60)
print('shrink ok')" > $OUT/sanitizer_shrink_$tool.log 2>&1
  echo "rc=$?" >> $OUT/sanitizer_shrink_$tool.log
done
