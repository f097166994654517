# W2 (smo_bincl): phase timers in shared memory
OUT=gpurun_out/r3x
mkdir -p $OUT
for rep in 1 2 3; do SVMB200_PHASE_TIMERS=0 timeout 300 python tools/phase_probe.py W2 >> $OUT/t.txt 2>&1; done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "binary or W2 or cluster or trajectory" > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
