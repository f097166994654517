# final library: smoke, all GPU tests, one W4 full ncu capture summarised on the box
# (the report itself exceeds gpurun's 64 MiB return limit)
OUT=gpurun_out/r3s
mkdir -p $OUT
timeout 300 python __graft_entry__.py smoke > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 2400 python -m pytest tests -m gpu -q --durations=15 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
SVMB200_PHASE_TIMERS=1 timeout 300 python tools/phase_probe.py W4:20000 W5@125000:5000:nocache W3:0 > $OUT/phase.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:smo_ -c 1 \
    -o /tmp/prof_smo_W4 python tools/one_solve.py W4 3000 > $OUT/ncu_full_w4.log 2>&1
ncu -i /tmp/prof_smo_W4.ncu-rep --page details --csv > $OUT/ncu_W4_details.csv 2>&1
python tools/ncu_line_hot.py /tmp/prof_smo_W4.ncu-rep 50 > $OUT/ncu_W4_line_hotspots.txt 2>&1
python tools/ncu_sass_hot.py /tmp/prof_smo_W4.ncu-rep 40 > $OUT/ncu_W4_sass_hotspots.txt 2>&1
ls -la /tmp/prof_smo_W4.ncu-rep >> $OUT/ncu_full_w4.log 2>&1
