mkdir -p gpurun_out/l2
for k in 0 32 64 80 96 110; do echo "== KEEP=$k"; SVMB200_L2_KEEP_MB=$k SVMB200_PHASE_TIMERS=1 timeout 300 python tools/phase_probe.py W4:20000 W5:2000 W3:0 2>&1 | grep -v "^\[svmb200\] cycles" ; SVMB200_L2_KEEP_MB=$k SVMB200_PHASE_TIMERS=1 timeout 300 python tools/phase_probe.py W4:20000 2>&1 | grep "cycles" | tail -1; done > gpurun_out/l2/sweep.txt 2>&1
