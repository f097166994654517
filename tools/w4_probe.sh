#!/bin/bash
# W4 per-phase probe: RBF vs linear (exp cost), RPT variants, W5 for comparison.
mkdir -p gpurun_out/w4
{
for spec in W4:20000 W4:20000:lin W5:2000 W5:2000:lin; do
  SVMB200_PHASE_TIMERS=1 timeout 300 python tools/phase_probe.py $spec 2>&1 | tail -2
done
for r in 2 1; do echo "== RPT=$r"; SVMB200_RPT=$r SVMB200_PHASE_TIMERS=1 timeout 300 python tools/phase_probe.py W4:20000 2>&1 | tail -2; done
} > gpurun_out/w4/probe.txt 2>&1
