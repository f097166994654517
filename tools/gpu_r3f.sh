# exchange skew diagnostic: per-CTA row-pass start / publish timestamps
OUT=gpurun_out/r3f
mkdir -p $OUT
SVMB200_PHASE_TIMERS=0 SVMB200_SKEW_TS=3000 timeout 600 python tools/phase_probe.py W4:3000 W5:1500 W5@125000:3000 W3:3000 > $OUT/skew.txt 2>&1
