# straggler hypothesis: the exp slow phase (~5e-5 of calls, ~0.4 per CTA per iteration on W4)
# on the critical path of every exchange.  Timing with the slow phase skipped (wrong values,
# diagnostic only) against the normal kernel.
OUT=gpurun_out/r3d
mkdir -p $OUT
for f in 0 1 0 1; do
  echo "== fast_only=$f" >> $OUT/fastonly.txt
  SVMB200_DBG_FAST_ONLY=$f SVMB200_PHASE_TIMERS=1 timeout 300 python tools/phase_probe.py W4:20000 W5@125000:5000 W5:1500 >> $OUT/fastonly.txt 2>&1
done
