#!/bin/bash
for cfg in "4 8" "4 4" "4 16" "2 16" "2 8" "1 32"; do set -- $cfg
  echo "== RPT=$1 KC=$2"; SVMB200_RPT=$1 SVMB200_KC=$2 timeout 300 python tools/phase_probe.py W4:20000 W5:2000 2>&1 | grep -v "^\[svmb200\]"
done
