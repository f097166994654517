#!/bin/bash
for cfg in "-1 4" "0 2" "0 4" "0 8"; do set -- $cfg
  echo "== DIRECTPOLL=$1 NREP=$2"; SVMB200_DIRECTPOLL=$1 SVMB200_NREP=$2 timeout 300 python tools/phase_probe.py W2 2>&1 | grep -v "^\[svmb200\]"
done
