#!/bin/bash
for rr in 0 1; do for n in 1 2 4; do
  echo "== RECROWS=$rr NREP=$n"; SVMB200_RECROWS=$rr SVMB200_NREP=$n timeout 300 python tools/phase_probe.py "$@" 2>&1 | tail -2
done; done
