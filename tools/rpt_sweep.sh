#!/bin/bash
# RPT sweep for the persistent kernel on one workload prefix
for r in 1 2 4; do SVMB200_RPT=$r timeout 300 python tools/phase_probe.py "$@" 2>&1 | sed "s/^/rpt$r /"; done
