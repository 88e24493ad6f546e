#!/bin/bash
# Experiment sweep (GPU box): k_spmv time per workload under env knobs.
#   bash tools/knob_sweep.sh "rmat24 mixed23" "" "CSR5G_YHINT=1" "CSR5G_XFRAC=0.75"
# Each configuration runs in its own process (the knobs are read once).
wls=$1; shift
for w in $wls; do
  for cfg in "$@"; do
    echo -n "[$cfg] "
    env $cfg python tools/plan_probe.py $w 2>&1 | tail -1
  done
done
