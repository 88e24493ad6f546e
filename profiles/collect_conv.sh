#!/bin/bash
# Converter evidence (GPU box, 1 GPU):  gpurun -- 'bash profiles/collect_conv.sh r01d'
# One plain run of tools/conv_probe.py per workload (must exit 0), then one
# `ncu --set full` capture of the last build's converter kernels, summarised
# on the box (profiles/summarize.py --kernels) so only text comes back.
set -u
tag=${1:-r01}
mkdir -p gpurun_out
for w in ${WORKLOADS:-st27_200 rmat24}; do
  cmd="python tools/conv_probe.py $w"
  if $cmd > gpurun_out/${tag}_${w}_conv_plain.log 2>&1; then
    ncu --set full --clock-control none \
        -k regex:"k_rowscan|k_tile_ptr|k_desc_transpose|k_eo|k_tile_work|k_locality|k_warp_bounds" \
        -c 10 -o gpurun_out/${tag}_${w}_conv $cmd > gpurun_out/${tag}_${w}_conv_ncu.log 2>&1
    python profiles/summarize.py --kernels gpurun_out/${tag}_${w}_conv.ncu-rep $w \
        gpurun_out/${tag}_ncu_conv_${w}.txt > /dev/null 2>&1
    [ "${KEEP_REP:-0}" = 1 ] || rm -f gpurun_out/${tag}_${w}_conv.ncu-rep
  else
    echo "plain conversion run of $w failed; not profiled" >&2
  fi
done
