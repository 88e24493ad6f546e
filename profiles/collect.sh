#!/bin/bash
# Round evidence, run on the GPU box via gpurun (1 GPU):
#   gpurun -- 'bash profiles/collect.sh r01'
# For each workload: the bench command exits 0 without ncu first, then the
# launch list (gpu__time_duration per launch, --clock-control none) of the
# same command, then one `ncu --set full` capture of the k_spmv launch.
# Outputs land in gpurun_out/; profiles/summarize.py turns them into the
# committed summaries.
set -u
tag=${1:-r01}
mkdir -p gpurun_out
for w in ${WORKLOADS:-st27_200 rmat24}; do
  cmd="python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline"
  if $cmd > gpurun_out/${tag}_${w}_plain.log 2>&1; then
    ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
        --log-file gpurun_out/${tag}_${w}_launches.csv $cmd > gpurun_out/${tag}_${w}_ncu_list.log 2>&1
    ncu --set full --clock-control none --import-source on -k regex:k_spmv -s 2 -c 1 \
        -o gpurun_out/${tag}_${w}_spmv $cmd > gpurun_out/${tag}_${w}_ncu_full.log 2>&1
  else
    echo "plain run of $w failed; not profiled" >&2
  fi
done
ls -la gpurun_out
