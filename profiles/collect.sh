#!/bin/bash
# Round evidence, run on the GPU box via gpurun (1 GPU):
#   gpurun -- 'bash profiles/collect.sh r01'
# For each workload: the bench command exits 0 without ncu first, then the
# launch list (gpu__time_duration per launch, --clock-control none) of the
# same command, then one `ncu --set full` capture of the k_spmv launch.
# Outputs land in gpurun_out/, summarised there by profiles/summarize.py
# (copy the .txt files into profiles/ to commit them).
set -u
tag=${1:-r01}
mkdir -p gpurun_out
for w in ${WORKLOADS:-st27_200 rmat24}; do
  cmd="python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --sub none"
  if $cmd > gpurun_out/${tag}_${w}_plain.log 2>&1; then
    ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
        --log-file gpurun_out/${tag}_${w}_launches.csv $cmd > gpurun_out/${tag}_${w}_ncu_list.log 2>&1
    ncu --set full --clock-control none --import-source on -k regex:k_spmv -s 2 -c 1 \
        -o gpurun_out/${tag}_${w}_spmv $cmd > gpurun_out/${tag}_${w}_ncu_full.log 2>&1
    # summarise on the box: full reports are ~20 MB each and gpurun copies back <= 64 MiB
    python profiles/summarize.py gpurun_out/${tag}_${w}_spmv.ncu-rep $w \
        gpurun_out/${tag}_ncu_full_${w}.txt > /dev/null 2>&1
    python profiles/summarize.py --launches gpurun_out/${tag}_${w}_launches.csv \
        gpurun_out/${tag}_launches_${w}.txt > /dev/null 2>&1
    [ "${KEEP_REP:-0}" = 1 ] || rm -f gpurun_out/${tag}_${w}_spmv.ncu-rep
  else
    echo "plain run of $w failed; not profiled" >&2
  fi
done
cp profiles/ncu_traffic.json gpurun_out/${tag}_ncu_traffic.json
ls -la gpurun_out
