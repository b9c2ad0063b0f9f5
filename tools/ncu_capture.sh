#!/bin/bash
# Profiling recipe (B200_PROFILING.md): plain run, then the launch list, then one
# --set full capture of the hot kernels.  Usage (on the gpurun box):
#   bash tools/ncu_capture.sh <tag> [kernel-regex]
TAG=${1:-r01}
KRE=${2:-"k_encode_pairs|k_decode_gemm|k_entropy|k_table|k_reduce|k_commit_norms"}
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-c5"
mkdir -p gpurun_out
$CMD > gpurun_out/plain_$TAG.log 2>&1 || { echo "plain run failed"; tail gpurun_out/plain_$TAG.log; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1
echo "launch-list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"$KRE" -s 7 -c ${NCU_COUNT:-8} \
    -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo "full rc=$?"
tail -3 gpurun_out/ncu_full_$TAG.log
