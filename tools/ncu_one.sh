#!/bin/bash
# One --set full capture of one kernel under the bench command (B200_PROFILING.md recipe):
#   bash tools/ncu_one.sh <tag> <kernel-regex> [env assignments...]
# Runs the bench plainly first; captures only if that exits 0.
TAG=$1; KRE=$2; shift 2
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
mkdir -p gpurun_out
env "$@" $CMD > gpurun_out/plain_$TAG.log 2>&1 || { echo "plain run failed"; tail gpurun_out/plain_$TAG.log; exit 1; }
env "$@" ncu --set full --clock-control none --import-source on -k regex:"$KRE" -s 3 -c ${NCU_COUNT:-1} \
    -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_full_$TAG.log 2>&1
echo "full rc=$?"
tail -2 gpurun_out/ncu_full_$TAG.log
