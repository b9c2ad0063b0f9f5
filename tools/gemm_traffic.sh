#!/bin/bash
# GEMM-only ncu DRAM traffic check (one launch) after a plain run
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/plain_gt.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:k_decode_gemm2 -s 3 -c 2 $CMD 2>&1 | grep -E "dram__|gpu__time|tensor|cycles_elapsed"
