mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-c5"
$CMD > gpurun_out/plain_r4e.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_nd_" -s 8 -c 4 -o gpurun_out/prof_r4e $CMD > gpurun_out/ncu_full_r4e.log 2>&1
echo "rc=$?"
