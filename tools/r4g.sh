mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/r4g_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r4g_tests.log
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-c5"
$CMD > gpurun_out/plain_r4g.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"k_nd_rowfft|k_nd_spread" -s 4 -c 2 -o gpurun_out/prof_r4g $CMD > gpurun_out/ncu_full_r4g.log 2>&1
echo "rc=$?"
