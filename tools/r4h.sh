mkdir -p gpurun_out
python -m pytest tests/test_gpu_nudecode.py -x -q > gpurun_out/r4h_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r4h_tests.log
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-c5 > gpurun_out/r4h_bench.json 2> gpurun_out/r4h_bench.err
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-c5"
$CMD > gpurun_out/plain_r4h.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_r4h.csv $CMD > gpurun_out/ncu_launch_r4h.log 2>&1
