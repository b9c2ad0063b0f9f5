# Round-2 re-entry measurement: GPU tests, bench, per-config record, launch list + full capture.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r4a_smi.txt 2>&1
python -m pytest tests -m gpu -x -q > gpurun_out/r4a_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r4a_tests.log
python bench.py --steps 30 --warmup 5 > gpurun_out/r4a_bench.json 2> gpurun_out/r4a_bench.err
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r4a_ref.json 2> gpurun_out/r4a_ref.err
python tools/config_bench.py r4a > gpurun_out/r4a_configs.log 2>&1
cp profiles/r4a_configs.json* gpurun_out/ 2>/dev/null
bash tools/ncu_capture.sh r4a "k_nu_|k_decode_gemm|k_entropy|k_table|k_commit" > gpurun_out/r4a_ncu.log 2>&1
