set -x
python -m pytest tests -m gpu -x -q -k "entropy or encode or quadrant or pipeline or c1 or c2" > gpurun_out/r2c_tests_focus.log 2>&1
echo "focus rc=$?" >> gpurun_out/r2c_tests_focus.log
python tools/enc_sweep.py "enc_x2=2" "enc_x2=4,enc_pairs_npoly=0" "enc_x2=4,enc_pairs_npoly=2" "enc_x2=4,enc_pairs_npoly=4" "enc_x2=4,enc_pairs_npoly=6" "enc_x2=4,enc_pairs_npoly=8" "enc_x2=4,enc_pairs_npoly=2,enc_pairs_minb=4" "enc_x2=4,enc_pairs_npoly=4,enc_x2_waves=2" "enc_x2=4,enc_pairs_npoly=4,enc_x2_waves=8" > gpurun_out/r2c_encsweep.jsonl 2>&1
python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/r2c_bench.json 2> gpurun_out/r2c_bench.err
