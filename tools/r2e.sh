python -m pytest tests -m gpu -x -q -k "entropy" > gpurun_out/r2e_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2e_tests.log
python tools/ent_bench.py "" "entropy_kernel=1" "entropy_rw=16" "entropy_rw=40" > gpurun_out/r2e_ent.jsonl 2>&1
python tools/enc_sweep.py "enc_x2=4" "enc_x2=4,enc_pairs_split=1" "enc_x2=4,enc_pairs_split=1,enc_pairs_npoly=2" "enc_x2=4,enc_pairs_split=1,enc_pairs_npoly=6" > gpurun_out/r2e_enc.jsonl 2>&1
python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-c5 > gpurun_out/r2e_bench.json 2> gpurun_out/r2e_bench.err
