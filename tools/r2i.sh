python -m pytest tests -m gpu -x -q -k "entropy or quadrant or c1 or c2 or pipeline" > gpurun_out/r2i_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2i_tests.log
python tools/ent_bench.py "" "entropy_rw=24" > gpurun_out/r2i_ent.jsonl 2>&1
CFG=C5 python tools/ent_bench.py "" > gpurun_out/r2i_ent_c5.jsonl 2>&1
CFG=C4 python tools/enc_sweep.py "" > gpurun_out/r2i_enc.jsonl 2>&1
python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-c5 > gpurun_out/r2i_bench.json 2> gpurun_out/r2i_bench.err
