python -m pytest tests -m gpu -x -q -k "entropy or c1 or c2" > gpurun_out/r2j_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2j_tests.log
python tools/ent_bench.py "" "entropy_rw=8" "entropy_rw=12" "entropy_rw=24" > gpurun_out/r2j_ent.jsonl 2>&1
CFG=C5 python tools/ent_bench.py "" "entropy_rw=32" > gpurun_out/r2j_ent_c5.jsonl 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_entropy_stream" -s 2 -c 1 -o gpurun_out/prof_r2j_ent python tools/ent_bench.py "" > gpurun_out/ncu_r2j_ent.log 2>&1
