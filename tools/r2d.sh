python tools/ent_bench.py "" "entropy_kernel=1" "entropy_rw=16" "entropy_rw=64" > gpurun_out/r2d_ent.jsonl 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_entropy_stream" -s 2 -c 1 -o gpurun_out/prof_r2d_ent python tools/ent_bench.py "" > gpurun_out/ncu_r2d_ent.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_encode_pairs" -s 2 -c 1 -o gpurun_out/prof_r2d_enc python tools/enc_sweep.py "" > gpurun_out/ncu_r2d_enc.log 2>&1
echo done
