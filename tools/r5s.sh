python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python bench.py --steps 60 --warmup 5 --no-cpu-baseline > gpurun_out/r5s_bench.json 2>/dev/null
python - <<PY
import json
d=json.load(open("gpurun_out/r5s_bench.json")); print("pipelined", d["ms_per_step"], "serial", d["serial"]["ms_per_step"], "e2e", d["e2e"]["ms_per_step"], "entropy", d["kernel_ms_per_step"]["entropy"], "c5", d["c5"]["ms_per_step"], d["c5"]["kernel_ms_per_step_rank0"]["entropy"])
PY
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-c5"
ncu --set full --clock-control none --import-source on -k regex:"k_entropy_cols" -s 4 -c 1 -o gpurun_out/prof_r5s $CMD > gpurun_out/ncu_full_r5s.log 2>&1; tail -1 gpurun_out/ncu_full_r5s.log
