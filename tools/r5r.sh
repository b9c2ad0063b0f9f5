python -m pytest tests/test_gpu_parity.py -x -q -k "entropy" 2>&1 | tail -3
for t in "entropy_kernel=0" "entropy_kernel=2" "entropy_kernel=2,entropy_rw=16" "entropy_kernel=2,entropy_rw=25" "entropy_kernel=2,entropy_rw=40" "entropy_kernel=2,entropy_rw=10"; do
python bench.py --steps 30 --warmup 5 --no-cpu-baseline --tuning $t > gpurun_out/r5r_$t.json 2>/dev/null
python - <<PY
import json
d=json.load(open("gpurun_out/r5r_$t.json")); print("$t", "pipelined", d["ms_per_step"], "serial", d["serial"]["ms_per_step"], "e2e", d["e2e"]["ms_per_step"], "entropy", d["kernel_ms_per_step"]["entropy"], "c5", d["c5"]["ms_per_step"], d["c5"]["kernel_ms_per_step_rank0"]["entropy"])
PY
done
