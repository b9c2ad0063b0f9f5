for t in "nd_bps=0" "nd_bps=2" "entropy_rw=14" "entropy_rw=32" "entropy_kernel=2" "pdl=0"; do
python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-c5 --tuning $t > gpurun_out/r7d.json 2>/dev/null
python - <<PY
import json
d=json.load(open("gpurun_out/r7d.json")); print("$t", "pipelined", d["ms_per_step"], "serial", d["serial"]["ms_per_step"], "e2e", d["e2e"]["ms_per_step"])
PY
done
