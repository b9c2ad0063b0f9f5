for pr in "0,0" "-1,0" "0,-1"; do
VSAOGM_BENCH_PRIO="$pr" VSAOGM_BENCH_PRIO_E2E="$pr" python bench.py --no-cpu-baseline --no-c5 > gpurun_out/r8b.json 2>/dev/null
python - <<PY
import json
d=json.load(open("gpurun_out/r8b.json")); print("prio $pr", "pipelined", d["ms_per_step"], "serial", d["serial"]["ms_per_step"], "e2e", d["e2e"]["ms_per_step"])
PY
done
for t in "entropy_kernel=2" "entropy_rw=14" "entropy_rw=32" "nd_bps=2"; do
python bench.py --no-cpu-baseline --no-c5 --tuning $t > gpurun_out/r8b.json 2>/dev/null
python - <<PY
import json
d=json.load(open("gpurun_out/r8b.json")); print("$t", "pipelined", d["ms_per_step"], "serial", d["serial"]["ms_per_step"], "e2e", d["e2e"]["ms_per_step"])
PY
done
