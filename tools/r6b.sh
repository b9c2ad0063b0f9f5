for t in "nd_bps=0" "nd_bps=2" "entropy_rw=16" "entropy_rw=32"; do
python bench.py --steps 60 --warmup 5 --no-cpu-baseline --no-c5 --tuning $t > gpurun_out/r6b_$t.json 2>/dev/null
python - <<PY
import json
d=json.load(open("gpurun_out/r6b_$t.json")); print("$t", "pipelined", d["ms_per_step"], "serial", d["serial"]["ms_per_step"], "e2e", d["e2e"]["ms_per_step"], d["kernel_ms_per_step"]["nd_rowfft"], d["kernel_ms_per_step"]["entropy"])
PY
done
