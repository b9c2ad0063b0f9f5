# quick check after a kernel change: NUFFT tests + short bench + launch list
TAG=${1:-r5b}
mkdir -p gpurun_out
python -m pytest tests/test_gpu_nudecode.py tests/test_gpu_parity.py -x -q > gpurun_out/${TAG}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_tests.log
tail -3 gpurun_out/${TAG}_tests.log
python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-c5"
$CMD > gpurun_out/plain_${TAG}.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_launch_${TAG}.log 2>&1
python - <<PY
import json
d=json.load(open("gpurun_out/${TAG}_bench.json"))
print("pipelined", d["ms_per_step"], "serial", d["serial"]["ms_per_step"], "e2e", d["e2e"]["ms_per_step"], "c5", d.get("c5",{}).get("ms_per_step"))
print(d["kernel_ms_per_step"])
PY
