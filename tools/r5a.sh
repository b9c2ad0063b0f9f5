TAG=${1:-r5z}
# Round-2 session-4 baseline: full GPU suite, bench (both arms), launch list, one full ncu capture of every hot kernel.
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_gpu_tests.log
python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_ref.json 2> gpurun_out/${TAG}_ref.err; echo "ref rc=$?"
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-c5"
$CMD > gpurun_out/plain_${TAG}.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_${TAG}.csv $CMD > gpurun_out/ncu_launch_${TAG}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_nu_bin|k_nu_spread_tiles|k_nu_rowfft|k_nu_colfft|k_nu_interp|k_commit_norms|k_nd_strength|k_nd_spread|k_nd_colfft|k_nd_rowfft|k_entropy_cols" -s 22 -c 11 -o gpurun_out/prof_${TAG} $CMD > gpurun_out/ncu_full_${TAG}.log 2>&1
echo "full rc=$?"; tail -2 gpurun_out/ncu_full_${TAG}.log
python tools/config_bench.py ${TAG} > gpurun_out/${TAG}_configs.log 2>&1; echo "configs rc=$?"
