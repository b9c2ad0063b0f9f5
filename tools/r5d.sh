TAG=${1:-r5d}; KRE=${2:-k_nd_rowfft}
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-c5"
mkdir -p gpurun_out
$CMD > gpurun_out/plain_${TAG}.log 2>&1 || { tail gpurun_out/plain_${TAG}.log; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:"$KRE" -s 4 -c ${NCU_COUNT:-1} -o gpurun_out/prof_${TAG} $CMD > gpurun_out/ncu_full_${TAG}.log 2>&1
echo "full rc=$?"; tail -2 gpurun_out/ncu_full_${TAG}.log
