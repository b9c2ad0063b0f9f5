#!/bin/bash
# decode GEMM variant sweep: per-kernel times from bench.py
run() { env "$@" python bench.py --steps 40 --warmup 3 --no-cpu-baseline 2>/dev/null | \
  python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernel_ms_per_step']; print('$*', 'ms/step', d['ms_per_step'], 'gemm', k['decode_gemm'], 'frac', d['decode_roofline']['frac'], 'entropy', k['entropy'], 'tableA', k['table_A'], 'enc', k['encode'], 'clk', d['clocks']['sm_mhz'])"; }
run VSAOGM_GEMM=1cta
for bn in 256 224 192; do run VSAOGM_GEMM_BN=$bn; done
run X=default
