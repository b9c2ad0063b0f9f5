#!/bin/bash
# Encode MUFU/polynomial split sweep: per-kernel times from bench.py for each VSAOGM_ENC_NPOLY
for np in ${@:-0 1 2 3}; do
  VSAOGM_ENC_NPOLY=$np python bench.py --steps 40 --warmup 3 --no-cpu-baseline 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernel_ms_per_step']; print('npoly=$np', 'ms/step', d['ms_per_step'], 'encode', k['encode'], 'gemm', k['decode_gemm'], 'tableA', k['table_A'], 'entropy', k['entropy'], 'reduce', k['reduce'], 'frac', d['roofline']['frac'], 'clk', d['clocks']['sm_mhz'])"
done
