#!/bin/bash
# generic knob sweep: each argument is an env assignment list, e.g. "VSAOGM_ENC_MINB=8"
# prints the pipelined ms/step (bench headline), the serial ms/step and the serial per-kernel times
for cfg in "$@"; do
  env $cfg python bench.py --steps 40 --warmup 3 --no-cpu-baseline 2>/dev/null | \
  python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernel_ms_per_step']; print('$cfg', 'ms/step', d['ms_per_step'], 'serial', d['serial']['ms_per_step'], ' '.join(f'{a}={b:.4f}' for a,b in k.items() if b), 'clk', d['clocks']['sm_mhz'])"
done
