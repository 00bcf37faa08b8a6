#!/bin/bash
# A/B of k2_horner staging at cfg2: ACEDAG_TMA=0 (k_tile_seeds pass) vs 1 (TMA from A)
for t in 0 1 0 1; do
  ACEDAG_TMA=$t python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-naive 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('TMA=$t step', round(d['ms_per_step'],4), 'k2', round(r['kernel_ms'],4), 'prep', round(r['phases_ms']['prep_ms'],4), 'value', round(d['value']/1e6,2))"
done
