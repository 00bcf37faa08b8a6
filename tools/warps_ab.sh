#!/bin/bash
# A/B of the fp64 k2_horner warp count at cfg2 (kernel ms from bench.py phases)
for w in 16 20 24 16 20 24; do
  ACEDAG_HWARPS64=$w python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-naive 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('W=$w', round(r['kernel_ms'],4), 'ms frac', round(r['frac'],4), 'value', round(d['value']/1e6,2))"
done
