#!/bin/bash
for t in 8 1 2 3 16; do
  ACEDAG_TAIL_PARTS=$t timeout 200 python bench.py --no-cpu-baseline --no-e2e --no-naive --steps 40 > gpurun_out/t.log 2>&1
  echo "tail_parts=$t $(grep -o '"kernel_ms": [0-9.]*\|"ms_per_step": [0-9.]*' gpurun_out/t.log | tr '\n' ' ')"
done
