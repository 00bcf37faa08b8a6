#!/bin/bash
# A/B: bench each library variant twice, interleaved.  usage (on the GPU
# box): tools/ab.sh base variant -- with abtest/base.so and abtest/variant.so
# built here (drop abtest/ from .gpurunignore for the call).
for rep in 1 2; do
for v in "$@"; do
  cp abtest/$v.so paper_2202_04140_b200/libacedag_b200.so
  timeout 200 python bench.py --no-cpu-baseline --no-e2e --no-naive --steps 40 > gpurun_out/ab_$v.log 2>&1
  echo "$v $(grep -o '"kernel_ms": [0-9.]*' gpurun_out/ab_$v.log) $(grep -o '"value": [0-9.]*' gpurun_out/ab_$v.log | head -1)"
done
done
