#!/bin/bash
# quick K2 check: cfg2 parity subset + 2 bench runs (fp64) + fp32
python -m pytest tests/test_gpu_parity.py -q -x -k "cfg2 or batch or fp32 or groups or variants" > gpurun_out/q.log 2>&1; tail -1 gpurun_out/q.log
for i in 1 2; do python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-naive | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('cfg2', round(d['value']/1e6,2), round(r['kernel_ms'],4), round(r['frac'],4))"; done
python bench.py --steps 10 --warmup 3 --prec f32 --no-cpu-baseline --no-e2e --no-naive | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('cfg2 f32', round(d['value']/1e6,2), round(r['kernel_ms'],4))"
