#!/bin/bash
# session-4 baseline: GPU suite, headline bench, ncu source capture of k2_horner
set -u
O=gpurun_out/s4
mkdir -p $O
python -m pytest tests -m gpu -x -q > $O/gpu_tests.log 2>&1; tail -3 $O/gpu_tests.log
C="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-naive"
for i in 1 2; do $C > $O/bench_cfg2_$i.jsonl 2> $O/bench_$i.err; python -c "import json;d=json.load(open('$O/bench_cfg2_$i.jsonl'));r=d['roofline'];print('cfg2',round(d['value']/1e6,2),r.get('kernel_ms'),round(r['frac'],4))"; done
C2="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-naive"
ncu --set full --import-source on --clock-control none -k regex:k2_horner -s 2 -c 1 -o $O/k2_horner_cfg2 $C2 > $O/ncu.log 2>&1; echo "ncu rc=$?"
ncu -i $O/k2_horner_cfg2.ncu-rep --page source --csv --print-source sass > $O/k2_src.csv 2>/dev/null
ls -la $O
