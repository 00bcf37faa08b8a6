#!/bin/bash
# env sweeps of the k2_horner chunk cost model on the headline bench (K2 ms)
one() { env "$@" python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-naive | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$*', round(d['value']/1e6,3), round(r['kernel_ms'],4), round(r['frac'],4))"; }
one X=0
one ACEDAG_HCOST_N=1.5 ACEDAG_HCOST_S=2
one ACEDAG_HCOST_N=1.5 ACEDAG_HCOST_S=2 ACEDAG_HCOST_R=8
one ACEDAG_HCOST_N=1.5 ACEDAG_HCOST_S=1 ACEDAG_HCOST_R=8 ACEDAG_HCOST_G=12
one ACEDAG_HCOST_N=1 ACEDAG_HCOST_S=2 ACEDAG_HCOST_R=8
one ACEDAG_HCOST_N=1.5 ACEDAG_HCOST_S=3 ACEDAG_HCOST_R=6 ACEDAG_HCOST_G=10
one ACEDAG_HCOST_N=1.25 ACEDAG_HCOST_S=2 ACEDAG_HCOST_R=6
one ACEDAG_HCOST_N=1.5 ACEDAG_HCOST_S=2 ACEDAG_HCOST_R=8 ACEDAG_CHUNKS=240
one X=0
