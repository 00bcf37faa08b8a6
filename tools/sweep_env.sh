#!/bin/bash
# env sweeps of the k2_horner chunk cost model on the headline bench (K2 ms)
one() { env "$@" python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-naive | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$*', round(d['value']/1e6,3), round(r['kernel_ms'],4), round(r['frac'],4))"; }
one X=0
one ACEDAG_HCOST_R=8
one ACEDAG_HCOST_R=12
one ACEDAG_HCOST_R=20
one ACEDAG_HCOST_N=3 ACEDAG_HCOST_R=12
one ACEDAG_HCOST_N=1.5 ACEDAG_HCOST_R=8
one ACEDAG_HCOST_G=12 ACEDAG_HCOST_R=8
one ACEDAG_HCOST_G=5 ACEDAG_HCOST_R=8
one ACEDAG_CHUNKS=192
one ACEDAG_CHUNKS=256
one ACEDAG_CHUNKS=96
one ACEDAG_HGUIDE=0.5
one X=0
