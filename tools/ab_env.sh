#!/bin/bash
# A/B of one env switch on the headline bench: tools/ab_env.sh VAR a b [bench args...]
# (parity subset first; each arm twice, alternating)
V=$1; A=$2; B=$3; shift 3
O=gpurun_out/ab; mkdir -p $O
python -m pytest tests/test_gpu_parity.py tests/test_gpu_prod_parity.py -q -x > $O/parity.log 2>&1; tail -1 $O/parity.log
one() { env $V=$1 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-naive "${@:2}" | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$V=$1', '${*:2}', round(d['value']/1e6,3), round(r['kernel_ms'],4), round(r['frac'],4))"; }
for i in 1 2; do one $A "$@"; one $B "$@"; done
one $A --prec f32 "$@"; one $B --prec f32 "$@"
