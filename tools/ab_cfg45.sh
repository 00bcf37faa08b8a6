#!/bin/bash
# A/B of library variants on the cfg4 (k2_quad) and cfg5 (k2_mma) workloads: tools/ab_cfg45.sh name...
P=paper_2202_04140_b200
cp $P/libacedag_b200.so /tmp/base.so
one() { python bench.py --no-cpu-baseline --no-e2e --no-naive "${@:2}" | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$1', '${*:2}', round(d['value']/1e3,2), 'k sites/s', round(r['frac'],4))"; }
for n in "$@"; do cp variants/$n.so $P/libacedag_b200.so
  python -m pytest tests/test_gpu_prod_parity.py -q -x -k "cfg4 or cfg5" 2>&1 | tail -1
  one $n --config cfg4 --sites 40000 --steps 2 --warmup 1
  one $n --config cfg5 --sites 20000 --steps 2 --warmup 1
done
cp /tmp/base.so $P/libacedag_b200.so
