#!/bin/bash
# A/B of library variants on cfg5 (pool + k2_mma): tools/ab_cfg5.sh name...
P=paper_2202_04140_b200
cp $P/libacedag_b200.so /tmp/base.so
for n in "$@"; do cp variants/$n.so $P/libacedag_b200.so
  python -m pytest tests/test_gpu_prod_parity.py -q -x -k "cfg5" 2>&1 | tail -1
  python bench.py --no-cpu-baseline --no-e2e --no-naive --config cfg5 --sites 20000 --steps 2 --warmup 1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$n cfg5', round(d['value']/1e3,2), 'k sites/s', round(r['frac'],4))"
done
cp /tmp/base.so $P/libacedag_b200.so
