#!/bin/bash
# A/B of library variants on cfg3 (positions: pool + K2), cfg5 and the naive kernel: tools/ab_cfg3.sh name...
P=paper_2202_04140_b200
cp $P/libacedag_b200.so /tmp/base.so
for n in "$@"; do cp variants/$n.so $P/libacedag_b200.so
  python -m pytest tests/test_gpu_prod_parity.py tests/test_gpu_parity.py -q -x 2>&1 | tail -1
  python bench.py --config cfg3 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$n cfg3', round(d['value']/1e6,2), 'M sites/s', r.get('phases_ms'), 'naive', d.get('naive_sites_per_s'))"
  python bench.py --config cfg5 --sites 20000 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-naive | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$n cfg5', round(d['value']/1e3,2), 'k sites/s', r.get('phases_ms'))"
  python bench.py --config cfg2 --steps 5 --warmup 2 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$n cfg2 naive', d.get('naive_sites_per_s'))"
done
cp /tmp/base.so $P/libacedag_b200.so
