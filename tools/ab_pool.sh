#!/bin/bash
# A/B of library variants on cfg3 (pool_positions5 + k2_horner): tools/ab_pool.sh name...
P=paper_2202_04140_b200
cp $P/libacedag_b200.so /tmp/base.so
for n in "$@"; do cp variants/$n.so $P/libacedag_b200.so
  python -m pytest tests/test_gpu_prod_parity.py -q -x -k "cfg3" 2>&1 | tail -1
  python bench.py --config cfg3 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$n cfg3', round(d['value']/1e6,2), 'M sites/s', round(d['ms_per_step'],2), r.get('phases_ms'))"
done
cp /tmp/base.so $P/libacedag_b200.so
