#!/bin/bash
# A/B of library variants (variants/*.so from tools/mkvariant.sh) on the headline bench:
#   tools/ab_libs.sh [name ...]   (default: every variant); prints K2 ms per variant, two rounds
P=paper_2202_04140_b200
O=gpurun_out/abl; mkdir -p $O
cp $P/libacedag_b200.so /tmp/base.so
names=("$@"); [ ${#names[@]} -eq 0 ] && names=($(ls variants/*.so | xargs -n1 basename | sed 's/\.so$//'))
one() { python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-naive $2 | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$1', '$2', round(d['value']/1e6,3), round(r['kernel_ms'],4), round(r['frac'],4))"; }
for n in "${names[@]}"; do
  cp variants/$n.so $P/libacedag_b200.so
  python -m pytest tests/test_gpu_prod_parity.py -q -x -k "cfg2" > $O/parity_$n.log 2>&1; echo "$n parity: $(tail -1 $O/parity_$n.log)"
done
for i in 1 2; do for n in "${names[@]}"; do cp variants/$n.so $P/libacedag_b200.so; one $n ""; done; done
for n in "${names[@]}"; do cp variants/$n.so $P/libacedag_b200.so; one $n "--prec f32"; done
cp /tmp/base.so $P/libacedag_b200.so
