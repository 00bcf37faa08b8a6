#!/bin/bash
# ncu --set full of k2_horner for library variants: tools/ncu_variant.sh name [name...]
P=paper_2202_04140_b200
O=gpurun_out/nv; mkdir -p $O
cp $P/libacedag_b200.so /tmp/base.so
C2="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-naive"
for n in "$@"; do
  cp variants/$n.so $P/libacedag_b200.so
  ncu --set full --import-source on --clock-control none -k regex:k2_horner -s 2 -c 1 -f -o $O/$n $C2 > $O/ncu_$n.log 2>&1; echo "ncu $n rc=$?"
  ncu -i $O/$n.ncu-rep --page source --csv --print-source sass > $O/${n}_src.csv 2>/dev/null
  ncu -i $O/$n.ncu-rep --page raw --csv > $O/${n}_raw.csv 2>/dev/null
  rm -f $O/$n.ncu-rep
done
cp /tmp/base.so $P/libacedag_b200.so
