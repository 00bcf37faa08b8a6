#!/bin/bash
# final round-2 session: full GPU suite, smoke, bench lines of the configs the
# late kernels changed, an ncu capture of pool_positions5 at cfg3
O=gpurun_out/r2f
mkdir -p $O
python -m pytest tests -m gpu -q > $O/gputest.log 2>&1; tail -1 $O/gputest.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py --steps 20 --warmup 5 > $O/bench_cfg2.jsonl 2>$O/bench_cfg2.err; echo "cfg2 rc=$?"
python bench.py --config cfg3 --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_cfg3.jsonl 2>$O/bench_cfg3.err; echo "cfg3 rc=$?"
python bench.py --config cfg5 --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_cfg5.jsonl 2>$O/bench_cfg5.err; echo "cfg5 rc=$?"
C="python bench.py --config cfg3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$C > $O/plain_pool5.log 2>&1 && ncu --set full --import-source on --clock-control none -k regex:pool_positions5 -s 3 -c 1 \
  -o $O/pool5_cfg3 $C > $O/ncu_pool5.log 2>&1; echo "ncu pool5 rc=$?"
$C > $O/plain_l3.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file $O/launches_cfg3.csv $C > $O/ncu_l3.log 2>&1; echo "launches cfg3 rc=$?"
