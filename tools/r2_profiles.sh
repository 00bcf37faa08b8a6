#!/bin/bash
# Round-2 evidence on one B200: bench lines for every config, the launch list
# of the headline step, and one `ncu --set full` capture per dominant kernel.
# Every ncu command runs right after the same command exited 0 without ncu.
set -u
O=gpurun_out/r2p
mkdir -p $O
B="python bench.py --no-cpu-baseline"
run() {  # name, bench args
  local name=$1; shift
  $B "$@" > $O/bench_$name.jsonl 2> $O/bench_$name.err; echo "bench $name rc=$?"
}
run cfg1 --config cfg1 --steps 50 --warmup 5
run cfg2_f32 --config cfg2 --prec f32 --steps 20 --warmup 5
run cfg3 --config cfg3 --steps 5 --warmup 3
run cfg4 --config cfg4 --steps 3 --warmup 3 --no-naive
run cfg5 --config cfg5 --steps 2 --warmup 3
run cfg2_gen2 --config cfg2 --alg gen --n 2 --steps 20 --warmup 5 --no-e2e
# launch list of the headline step (cold-cache, serialised: compare shares)
C="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-naive"
$C > $O/plain_cfg2.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
  --log-file $O/launches_cfg2.csv $C > $O/ncu_launch.log 2>&1; echo "launches rc=$?"
prof() {  # name, kernel regex, skip, cmd...
  local name=$1 k=$2 s=$3; shift 3
  "$@" > $O/plain_$name.log 2>&1 && ncu --set full --import-source on --clock-control none -k regex:$k -s $s -c 1 \
    -o $O/$name "$@" > $O/ncu_$name.log 2>&1; echo "ncu $name rc=$?"
}
prof k2_horner_cfg2 k2_horner 2 $C
prof k_tile_seeds_cfg2 k_tile_seeds 2 $C
prof pool4_cfg3 pool_positions4 3 python bench.py --config cfg3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e
prof k2_quad_cfg4 k2_quad 1 python bench.py --config cfg4 --sites 40000 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-naive
prof k2_mma_cfg5 k2_mma 2 python bench.py --config cfg5 --sites 20000 --steps 1 --warmup 2 --no-cpu-baseline --no-e2e
ls -la $O | tail -30
