#!/bin/bash
# Round-2 final evidence on one B200: GPU suite, smoke, a bench line per
# config, launch lists, and one `ncu --set full` summary per dominant kernel
# (each ncu command right after the same command exited 0 without ncu).
set -u
O=gpurun_out/r2x
mkdir -p $O
python -m pytest tests -m gpu -q > $O/gputest.log 2>&1; tail -1 $O/gputest.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
B="python bench.py"
run() { local name=$1; shift; $B "$@" > $O/bench_$name.jsonl 2> $O/bench_$name.err; echo "bench $name rc=$?"; }
run cfg2 --steps 20 --warmup 5
run reference_cfg2 --impl reference --steps 2 --warmup 1
run cfg1 --config cfg1 --steps 50 --warmup 5 --no-cpu-baseline
run cfg2_f32 --config cfg2 --prec f32 --steps 20 --warmup 5 --no-cpu-baseline
run cfg3 --config cfg3 --steps 5 --warmup 3 --no-cpu-baseline
run cfg4 --config cfg4 --steps 3 --warmup 3 --no-naive --no-cpu-baseline
run cfg4_f32 --config cfg4 --prec f32 --steps 3 --warmup 3 --no-naive --no-cpu-baseline --no-e2e
run cfg5 --config cfg5 --steps 2 --warmup 3 --no-cpu-baseline
run cfg2_gen2 --config cfg2 --alg gen --n 2 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline
run cfg2_gen3 --config cfg2 --alg gen --n 3 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline
C="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-naive"
$C > $O/plain_cfg2.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv \
  --log-file $O/launches_cfg2.csv $C > $O/ncu_launch.log 2>&1; echo "launches cfg2 rc=$?"
C3="python bench.py --config cfg3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$C3 > $O/plain_cfg3.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv \
  --log-file $O/launches_cfg3.csv $C3 > $O/ncu_l3.log 2>&1; echo "launches cfg3 rc=$?"
prof() {  # name, kernel regex, skip, cmd...
  local name=$1 k=$2 s=$3; shift 3
  "$@" > $O/plain_$name.log 2>&1 && ncu --set full --import-source on --clock-control none -k regex:$k -s $s -c 1 -f \
    -o $O/$name "$@" > $O/ncu_$name.log 2>&1; echo "ncu $name rc=$?"
  python tools/ncu_summary.py $O/$name.ncu-rep > $O/${name}_ncu_full.json 2> $O/sum_$name.err
  rm -f $O/$name.ncu-rep
}
prof k2_horner_cfg2 k2_horner 2 $C
prof k_tile_seeds_cfg2 k_tile_seeds 2 $C
prof pool5_cfg3 pool_positions5 3 $C3
prof k2_quad_cfg4 k2_quad 1 python bench.py --config cfg4 --sites 40000 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-naive
prof k2_mma_cfg5 k2_mma 2 python bench.py --config cfg5 --sites 20000 --steps 1 --warmup 2 --no-cpu-baseline --no-e2e
ls -la $O | tail -40
