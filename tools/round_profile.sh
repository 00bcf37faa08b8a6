#!/bin/bash
# One GPU call producing the round's measurement artefacts under gpurun_out/prof/:
# bench lines for every BASELINE config, the reference arm, the ncu launch
# list of the default bench command and --set full captures of the K2 kernel
# and the seed-table prep kernel.
set -u
O=gpurun_out/prof
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
timeout 600 python bench.py > $O/bench_cfg2.jsonl 2> $O/bench_cfg2.err
timeout 600 python bench.py --impl reference > $O/bench_reference.jsonl 2> $O/bench_reference.err
for c in cfg1 cfg3 cfg4 cfg5; do
  timeout 900 python bench.py --config $c --steps 20 > $O/bench_$c.jsonl 2> $O/bench_$c.err
done
timeout 600 python bench.py --prec f32 --steps 30 --no-cpu-baseline > $O/bench_cfg2_f32.jsonl 2> $O/bench_cfg2_f32.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_cfg2.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/launches.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k2_horner -c 1 -o $O/k2_horner_cfg2 \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-naive > $O/ncu_k2.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:k_tile_seeds -c 1 -o $O/k_tile_seeds_cfg2 \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-naive > $O/ncu_prep.log 2>&1
ls -la $O
