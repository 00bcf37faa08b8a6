#!/bin/bash
# round-2 GPU session: tests, headline bench, Alg. 1 vs Alg. 2 DAG lines, reference arm
mkdir -p gpurun_out/r2
python -m pytest tests -m gpu -q -x > gpurun_out/r2/gputest.log 2>&1; tail -2 gpurun_out/r2/gputest.log
python bench.py --steps 20 --warmup 5 > gpurun_out/r2/bench_cfg2.jsonl 2>gpurun_out/r2/bench_cfg2.err; tail -c 400 gpurun_out/r2/bench_cfg2.jsonl
for n in 2 3; do
  python bench.py --steps 20 --warmup 5 --alg gen --n $n --no-cpu-baseline --no-e2e > gpurun_out/r2/bench_cfg2_gen$n.jsonl 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/r2/bench_cfg2_gen$n.jsonl').read().strip().splitlines()[-1]); print('gen$n', d['value'], d['config']['dag_nodes'], d['plan']['products'], d['roofline']['kernel_ms'], d['roofline']['frac'])"
done
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2/bench_reference_cfg2.jsonl 2>&1; tail -c 300 gpurun_out/r2/bench_reference_cfg2.jsonl
