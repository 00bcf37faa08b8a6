one() { env "$@" python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --no-naive | python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print('$*', round(d['value']/1e6,3), round(r['kernel_ms'],4), round(r['frac'],4))"; }
python -m pytest tests/test_gpu_parity.py tests/test_gpu_prod_parity.py -q -x 2>&1 | tail -1
one X=0
one ACEDAG_CHUNKS=192
one ACEDAG_CHUNKS=256
one ACEDAG_CHUNKS=384
one ACEDAG_CHUNKS=192 ACEDAG_HCOST_R=8
one X=0
python bench.py --config cfg1 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg1', d['value'])"
python bench.py --config cfg3 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg3', d['value'])"
