O=gpurun_out/r2x; mkdir -p $O
C="python bench.py --config cfg5 --sites 20000 --steps 1 --warmup 2 --no-cpu-baseline --no-e2e"
$C > $O/plain_k2_mma_cfg5.log 2>&1 && ncu --set full --import-source on --clock-control none -k regex:k2_mma -s 2 -c 1 -f -o $O/k2_mma_cfg5 $C > $O/ncu_k2_mma_cfg5.log 2>&1; echo rc=$?
python tools/ncu_summary.py $O/k2_mma_cfg5.ncu-rep > $O/k2_mma_cfg5_ncu_full.json; rm -f $O/k2_mma_cfg5.ncu-rep
