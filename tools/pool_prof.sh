O=gpurun_out/pp; mkdir -p $O
C3="python bench.py --config cfg3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
ncu --set full --import-source on --clock-control none -k regex:pool_positions5 -s 3 -c 1 -f -o $O/pool5 $C3 > $O/ncu.log 2>&1; echo rc=$?
ncu -i $O/pool5.ncu-rep --page source --csv --print-source sass > $O/pool5_src.csv 2>/dev/null
ncu -i $O/pool5.ncu-rep --page raw --csv > $O/pool5_raw.csv 2>/dev/null
rm -f $O/pool5.ncu-rep
