# one --set full capture of the C3 level-0 NCC sweep, per-line listing (all lines)
OUT=gpurun_out/c3s; mkdir -p $OUT
B="python bench.py --workload c3 --steps 1 --warmup 1 --inflight 1 --ring 2 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_ncc_tiled --launch-skip 1 -c 1 -f -o $OUT/s $B > $OUT/log 2>&1
python scripts/ncu_lines.py $OUT/s.ncu-rep 400 > $OUT/lines.txt
ncu -i $OUT/s.ncu-rep --page raw --csv > $OUT/raw.csv 2>/dev/null
ncu -i $OUT/s.ncu-rep --page source --csv --print-source sass > $OUT/sass.csv 2>/dev/null
gzip -f $OUT/sass.csv
rm -f $OUT/s.ncu-rep
