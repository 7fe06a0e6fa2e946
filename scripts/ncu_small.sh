# ncu --set full of the level-0 launch of the per-pixel kernels (C2), summarised on the box
B="python bench.py --steps 1 --warmup 1 --inflight 1 --ring 2 --no-cpu-baseline"
for k in normal_offsets_kernel:2 wta_depth_kernel:5 median5_kernel:5 smooth_conf_tiled_kernel:5 range_rows_kernel:5; do
  name=${k%%:*}; skip=${k#*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$name --launch-skip $skip -c 1 -f -o gpurun_out/s_$name $B > /dev/null 2>&1
  python scripts/ncu_lines.py gpurun_out/s_$name.ncu-rep 12 > gpurun_out/s_${name}_lines.txt
  ncu -i gpurun_out/s_$name.ncu-rep --page raw --csv 2>/dev/null | python3 -c "
import csv,sys
r=list(csv.reader(sys.stdin)); d=dict(zip(r[0],r[2]))
print('$name', {k:d.get(k) for k in ['gpu__time_duration.sum','launch__grid_size','launch__registers_per_thread','sm__warps_active.avg.pct_of_peak_sustained_active','smsp__issue_active.avg.pct_of_peak_sustained_active','dram__bytes_read.sum','dram__bytes_write.sum','dram__throughput.avg.pct_of_peak_sustained_elapsed']})" >> gpurun_out/s_summary.txt
  rm -f gpurun_out/s_$name.ncu-rep
done
