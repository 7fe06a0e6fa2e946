# Bench + ncu part of the checkpoint, keeping gpurun_out/ under 64 MiB: the
# ncu reports are summarised on the box (scripts/ncu_summary.py,
# scripts/ncu_lines.py) and deleted.
timeout 900 python bench.py --steps 30 --warmup 3 --cpu-baseline-1t > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?; head -c 300 gpurun_out/bench.json; echo
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>gpurun_out/bench_ref.err; echo ref rc=$?
for wl in ${WLS:-c1 c3 c4 c2pg c2ncc c5}; do
  m=3; st=${STEPS:-6}; [ $wl = c4 ] && m=1; [ $wl = c3 ] && st=4
  timeout 900 python bench.py --workload $wl --steps $st --warmup 3 --inflight $m --ring 4 --no-cpu-baseline > gpurun_out/bench_$wl.json 2>gpurun_out/bench_$wl.err
  python -c "import json;d=json.load(open('gpurun_out/bench_$wl.json'));print('$wl', d['value'], 'maps/s', d['mde_per_s'], 'MDE/s lat', d['latency_ms'])" || tail -3 gpurun_out/bench_$wl.err
done
for wl in ${WLS_NCU:-c2 c2ncc c3}; do
  WL=$wl bash scripts/ncu_capture.sh
  python scripts/ncu_summary.py gpurun_out/ncu_$wl gpurun_out/ncu_$wl/ncu_$wl \
    "python bench.py --workload $wl --steps 2 --warmup 1 --inflight 1 --ring 2 --no-cpu-baseline" > /dev/null
  for r in gpurun_out/ncu_$wl/full_*.ncu-rep; do
    python scripts/ncu_lines.py $r 40 > ${r%.ncu-rep}_lines.txt
  done
  rm -f gpurun_out/ncu_$wl/*.ncu-rep gpurun_out/ncu_$wl/launches.csv
done
du -sh gpurun_out
