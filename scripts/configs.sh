# One short bench per BASELINE config (device numbers only)
for wl in c1 c3 c4; do
  m=3; [ $wl = c4 ] && m=1
  timeout 600 python bench.py --workload $wl --steps ${STEPS:-4} --warmup 3 --inflight $m --ring 4 --no-cpu-baseline > gpurun_out/bench_$wl.json 2>gpurun_out/bench_$wl.err
  python -c "import json;d=json.load(open('gpurun_out/bench_$wl.json'));print('$wl', d['value'], 'maps/s', d['mde_per_s'], 'MDE/s lat', d['latency_ms'], {k: round(v['ms_per_step'],2) for k,v in d['stages'].items()})" || tail -5 gpurun_out/bench_$wl.err
done
