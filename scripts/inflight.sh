for m in 1 2 3 4; do
  timeout 300 python bench.py --steps 24 --warmup 2 --inflight $m --no-cpu-baseline > gpurun_out/bench_m$m.json 2>gpurun_out/bench_m$m.err
  python -c "import json;d=json.load(open('gpurun_out/bench_m$m.json'));print('M=$m', d['value'], 'e2e', d['e2e']['value'], 'lat', d['latency_ms'])" || tail -5 gpurun_out/bench_m$m.err
done
