# Round checkpoint on the GPU box: smoke, full GPU suite, headline bench with
# the CPU baseline (all host threads + one thread), reference arm, the other
# workloads, and per-workload ncu evidence (WLS_NCU).
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 30 --warmup 3 --cpu-baseline-1t > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?; head -c 300 gpurun_out/bench.json; echo
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2>gpurun_out/bench_ref.err; echo ref rc=$?
for wl in ${WLS:-c1 c3 c4 c2pg c2ncc c5}; do
  m=3; st=${STEPS:-6}; [ $wl = c4 ] && m=1; [ $wl = c3 ] && st=4
  timeout 900 python bench.py --workload $wl --steps $st --warmup 3 --inflight $m --ring 4 --no-cpu-baseline > gpurun_out/bench_$wl.json 2>gpurun_out/bench_$wl.err
  python -c "import json;d=json.load(open('gpurun_out/bench_$wl.json'));print('$wl', d['value'], 'maps/s', d['mde_per_s'], 'MDE/s lat', d['latency_ms'])" || tail -3 gpurun_out/bench_$wl.err
done
for wl in ${WLS_NCU:-c2 c2ncc c3}; do WL=$wl bash scripts/ncu_capture.sh; done
