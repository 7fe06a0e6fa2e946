# SGM lane-blocking / prefetch sweep on the C2 bench (device time per stage)
for cfg in ${SGM_CFGS:-4x4p1 8x2p1 8x4p1 4x4p0 8x2p0}; do
  gk=${cfg%p*}; pf=${cfg#*p}; g=${gk%x*}; k=${gk#*x}
  FMVS_SGM_G=$g FMVS_SGM_K=$k FMVS_SGM_PF=$pf timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_g$cfg.json 2>gpurun_out/bench_g$cfg.err
  python -c "import json;d=json.load(open('gpurun_out/bench_g$cfg.json'));s=d['stages'];print('$cfg', d['value'], 'lat', d['latency_ms'], 'sgm', s['sgm']['ms_per_step'], 'sgm_l0', s['sgm_l0']['ms_per_step'])" || tail -3 gpurun_out/bench_g$cfg.err
done
