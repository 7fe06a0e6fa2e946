# SGM group-size sweep on the C2 bench (device time per stage)
for g in 8 16 32 0; do
  FMVS_SGM_G=$g timeout 300 python bench.py --steps 5 --warmup 2 --no-cpu-baseline > gpurun_out/bench_g$g.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/bench_g$g.json'));s=d['stages'];print('G=$g', d['value'], 'sgm', s['sgm']['ms_per_step'], 'sgm_l0', s['sgm_l0']['ms_per_step'])"
done
