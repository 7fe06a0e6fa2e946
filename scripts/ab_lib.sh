# A/B of library builds on bench workloads (variants under paper_2112_00821_b200/_lib/var/):
#   LIBS="base unroll" WLS="c2 c3" bash scripts/ab_lib.sh
for wl in ${WLS:-c2}; do
  for v in ${LIBS}; do
    FMVS_LIB=paper_2112_00821_b200/_lib/var/$v.so timeout 300 python bench.py --workload $wl --steps ${STEPS:-10} --warmup 3 --no-cpu-baseline > gpurun_out/ab_${wl}_$v.json 2>gpurun_out/ab_${wl}_$v.err
    python -c "import json;d=json.load(open('gpurun_out/ab_${wl}_$v.json'));s=d['stages'];print('$wl $v', d['value'], 'lat', d['latency_ms'], {k: round(v['ms_per_step'],3) for k,v in s.items() if k.startswith(('sweep','sgm'))})" || tail -5 gpurun_out/ab_${wl}_$v.err
  done
done
