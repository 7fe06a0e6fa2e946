# A/B of library variants on the C2 bench: VARIANTS="default minb2 ..."
for v in ${VARIANTS:-default}; do
  lib=""; [ "$v" != default ] && lib=paper_2112_00821_b200/_lib/$v/libfmvs.so
  FMVS_LIB=$lib timeout 300 python bench.py --steps ${STEPS:-20} --warmup 3 --no-cpu-baseline ${BARGS} > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err
  python -c "import json;d=json.load(open('gpurun_out/ab_$v.json'));s=d['stages'];print('$v', d['value'], 'lat', d['latency_ms'], {k: round(v['ms_per_step'],3) for k,v in s.items() if k.startswith(('sweep','sgm'))})" || tail -3 gpurun_out/ab_$v.err
done
