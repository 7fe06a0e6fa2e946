# A/B of environment settings on a bench workload:
#   ENVS_LIST="name1:VAR=1,VAR2=3 name2:" WL=c2 bash scripts/ab_env.sh
for item in ${ENVS_LIST}; do
  name=${item%%:*}; envs=${item#*:}; envs=${envs//,/ }
  env $envs timeout 300 python bench.py --workload ${WL:-c2} --steps ${STEPS:-20} --warmup 3 --no-cpu-baseline ${BARGS} > gpurun_out/ab_$name.json 2>gpurun_out/ab_$name.err
  python -c "import json;d=json.load(open('gpurun_out/ab_$name.json'));s=d['stages'];print('$name', d['value'], 'lat', d['latency_ms'], {k: round(v['ms_per_step'],3) for k,v in s.items() if k.startswith(('sweep','sgm'))})" || tail -5 gpurun_out/ab_$name.err
done
