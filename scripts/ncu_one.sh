# one ncu --set full capture of kernel $K (regex), launch-skip $SKIP, of a short bench
# run with extra env $ENVS; report -> gpurun_out/$NAME.ncu-rep
B="python bench.py --steps 2 --warmup 1 --inflight 1 --ring 2 --no-cpu-baseline ${BENCH_EXTRA}"
env $ENVS timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K \
  --launch-skip ${SKIP:-5} -c 1 -f -o gpurun_out/$NAME $B > gpurun_out/ncu_$NAME.log 2>&1
echo ncu $NAME rc=$?
