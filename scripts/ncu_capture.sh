# ncu evidence for the bench command: launch list (cold, serialised) and one
# --set full capture per dominant kernel (L0 launch of bundle 2).
set -x
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --inflight 1 --ring 2 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1; echo launches rc=$?
for k in ${NCU_KERNELS:-sweep_census_tiled sgm_lanes_kernel}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k \
    --launch-skip ${NCU_SKIP:-5} -c 1 -f -o gpurun_out/full_$k $B > gpurun_out/ncu_full_$k.log 2>&1
  echo full $k rc=$?
done
