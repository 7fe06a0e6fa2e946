# Quick GPU round trip: GPU parity suite (-x), then A/B of env settings on C2.
#   ENVS_LIST="new: old:FMVS_SGM_LINE=0" bash scripts/quick_check.sh
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -15 gpurun_out/pytest_gpu.log
WL=${WL:-c2} ENVS_LIST="${ENVS_LIST:-cur:}" bash scripts/ab_env.sh
