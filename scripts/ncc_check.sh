# NCC sweep round trip: NCC parity tests, full-size C2-NCC / C3 / C4 parity,
# certification stats of C3, and the C3 / C2-NCC benches.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "ncc or c3 or c4" > gpurun_out/pytest_ncc.log 2>&1; echo pytest rc=$?; tail -4 gpurun_out/pytest_ncc.log
timeout 300 python scripts/sweep_diag.py c3 2>&1 | tail -3
for wl in c3 c2ncc; do WL=$wl ENVS_LIST="$wl:" STEPS=${STEPS:-10} bash scripts/ab_env.sh; done
