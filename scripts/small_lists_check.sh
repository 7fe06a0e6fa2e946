# NCC exact-list overflow paths (FMVS_NCC_SMALL_LISTS) + NCC parity + perf A/B
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -k "ncc or c3 or c4 or small_lists or overflow" > gpurun_out/pytest_ncc.log 2>&1; echo pytest rc=$?; tail -4 gpurun_out/pytest_ncc.log
LIBS="wtaw small" WLS="c3 c2ncc" bash scripts/ab_lib.sh
