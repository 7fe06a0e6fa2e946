# GPU parity suite + sanitizers over dense-level cases (warp-cooperative WTA)
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log
SAN_K="(estimate_bundle_bitexact and (dense_216_planes or c4_fronto_ncc_pi) and 4x4-None)" bash scripts/sanitize.sh 2>&1 | grep -v "^+"
