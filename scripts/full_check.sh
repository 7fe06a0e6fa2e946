# Full GPU parity suite + sanitizers over the NCC batched-resolution cases
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log
SAN_K="(estimate_bundle_bitexact and (ncc9_sn_7views or c4_fronto_ncc_pi) and 4x4-None) or (sweep_certified_census_ties and ncc5-quantized)" bash scripts/sanitize.sh 2>&1 | grep -v "^+"
