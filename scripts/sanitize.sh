# compute-sanitizer passes over small parity cases (memcheck: out-of-bounds /
# misaligned accesses; racecheck: shared-memory hazards; synccheck: barrier use)
set -x
K="${SAN_K:-estimate_bundle_bitexact and census_sn_3lvl and 4x4}"
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
    python -m pytest tests/test_parity_gpu.py -m gpu -q -x -k "$K" > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/san_$tool.log | tail -3
done
