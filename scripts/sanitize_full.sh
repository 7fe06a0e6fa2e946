# compute-sanitizer memcheck over the whole GPU suite (except the bench-contract
# tests, which spawn subprocesses)
timeout 3000 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 30 \
  python -m pytest tests -m gpu -q --deselect tests/test_bench_gpu.py > gpurun_out/san_full_memcheck.log 2>&1
echo "memcheck rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/san_full_memcheck.log | tail -3
