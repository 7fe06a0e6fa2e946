set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -30 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 --cpu-baseline-steps 1 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo bench rc=$?
cat gpurun_out/bench1.json; tail -20 gpurun_out/bench1.err
cat gpurun_out/smoke.log | tail -5
