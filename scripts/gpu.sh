#!/bin/bash
# Local helper: one gpurun call with a clean gpurun_out/, keeping any ncu
# reports it brings back under .ncu_keep/ (git- and gpurun-ignored).
# usage: bash scripts/gpu.sh <timeout-seconds> '<command run on the GPU box>'
cd "$(dirname "$0")/.."
mkdir -p gpurun_out .ncu_keep
find gpurun_out -mindepth 1 -delete
timeout $(( $1 + 1200 )) /usr/local/graft/bin/gpurun --timeout "$1" -- "$2" 2>&1 | tail -${TAIL:-40}
for f in gpurun_out/*.ncu-rep; do [ -e "$f" ] && cp "$f" .ncu_keep/; done
exit 0
