#!/bin/bash
# One GPU-box pass: smoke, the gpu-marked tests, the default bench line.
# Usage (from the repo root, via gpurun): bash tools/gpu_round.sh [tag]
tag=${1:-run}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo smoke $?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_gpu_tests.log 2>&1; echo tests $?
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo bench $?
cat gpurun_out/${tag}_bench.json
