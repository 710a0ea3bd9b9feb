#!/bin/bash
# Both bench arms back to back (as the driver runs them): the reference arm
# (CPU port, one real n = 8192 refinement) and our arm (default bench line).
tag=${1:-both}
mkdir -p gpurun_out
nproc; python -c "import threadpoolctl, json; print(json.dumps(threadpoolctl.threadpool_info()))" | head -c 600; echo
timeout 3000 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/${tag}_ref.json 2> gpurun_out/${tag}_ref.err; echo ref rc $?

cat gpurun_out/${tag}_ref.json
timeout 1500 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo bench rc $?

cat gpurun_out/${tag}_bench.json
