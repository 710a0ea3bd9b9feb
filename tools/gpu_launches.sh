#!/bin/bash
# Launch lists (ncu, gpu__time_duration only) of the bench command and of one
# refinement with the solver's kernels launched directly (no CUDA graph).
tag=${1:-run}
mkdir -p gpurun_out
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_bench_pre.json 2>/dev/null; echo bench $?
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --profile-from-start off \
  --log-file gpurun_out/${tag}_refine_launches.csv env SR_SOLVE_NO_GRAPH=1 python tools/profile_refine.py 8192 > gpurun_out/${tag}_refine_ncu.log 2>&1; echo ncu_refine $?
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${tag}_bench_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_bench_ncu.log 2>&1; echo ncu_bench $?
