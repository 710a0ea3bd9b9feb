#!/bin/bash
# ncu --set full of mid-sweep solver launches (first solve of one n=8192 refinement, no CUDA graph)
mkdir -p gpurun_out
export SR_SOLVE_NO_GRAPH=1
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:far_tc_kernel \
  --launch-skip 60 --launch-count 2 -o gpurun_out/far_tc -f python tools/profile_refine.py 8192 > gpurun_out/ncu_far.log 2>&1; echo far $?
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"solve_kernel|near_kernel" \
  --launch-skip 240 --launch-count 2 -o gpurun_out/solve_near -f python tools/profile_refine.py 8192 > gpurun_out/ncu_solve.log 2>&1; echo solve $?
