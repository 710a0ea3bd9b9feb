#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/h_gpu_tests.log 2>&1; echo gpu_tests $?; tail -2 gpurun_out/h_gpu_tests.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:oz_gemm --launch-skip 9 --launch-count 1 \
  -o gpurun_out/oz_gauss_hp -f python tools/oz_product_bench.py 8192 1 > gpurun_out/ncu_gauss.log 2>&1; echo ncu $?
tail -3 gpurun_out/ncu_gauss.log
