#!/bin/bash
# Round-2 ncu captures (one GPU; each command has exited 0 without ncu first):
# the Gaussian hp GEMM, the encode / decode kernels, the solver's far / solve /
# near kernels mid-sweep.  Reports land in gpurun_out/; summaries go to profiles/.
mkdir -p gpurun_out
python tools/oz_product_bench.py 8192 1 > gpurun_out/r2n_product_bench.log 2>&1; echo products $?
python tools/solve_bench.py 8192 1 > gpurun_out/r2n_solve_bench.log 2>&1; echo solve $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"oz_gemm_kernel" --launch-skip 12 --launch-count 3 \
  -o gpurun_out/r2n_gemm -f python tools/oz_product_bench.py 8192 1 > gpurun_out/r2n_ncu_gemm.log 2>&1; echo ncu_gemm $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"encode_kernel|decode_kernel" --launch-skip 24 --launch-count 6 \
  -o gpurun_out/r2n_encdec -f python tools/oz_product_bench.py 8192 1 > gpurun_out/r2n_ncu_encdec.log 2>&1; echo ncu_encdec $?
SR_SOLVE_NO_GRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"far_tc_kernel" --launch-skip 60 --launch-count 2 \
  -o gpurun_out/r2n_far -f python tools/solve_bench.py 8192 1 > gpurun_out/r2n_ncu_far.log 2>&1; echo ncu_far $?
SR_SOLVE_NO_GRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"solve_kernel|near_kernel" --launch-skip 250 --launch-count 4 \
  -o gpurun_out/r2n_chain -f python tools/solve_bench.py 8192 1 > gpurun_out/r2n_ncu_chain.log 2>&1; echo ncu_chain $?
ls -la gpurun_out/r2n_*
