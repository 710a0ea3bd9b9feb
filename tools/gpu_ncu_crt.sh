#!/bin/bash
# ncu --set full of the tensor-core CRT decode (hp complex and lp) from tools/crt_bench.py
mkdir -p gpurun_out
tag=${1:-crt}
python tools/crt_bench.py 8192 2 > gpurun_out/${tag}_bench.log 2>&1; echo bench $?
cat gpurun_out/${tag}_bench.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"decode_tc_kernel" --launch-count 1 \
  -o gpurun_out/${tag}_hp -f python tools/crt_bench.py 8192 2 > gpurun_out/${tag}_ncu_hp.log 2>&1; echo ncu_hp $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"decode_tc_kernel" --launch-skip 9 --launch-count 1 \
  -o gpurun_out/${tag}_lp -f python tools/crt_bench.py 8192 2 > gpurun_out/${tag}_ncu_lp.log 2>&1; echo ncu_lp $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"decode_kernel" --launch-count 1 \
  -o gpurun_out/${tag}_simt -f python tools/crt_bench.py 8192 2 > gpurun_out/${tag}_ncu_simt.log 2>&1; echo ncu_simt $?
