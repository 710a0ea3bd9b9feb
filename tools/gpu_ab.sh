#!/bin/bash
# A/B of oz_gemm settings on the per-product bench: bash tools/gpu_ab.sh "ENV=.. ENV2=.." "..." ...
mkdir -p gpurun_out
for cfg in "$@"; do
  echo "== $cfg"
  env $cfg timeout 300 python tools/oz_product_bench.py 8192 5 2>&1 | grep -E "^(G-)?(hp|lp)"
done
