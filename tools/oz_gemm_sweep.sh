#!/bin/bash
# Time the Ozaki products at n=8192 for rasterisation-group variants, then
# read the GEMM's DRAM traffic with ncu (one launch per product kind).
# Usage: bash tools/oz_gemm_sweep.sh "8 16 32 64" > gpurun_out/sweep.log
GROUPS_M=${1:-"8 16 32 64"}
for g in $GROUPS_M; do
  echo "== SR_OZ_GROUP_M=$g"
  SR_OZ_GROUP_M=$g python tools/oz_product_bench.py 8192 5 2>&1 | grep -v Warn
done
for g in $GROUPS_M; do
  echo "== ncu SR_OZ_GROUP_M=$g"
  SR_OZ_GROUP_M=$g timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second \
    --clock-control none -k regex:oz_gemm -c 3 --csv python tools/oz_product_bench.py 8192 1 2>/dev/null \
    | grep '^"[0-9]' | python -c "
import csv, sys
for r in csv.reader(sys.stdin): print('  launch', r[0], r[12], r[14])"
done
