#!/bin/bash
# time the hp Ozaki product at n=8192 for cluster / group-size variants
for cfg in "SR_OZ_NO_CLUSTER=1 SR_OZ_GROUP_M=16" "SR_OZ_NO_CLUSTER=1 SR_OZ_GROUP_M=8" "SR_OZ_GROUP_M=16" "SR_OZ_GROUP_M=8" "SR_OZ_GROUP_M=32" "SR_OZ_GROUP_M=4"; do
  echo "== $cfg"
  env $cfg python tools/time_refine.py 8192 2>&1 | grep "ozaki"
done
