#!/bin/bash
# Diagnostic builds with per-kernel timeline marks: bash tools/build_timeline.sh NAME "extra nvcc flags"
# -> tools/_ab/libsr_NAME.so (python tools/solve_timeline.py 8192 tools/_ab/libsr_NAME.so)
set -e
name=$1; flags=$2
cd "$(dirname "$0")/.."
mkdir -p tools/_ab/$name
for f in paper_2203_10879_b200/csrc/*.cu; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC \
    --expt-relaxed-constexpr -I include -DSR_TIMELINE $flags -c $f -o tools/_ab/$name/$(basename $f .cu).o &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o tools/_ab/libsr_$name.so tools/_ab/$name/*.o
echo built tools/_ab/libsr_$name.so
