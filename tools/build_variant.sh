#!/bin/bash
# Build an A/B variant of libsr.so with extra nvcc flags for one source file:
#   bash tools/build_variant.sh NAME csrc_file.cu "-DFLAG=1 ..."  -> tools/_ab/libsr_NAME.so
# (load it with SR_LIB_PATH=tools/_ab/libsr_NAME.so)
set -e
name=$1; src=$2; flags=$3; srcpath=${4:-csrc/$2}  # optional: another version of the file
cd "$(dirname "$0")/../paper_2203_10879_b200"
make -s libsr.so
mkdir -p ../tools/_ab/$name
objs=""
for o in build/*.o; do
  b=$(basename $o .o)
  if [ "$b.cu" == "$src" ]; then
    /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
      --expt-relaxed-constexpr $flags -I csrc -c $srcpath -o ../tools/_ab/$name/$b.o
    objs="$objs ../tools/_ab/$name/$b.o"
  else
    objs="$objs $o"
  fi
done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../tools/_ab/libsr_$name.so $objs
echo built tools/_ab/libsr_$name.so
