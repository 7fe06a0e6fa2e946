#!/bin/bash
# Build a variant of libfmvs.so with extra nvcc defines for one source file
# (A/B experiments): bash scripts/build_variant.sh <name> <file.cu> "<-Ddefs>"
# -> paper_2112_00821_b200/_lib/<name>/libfmvs.so (select with FMVS_LIB=...)
set -e
cd "$(dirname "$0")/../paper_2112_00821_b200"
name=$1; src=$2; defs=$3
out=_lib/$name; mkdir -p $out
objs=""
for o in _lib/obj/*.o; do
  b=$(basename $o .o)
  if [ "$b.cu" = "$src" ]; then
    /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 \
      -Xcompiler -fPIC,-ffp-contract=off -Xptxas -v -I../include -Icsrc $defs -c csrc/$src -o $out/$b.o 2> $out/$b.ptxas.txt
    objs="$objs $out/$b.o"
  else
    objs="$objs $o"
  fi
done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $out/libfmvs.so $objs
echo built $out/libfmvs.so
