#!/bin/bash
# Build an A/B variant of libamgf.so with extra nvcc defines: tools/ab_build.sh NAME -DFOO=1 ...
# (objects in build_NAME/, library paper_2505_18576_b200/libamgf_NAME.so; select with AMGF_LIB=libamgf_NAME.so)
NAME=$1; shift
cd "$(dirname "$0")/../paper_2505_18576_b200" || exit 1
mkdir -p build_$NAME
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 -Xcompiler -fPIC -Xcompiler -ffp-contract=off"
pids=""
for f in solve setup filter tail io api; do
  /usr/local/cuda/bin/nvcc $F "$@" -c -o build_$NAME/$f.o csrc/$f.cu & pids="$pids $!"
done
for p in $pids; do wait $p || exit 1; done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o libamgf_$NAME.so build_$NAME/*.o
