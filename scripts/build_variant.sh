#!/bin/bash
# Build an A/B variant of the library: scripts/build_variant.sh NAME -DFOO=1 ...
# -> paper_2409_20156_b200/libastra_b200_NAME.so (load with ASTRA_LIB_VARIANT=NAME)
set -e
name=$1; shift
d=paper_2409_20156_b200
mkdir -p /tmp/variant_$name
for src in capi sampler step refresh refresh_tc dense dense_tc; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr \
    -Xcompiler -fPIC,-O2 "$@" -c $d/csrc/$src.cu -o /tmp/variant_$name/$src.o &
done
wait
nvcc -shared -gencode arch=compute_100a,code=sm_100a /tmp/variant_$name/*.o -o $d/libastra_b200_$name.so -cudart static
echo $d/libastra_b200_$name.so
