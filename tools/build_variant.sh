#!/bin/bash
# Dev A/B helper: build the product library with extra -D flags into
# scratch/<name>/libqpscat_b200.so (load with QPS_PRODUCT_LIB=...).
# usage: tools/build_variant.sh <name> "-DFOO=1 -DBAR=2"
set -e
name=$1; defs=$2
root=$(cd "$(dirname "$0")/.." && pwd)
src=$root/paper_1410_5003_b200/csrc
obj=/tmp/qps_variant_$name
mkdir -p $obj $root/scratch/$name
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I$root/include --expt-relaxed-constexpr"
for f in capi solver fill sweep field bcr_lr linalg prof; do nvcc $F $defs -c $src/$f.cu -o $obj/$f.o & done
nvcc $F $defs -x cu -c $src/geometry_host.cpp -o $obj/geometry_host.o
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared $obj/*.o -o $root/scratch/$name/libqpscat_b200.so -lcudart
echo "built scratch/$name/libqpscat_b200.so"
