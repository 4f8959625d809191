#!/bin/bash
# build_variant.sh NAME -DMACRO=V ... : libapb with extra compile-time defines -> build_variants_NAME.so
# (A/B experiments: bench.py / the tests load it through APB_LIB).
set -e
name=$1; shift
d=build/variant_$name; mkdir -p $d
for f in paper_2502_12085_b200/csrc/*.cu; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    "$@" -I include -c -o $d/$(basename $f).o $f &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o build_variants_$name.so $d/*.o -ldl
rm -rf $d
