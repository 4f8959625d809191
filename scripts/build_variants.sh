#!/bin/bash
# Cross-compile libapb variants with extra -D flags for timing experiments:
#   scripts/build_variants.sh name1="-DFOO=1" name2="-DBAR -DBAZ=2" ...
# writes build_variants_<name>.so in the repo root (git-ignored, travels with gpurun);
# time them with scripts/gpu/variants.sh <name> ...
set -e
cd "$(dirname "$0")/.."
for spec in "$@"; do
  name="${spec%%=*}"; defs="${spec#*=}"
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
    -Xcompiler -fPIC -shared $defs -I include -o build_variants_$name.so \
    paper_2502_12085_b200/csrc/*.cu -ldl &
done
wait
ls -la build_variants_*.so
