#!/bin/bash
# time attention build variants (build_variants_<name>.so in the repo root) against the default libapb.so
# (critical host of L8-128K, LOCAL and PASSING launches, plus NVML clock-normalised tensor fraction)
for v in base "$@"; do
  if [ $v = base ]; then L=$PWD/paper_2502_12085_b200/libapb.so; else L=$PWD/build_variants_$v.so; fi
  echo "== $v"; APB_LIB=$L timeout -k 5 90 python scripts/attn_profile.py --iters 3 --phase all --clock 20 | tail -2
done
