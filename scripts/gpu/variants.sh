#!/bin/bash
# time attention build variants (build_variants_<name>.so in the repo root) against the default libapb.so
for v in base "$@"; do
  if [ $v = base ]; then L=$PWD/paper_2502_12085_b200/libapb.so; else L=$PWD/build_variants_$v.so; fi
  echo "== $v"; APB_LIB=$L timeout -k 5 60 python scripts/attn_profile.py --iters 4 | tail -1
  APB_LIB=$L timeout -k 5 60 python scripts/attn_profile.py --iters 4 --phase passing | tail -1
done
