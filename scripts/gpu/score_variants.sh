#!/bin/bash
for v in "$@"; do echo "== $v"; for i in 1 2; do APB_LIB=$PWD/build_variants_$v.so timeout -k 5 60 python scripts/attn_profile.py --iters 4 --score | tail -1; done; done
