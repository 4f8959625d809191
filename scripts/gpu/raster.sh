#!/bin/bash
for g in "" m8 m20 m40 n4 n8 n16; do echo "== APB_GEMM_GROUP=$g"; APB_GEMM_GROUP=$g timeout 120 python scripts/gemm_profile.py --iters 10 2>&1 | grep -v "^{"; done
for g in m8 m20 n8; do APB_GEMM_GROUP=$g timeout 300 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:gemm_kernel -c 4 python scripts/gemm_profile.py --iters 1 2>&1 | grep -E "dram__bytes_read|duration" | paste - - | sed "s/^/$g /"; done
