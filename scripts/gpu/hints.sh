#!/bin/bash
for h in none wc w c none wc; do echo "== APB_GEMM_HINTS=$h"; APB_GEMM_HINTS=$h timeout 120 python scripts/gemm_profile.py --iters 10 2>&1 | grep -v "^{"; done
for h in none wc; do APB_GEMM_HINTS=$h timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:gemm_kernel -c 4 python scripts/gemm_profile.py --iters 1 2>&1 | grep -E "dram__bytes|duration" | paste - - - | sed "s/^/$h /"; done
timeout -k 10 300 python -m pytest tests/test_gpu_gemm.py -q -x 2>&1 | tail -1
