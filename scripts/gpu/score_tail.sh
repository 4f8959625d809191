#!/bin/bash
timeout -k 10 300 python -m pytest tests/test_gpu.py -q -x -k "retain or prefill" > gpurun_out/st_tests.log 2>&1; echo "TESTS $?"; tail -2 gpurun_out/st_tests.log
for sp in 1 0 1 0; do echo "tail split $sp"; APB_GEMM_TAIL_SPLIT=$sp timeout 60 python scripts/attn_profile.py --score --iters 3 --queued 20 | tail -1; done
timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -x -k "128k_full" 2>&1 | tail -1
