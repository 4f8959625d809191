#!/bin/bash
timeout -k 10 300 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_model.py -q -x > gpurun_out/gt_tests.log 2>&1; echo "TESTS $?"; tail -2 gpurun_out/gt_tests.log
for sp in 1 0 1 0; do echo "tail split $sp"; APB_GEMM_TAIL_SPLIT=$sp timeout 120 python scripts/gemm_profile.py --iters 10 2>&1 | grep -E "o\+res|down"; done
