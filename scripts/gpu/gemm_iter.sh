#!/bin/bash
mkdir -p gpurun_out
timeout -k 10 300 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_model.py -q -x > gpurun_out/gemm_tests.log 2>&1; echo "TESTS $?"; tail -15 gpurun_out/gemm_tests.log
timeout -k 10 120 python scripts/gemm_profile.py 2>&1 | tail -6
