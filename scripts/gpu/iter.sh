#!/bin/bash
# one attention iteration: attention parity tests, then timing of the listed variants vs base
mkdir -p gpurun_out
timeout -k 10 400 python -m pytest tests/test_gpu.py tests/test_gpu_variants.py -q -x --timeout=200 --timeout_method=thread -k "attention or ring or full_size or determinism or end_to_end" > gpurun_out/i_tests.log 2>&1; echo "TESTS $?"; tail -3 gpurun_out/i_tests.log
bash scripts/gpu/variants.sh "$@" 2>&1 | tee gpurun_out/i_var.txt
