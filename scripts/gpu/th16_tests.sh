#!/bin/bash
timeout -k 10 1500 python -m pytest tests/ -q -m gpu -x > gpurun_out/th16_tests.log 2>&1; echo "TESTS $?"; tail -3 gpurun_out/th16_tests.log
grep -E "max [0-9.e-]+ mean" gpurun_out/th16_tests.log | head -3
timeout 300 python -m pytest tests/test_gpu_fullsize.py -q -s -k "d3" 2>&1 | grep -E "host 7|passed|failed" | tail -3
