#!/bin/bash
mkdir -p gpurun_out
nproc; free -g | head -2
timeout -k 10 1500 python -m pytest tests/test_gpu_fullsize.py -q -x -s --durations=5 > gpurun_out/r2_fullsize.log 2>&1; echo "FULLSIZE $?"; grep -E "scores:|host 7|passed|failed|Error" gpurun_out/r2_fullsize.log | tail -30
