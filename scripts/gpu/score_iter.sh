#!/bin/bash
mkdir -p gpurun_out
timeout -k 10 300 python -m pytest tests/test_gpu.py -q -x -k "retain or prefill_layer" > gpurun_out/score_tests.log 2>&1; echo "TESTS $?"; tail -3 gpurun_out/score_tests.log
for plan in "" legacy; do echo "plan '$plan'"; APB_SCORE_PLAN=$plan timeout 60 python scripts/attn_profile.py --score --iters 3 --queued 20 | tail -1; done
