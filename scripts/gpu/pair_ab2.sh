#!/bin/bash
# paired attention for every g: parity + bit identity, then steady-state A/B on the odd-g configs
mkdir -p gpurun_out
timeout -k 10 300 python -m pytest tests/test_gpu.py -q -x --timeout=200 --timeout_method=thread -k "paired or attention_parity or full_size" > gpurun_out/p2_tests.log 2>&1; echo "PTESTS $?"; tail -3 gpurun_out/p2_tests.log
for c in qwen14b-128k yi34b-200k llama8b-128k; do for pair in 1 0; do
  echo "== $c APB_ATTN_PAIR=$pair"; APB_ATTN_PAIR=$pair timeout -k 5 120 python scripts/attn_profile.py --config $c --iters 3 --phase all --clock ${CLK:-100} 2>&1 | tail -1
done; done
