#!/bin/bash
mkdir -p gpurun_out
python scripts/attn_profile.py --iters 5 > gpurun_out/p_local.txt 2>&1; cat gpurun_out/p_local.txt
python scripts/attn_profile.py --iters 5 --phase passing > gpurun_out/p_pass.txt 2>&1; cat gpurun_out/p_pass.txt
python scripts/attn_profile.py --iters 2 --trace 0 > gpurun_out/p_trace.txt 2>&1; head -40 gpurun_out/p_trace.txt
timeout -k 10 600 ncu --set full --clock-control none --import-source on -k regex:apb_attention -s 2 -c 1 -o gpurun_out/attn_v2 python scripts/attn_profile.py --iters 3 > gpurun_out/ncu_v2.log 2>&1; echo NCU $?
