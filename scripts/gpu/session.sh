#!/bin/bash
# One GPU session: full-size parity, bench, ncu launch list, ncu full captures.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt
timeout -k 10 900 python -m pytest tests/test_gpu.py -q -rA --timeout=800 --timeout_method=thread -k full_size > gpurun_out/gpu_full.log 2>&1; echo "FULL $?"
timeout -k 10 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "BENCH $?"
timeout -k 10 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --layers 2 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_list.log 2>&1; echo "NCU1 $?"
timeout -k 10 900 ncu --set full --clock-control none --import-source on -k regex:apb_attention -s 7 -c 8 -o gpurun_out/attn_full python bench.py --layers 1 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo "NCU2 $?"
timeout -k 10 600 ncu --set full --clock-control none --import-source on -k regex:"retain|select|compact" -c 3 -o gpurun_out/aux_full python bench.py --layers 1 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_aux.log 2>&1; echo "NCU3 $?"
