#!/bin/bash
# (round 2: c2_ outputs) Re-measure the other BASELINE configs, the Table-4 variants, the method table and the decode step (one gpurun call).
mkdir -p gpurun_out
for c in llama8b-32k llama8b-128k qwen14b-128k yi34b-200k llama8b-512k llama8b-1m; do
  timeout -k 10 600 python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c2_$c.json 2> gpurun_out/c2_$c.err; echo "CFG $c $?"
done
timeout -k 10 600 python bench.py --compressor random --no-e2e --no-cpu-baseline > gpurun_out/c2_random.json 2> gpurun_out/c2_random.err; echo "RANDOM $?"
timeout -k 10 600 python bench.py --shared-set --no-e2e --no-cpu-baseline > gpurun_out/c2_shared.json 2> gpurun_out/c2_shared.err; echo "SHARED $?"
timeout -k 10 600 python scripts/method_table.py > gpurun_out/c2_method.json 2> gpurun_out/c2_method.err; echo "METHOD $?"
timeout -k 10 300 python scripts/decode_profile.py > gpurun_out/c2_decode.json 2> gpurun_out/c2_decode.err; echo "DECODE $?"
timeout -k 10 300 python scripts/decode_profile.py --per-host > gpurun_out/c2_decode_ph.json 2> gpurun_out/c2_decode_ph.err; echo "DECODE_PH $?"
