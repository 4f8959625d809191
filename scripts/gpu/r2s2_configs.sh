#!/bin/bash
# Session-2 code: the other BASELINE configs, the H = N reading, Table-4 variants, method table.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
for c in llama8b-32k llama8b-128k qwen14b-128k yi34b-200k llama8b-512k llama8b-1m; do
  timeout -k 10 900 python bench.py --config $c --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c3_$c.json 2> gpurun_out/c3_$c.err; echo "CFG $c $?"
done
for H in 1 2 4; do
  timeout -k 10 600 python bench.py --hosts $H --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c3_hosts$H.json 2> gpurun_out/c3_hosts$H.err; echo "HOSTS $H $?"
done
timeout -k 10 600 python bench.py --compressor random --steps 3 --no-e2e --no-cpu-baseline > gpurun_out/c3_random.json 2> gpurun_out/c3_random.err; echo "RANDOM $?"
timeout -k 10 600 python bench.py --shared-set --steps 3 --no-e2e --no-cpu-baseline > gpurun_out/c3_shared.json 2> gpurun_out/c3_shared.err; echo "SHARED $?"
timeout -k 10 600 python scripts/method_table.py > gpurun_out/c3_method.json 2> gpurun_out/c3_method.err; echo "METHOD $?"
for f in gpurun_out/c3_*.json; do python -c "import json,sys;d=json.load(open('$f'));print('$f',round(d['value']),d['ms_per_step'],d['roofline']['frac'],d['clocks']['sm_mhz'])" 2>/dev/null; done
