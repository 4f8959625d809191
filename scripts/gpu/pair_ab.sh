#!/bin/bash
# paired (2-CTA multicast) vs single-CTA attention: parity, bit-identity, steady-state timing, bench
mkdir -p gpurun_out
timeout -k 10 240 python -m pytest tests/test_gpu.py -q -x --timeout=120 --timeout_method=thread -k "paired or (attention_parity and (d128 or toy))" > gpurun_out/p_tests.log 2>&1; echo "PTESTS $?"; tail -3 gpurun_out/p_tests.log
[ "$1" = "tests" ] && exit 0
for pair in 1 0 1 0; do
  echo "== APB_ATTN_PAIR=$pair"; APB_ATTN_PAIR=$pair timeout -k 5 120 python scripts/attn_profile.py --iters 3 --phase all --clock ${CLK:-200} 2>&1 | tail -2
done
for pair in 1 0; do
  APB_ATTN_PAIR=$pair timeout -k 10 200 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/p_bench$pair.json 2> gpurun_out/p_bench$pair.err
  python -c "import json;d=json.load(open('gpurun_out/p_bench$pair.json'));print('PAIR=$pair tok/s',round(d['value']),'attn TF/s',d['roofline']['achieved'],'frac',d['roofline']['frac'],'clk',d['clocks']['sm_mhz'])"
done
