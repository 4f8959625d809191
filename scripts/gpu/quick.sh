#!/bin/bash
# quick GPU iteration: parity tests + a short bench (each command under its own timeout)
mkdir -p gpurun_out
timeout -k 10 300 python -m pytest tests/test_gpu.py -q -x --timeout=120 --timeout_method=thread -k "not full_size" > gpurun_out/q_tests.log 2>&1; echo "TESTS $?"; tail -3 gpurun_out/q_tests.log
timeout -k 10 200 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err; echo "BENCH $?"
python -c "import json;d=json.load(open('gpurun_out/q_bench.json'));print('tok/s',round(d['value']),'attn TF/s',d['roofline']['achieved'],'frac',d['roofline']['frac'],'ms/step',round(d['ms_per_step'],1),'attn ms',d['roofline']['attn_ms_per_step'],'clk',d['clocks'])"
