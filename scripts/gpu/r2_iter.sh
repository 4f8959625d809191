#!/bin/bash
# round-2 iteration: parity (fast suite + full size) and timings of the changed kernels
mkdir -p gpurun_out
timeout -k 10 900 python -m pytest tests/test_gpu.py tests/test_gpu_variants.py -q -x > gpurun_out/it_tests.log 2>&1; echo "TESTS $?"; tail -3 gpurun_out/it_tests.log
timeout -k 10 900 python -m pytest tests/test_gpu_fullsize.py -q -s > gpurun_out/it_full.log 2>&1; echo "FULL $?"; grep -E "scores:|max [0-9.e-]+ mean|passed|failed" gpurun_out/it_full.log | sort -t: -k4 | tail -12
for m in "" legacy; do echo "select $m"; APB_SELECT=$m timeout 60 python scripts/attn_profile.py --select --iters 5 | tail -2; done
echo "attention critical host (all), 400-launch clock run"
timeout 120 python scripts/attn_profile.py --phase all --iters 3 --clock 400 | tail -2
timeout -k 10 300 python bench.py --steps 5 --no-e2e --no-cpu-baseline > gpurun_out/it_bench.json 2> gpurun_out/it_bench.err; echo "BENCH $?"
python -c "import json;d=json.load(open('gpurun_out/it_bench.json'));print('tok/s',round(d['value']),'frac',d['roofline']['frac'],'clk',d['clocks']['sm_mhz']);print({k:(v['us_per_launch'] if isinstance(v,dict) and 'us_per_launch' in v else None) for k,v in d['breakdown'].items()})"
