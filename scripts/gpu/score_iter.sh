#!/bin/bash
# scoring kernel iteration: parity tests, standalone timing vs the old build, short bench
mkdir -p gpurun_out
timeout -k 10 400 python -m pytest tests/test_gpu.py tests/test_gpu_variants.py tests/test_gpu_model.py -q -x --timeout=200 --timeout_method=thread -k "retain or score or select or end_to_end or layer or prefill or lattice" > gpurun_out/s_tests.log 2>&1; echo "TESTS $?"; tail -3 gpurun_out/s_tests.log
for v in base "$@"; do
  if [ $v = base ]; then L=$PWD/paper_2502_12085_b200/libapb.so; else L=$PWD/build_variants_$v.so; fi
  echo "== $v"; APB_LIB=$L timeout -k 5 90 python scripts/attn_profile.py --score --iters 6 | tail -2
done
timeout -k 10 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/q_bench.json 2> gpurun_out/q_bench.err; echo "BENCH $?"
python -c "import json;d=json.load(open('gpurun_out/q_bench.json'));print('tok/s',round(d['value']),'attn TF/s',d['roofline']['achieved'],'frac',d['roofline']['frac'],'ms/step',round(d['ms_per_step'],1),'clk',d['clocks'])"
