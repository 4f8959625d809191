#!/bin/bash
mkdir -p gpurun_out
timeout -k 10 600 python -m pytest tests/test_gpu_model.py tests/test_gpu_gemm.py -q -s -x -k "whole or gemm or stepwise" > gpurun_out/b1_model_tests.log 2>&1; echo "MODELTESTS $?"; grep -E "selection|passed|failed" gpurun_out/b1_model_tests.log | tail -12
timeout -k 10 600 python -m pytest tests/test_gpu.py -q -x -k "retain or select or prefill" > gpurun_out/b1_tests.log 2>&1; echo "TESTS $?"; tail -2 gpurun_out/b1_tests.log
APB_SCORE_PLAN= timeout 60 python scripts/attn_profile.py --score --iters 3 --queued 20 | tail -1
for v in base rowfp32 base rowfp32; do
  if [ $v = base ]; then L=$PWD/paper_2502_12085_b200/libapb.so; else L=$PWD/build_variants_$v.so; fi
  echo "== $v"; APB_LIB=$L timeout -k 5 120 python scripts/attn_profile.py --iters 2 --phase all --clock 400 | tail -1
done
timeout -k 10 600 python bench.py --workload model --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/b1_model.json 2>/dev/null; echo "MODEL $?"
python -c "import json;d=json.load(open('gpurun_out/b1_model.json'));print('model tok/s',round(d['value']),'frac',d['roofline']['frac'],d['clocks'])"
