#!/bin/bash
mkdir -p gpurun_out
timeout -k 10 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_model.py -q -x > gpurun_out/g2_tests.log 2>&1; echo "TESTS $?"; tail -3 gpurun_out/g2_tests.log
timeout -k 10 300 python -m pytest tests/test_gpu.py -q -x -k "retain or prefill" > gpurun_out/g2_tests2.log 2>&1; echo "TESTS2 $?"; tail -2 gpurun_out/g2_tests2.log
timeout -k 10 120 python scripts/gemm_profile.py 2>&1 | grep -v "^{"
timeout -k 10 600 python bench.py --workload model --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/g2_model.json 2>/dev/null; echo "MODEL $?"
python -c "import json;d=json.load(open('gpurun_out/g2_model.json'));print('model tok/s',round(d['value']),'frac',d['roofline']['frac'],d['clocks'])"
