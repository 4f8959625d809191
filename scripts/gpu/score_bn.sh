#!/bin/bash
mkdir -p gpurun_out
timeout -k 10 300 python -m pytest tests/test_gpu.py -q -x -k "retain or prefill" > gpurun_out/sbn_tests.log 2>&1; echo "TESTS $?"; tail -2 gpurun_out/sbn_tests.log
timeout -k 10 300 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_model.py -q -x > gpurun_out/sbn_tests2.log 2>&1; echo "TESTS2 $?"; tail -2 gpurun_out/sbn_tests2.log
for bn in 128 256 128 256; do echo "BN $bn"; APB_SCORE_BN=$bn timeout 60 python scripts/attn_profile.py --score --iters 3 --queued 20 | tail -1; done
APB_SCORE_BN=128 timeout 300 ncu --set full --clock-control none -k regex:gemm_kernel -c 1 python scripts/attn_profile.py --score --iters 1 > gpurun_out/sbn_ncu.txt 2>&1; grep -E "Duration|dram__bytes|Memory Throughput|L2 Hit" gpurun_out/sbn_ncu.txt | head
for bn in 128 256; do APB_SCORE_BN=$bn timeout -k 10 300 python bench.py --steps 5 --no-e2e --no-cpu-baseline > gpurun_out/sbn_bench_$bn.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/sbn_bench_$bn.json'));print('BN $bn bench',round(d['value']),d['roofline']['frac'],d['breakdown']['score']['us_per_launch'])"; done
