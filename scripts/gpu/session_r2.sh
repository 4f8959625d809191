#!/bin/bash
# Round-2 measurement session (one gpurun call): tests, smoke, bench, ncu launch lists + full captures.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt
timeout -k 10 1500 python -m pytest tests/ -q -m gpu --durations=10 > gpurun_out/s2_tests.log 2>&1; echo "TESTS $?"; tail -14 gpurun_out/s2_tests.log
timeout -k 10 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s2_smoke.log 2>&1; echo "SMOKE $?"; tail -1 gpurun_out/s2_smoke.log
timeout -k 10 900 python bench.py > gpurun_out/s2_bench.json 2> gpurun_out/s2_bench.err; echo "BENCH $?"
timeout -k 10 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/s2_bench_ref.json 2> gpurun_out/s2_bench_ref.err; echo "REF $?"
timeout -k 10 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s2_launches.csv python bench.py --layers 2 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-breakdown > gpurun_out/s2_ncu_list.log 2>&1; echo "NCU1 $?"
timeout -k 10 900 ncu --set full --clock-control none --import-source on -k regex:apb_attention -c 15 -o gpurun_out/s2_attn_full python bench.py --layers 1 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-breakdown > gpurun_out/s2_ncu_full.log 2>&1; echo "NCU2 $?"
timeout -k 10 600 ncu --set full --clock-control none --import-source on -k regex:"gemm_kernel|score_finalize|select|gather" -c 4 -o gpurun_out/s2_aux_full python bench.py --layers 1 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-breakdown > gpurun_out/s2_ncu_aux.log 2>&1; echo "NCU3 $?"
timeout -k 10 900 python bench.py --workload model > gpurun_out/s2_bench_model.json 2> gpurun_out/s2_bench_model.err; echo "MODEL $?"
timeout -k 10 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s2_model_launches.csv python bench.py --workload model --layers 2 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-breakdown > gpurun_out/s2_ncu_model.log 2>&1; echo "NCU4 $?"
timeout -k 10 600 ncu --set full --clock-control none -k regex:gemm_kernel -s 4 -c 4 -o gpurun_out/s2_gemm_full python bench.py --workload model --layers 1 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-breakdown > gpurun_out/s2_ncu_gemm.log 2>&1; echo "NCU5 $?"
timeout -k 10 300 python scripts/gemm_profile.py > gpurun_out/s2_gemm_profile.txt 2>&1; echo "GEMMPROF $?"; tail -1 gpurun_out/s2_gemm_profile.txt
for h in 1 2 4; do timeout -k 10 600 python bench.py --hosts $h --steps 3 --no-e2e --no-cpu-baseline > gpurun_out/s2_bench_hosts$h.json 2>/dev/null; echo "HOSTS$h $?"; done
