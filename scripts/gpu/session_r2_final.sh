#!/bin/bash
# Round-2 final measurement session: bench lines (default, reference arm, model, D2), launch lists, ncu full captures.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/f_smi.txt
timeout -k 10 900 python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err; echo "BENCH $?"
timeout -k 10 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/f_bench_ref.json 2> gpurun_out/f_bench_ref.err; echo "REF $?"
timeout -k 10 900 python bench.py --workload model > gpurun_out/f_bench_model.json 2> gpurun_out/f_bench_model.err; echo "MODEL $?"
timeout -k 10 300 python bench.py --dist D2 --steps 3 --no-e2e --no-cpu-baseline > gpurun_out/f_bench_d2.json 2>/dev/null; echo "D2 $?"
timeout -k 10 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f_launches.csv python bench.py --layers 2 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-breakdown > /dev/null 2>&1; echo "NCU1 $?"
timeout -k 10 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f_model_launches.csv python bench.py --workload model --layers 2 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-breakdown > /dev/null 2>&1; echo "NCU2 $?"
timeout -k 10 600 ncu --set full --clock-control none -k regex:gemm_kernel -s 4 -c 4 -o gpurun_out/f_gemm_full python bench.py --workload model --layers 1 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-breakdown > /dev/null 2>&1; echo "NCU3 $?"
timeout -k 10 300 python scripts/gemm_profile.py > gpurun_out/f_gemm_profile.txt 2>&1; echo "GEMMPROF $?"; grep -v '^{' gpurun_out/f_gemm_profile.txt
for f in f_bench f_bench_model f_bench_d2; do python -c "import json;d=json.load(open('gpurun_out/$f.json'));print('$f',round(d['value']),d['roofline']['frac'],(d.get('e2e') or {}).get('value'),d['clocks'])"; done
