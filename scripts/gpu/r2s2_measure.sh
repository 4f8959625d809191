#!/bin/bash
# Round-2 session-2 measurements on the current code: bench lines, launch lists, ncu full captures.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout -k 10 1200 python -m pytest tests -m gpu -q --durations=8 > gpurun_out/y_tests.log 2>&1; echo "TESTS $?"; tail -2 gpurun_out/y_tests.log
timeout -k 10 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/y_smoke.log 2>&1; echo "SMOKE $?"; tail -1 gpurun_out/y_smoke.log
timeout -k 10 400 python bench.py > gpurun_out/y_bench.json 2> gpurun_out/y_bench.err; echo "BENCH $?"
timeout -k 10 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/y_bench_ref.json 2> gpurun_out/y_bench_ref.err; echo "REF $?"
timeout -k 10 400 python bench.py --workload model > gpurun_out/y_bench_model.json 2> gpurun_out/y_bench_model.err; echo "MODEL $?"
timeout -k 10 200 python bench.py --dist D2 --steps 3 --no-e2e --no-cpu-baseline > gpurun_out/y_bench_d2.json 2>/dev/null; echo "D2 $?"
timeout -k 10 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/y_launches.csv python bench.py --layers 2 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-breakdown > /dev/null 2>&1; echo "NCU1 $?"
timeout -k 10 900 ncu --set full --clock-control none --import-source on -k regex:apb_attention -c 1 -o gpurun_out/y_attn_full python bench.py --layers 1 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-breakdown > /dev/null 2>&1; echo "NCU3 $?"
timeout -k 10 600 ncu --set full --clock-control none -k regex:"gemm_kernel|score_finalize|select|gather" -c 4 -o gpurun_out/y_aux_full python bench.py --layers 1 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-breakdown > /dev/null 2>&1; echo "NCU4 $?"
for f in y_bench y_bench_model y_bench_d2; do python -c "import json;d=json.load(open('gpurun_out/$f.json'));print('$f',round(d['value']),d['roofline']['frac'],(d.get('e2e') or {}).get('value'),d['clocks'])"; done
timeout -k 10 300 python scripts/decode_profile.py > gpurun_out/y_decode.json 2> gpurun_out/y_decode.err; echo "DECODE $?"; tail -1 gpurun_out/y_decode.json
timeout -k 10 300 python scripts/decode_profile.py --per-host > gpurun_out/y_decode_ph.json 2> gpurun_out/y_decode_ph.err; echo "DECODE_PH $?"; tail -1 gpurun_out/y_decode_ph.json
