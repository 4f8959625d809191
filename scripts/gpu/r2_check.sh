#!/bin/bash
# round-2 check: full GPU suite + default bench (breakdown, cpu_baseline) + a D2 line
mkdir -p gpurun_out
timeout -k 10 1500 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/r2_tests.log 2>&1; echo "TESTS $?"; tail -25 gpurun_out/r2_tests.log
timeout -k 10 600 python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; echo "BENCH $?"; tail -3 gpurun_out/r2_bench.err
timeout -k 10 300 python bench.py --dist D2 --steps 3 --no-e2e --no-cpu-baseline > gpurun_out/r2_bench_d2.json 2> gpurun_out/r2_bench_d2.err; echo "BENCH D2 $?"
python - <<'PY'
import json
for f in ("gpurun_out/r2_bench.json", "gpurun_out/r2_bench_d2.json"):
    try:
        d = json.load(open(f))
        print(f, round(d["value"]), d["roofline"]["frac"], json.dumps(d.get("breakdown"))[:1500])
    except Exception as e:
        print(f, "ERR", e)
PY
