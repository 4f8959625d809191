#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout -k 10 600 python -m pytest tests/test_gpu.py -q -x -k "attention or hosts or end_to_end" 2>&1 | tail -2
run() { echo "== $*"; timeout -k 5 200 "$@" > gpurun_out/h.json 2>gpurun_out/h.err; echo "rc $?"; python -c "import json;d=json.load(open('gpurun_out/h.json'));print(round(d['value']),d['e2e']['value'] if d.get('e2e') else None,d['ms_per_step'],d['roofline']['frac'],d['clocks']['sm_mhz'])" 2>/dev/null; }
run python bench.py --steps 3 --warmup 3 --e2e-steps 2 --no-cpu-baseline --no-breakdown
run python bench.py --steps 3 --warmup 3 --e2e-steps 2 --no-cpu-baseline --no-breakdown --attn-launch per-host
run python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline
