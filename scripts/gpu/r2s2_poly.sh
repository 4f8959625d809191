#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout -k 10 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
for cfg in llama8b-128k llama8b-32k qwen14b-128k; do
timeout -k 5 600 python bench.py --config $cfg --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-breakdown 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('$cfg',round(d['value']),d['ms_per_step'],d['roofline']['frac'],d['clocks']['sm_mhz'])"
done
timeout -k 5 300 python bench.py --dist D2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-breakdown 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('D2',round(d['value']),d['roofline']['frac'])"
