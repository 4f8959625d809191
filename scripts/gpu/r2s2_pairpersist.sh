#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout -k 10 600 python -m pytest tests/test_gpu.py -q -x -k "attention or hosts or end_to_end" 2>&1 | tail -2
APB_ATTN_PAIR=1 timeout -k 10 300 python -m pytest tests/test_gpu.py -q -x -k "stress or steal or hosts_equals" 2>&1 | tail -2
APB_ATTN_PAIR=all timeout -k 5 420 python scripts/hang_repro.py --no-cpu-baseline --no-e2e --steps 6 --warmup 3 2>&1 | grep -v "^bench \[" | tail -2 | cut -c1-300
for rep in 1 2; do for v in unpaired paired; do
  P=""; [ $v = paired ] && P=all
  APB_ATTN_PAIR=$P timeout -k 10 300 python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/pp.json 2>gpurun_out/pp.err || tail -3 gpurun_out/pp.err
  python -c "import json;d=json.load(open('gpurun_out/pp.json'));print('$v',round(d['value']),d['ms_per_step'],d['roofline']['frac'],d['clocks']['sm_mhz'])"
done; done
