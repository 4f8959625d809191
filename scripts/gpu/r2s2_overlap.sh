#!/bin/bash
# A/B: side-stream overlap (default) vs compress-then-attend (--no-overlap), alternated
python -c "import __graft_entry__ as g; g.build()" > /dev/null
for rep in 1 2; do
  for mode in default no-overlap; do
    extra=""; [ $mode = no-overlap ] && extra="--no-overlap"
    timeout 300 python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-breakdown $extra > gpurun_out/ov.json 2>gpurun_out/ov.err
    python -c "import json;d=json.load(open('gpurun_out/ov.json'));print('$mode',round(d['value']),d['ms_per_step'],d['roofline']['frac'],d['roofline']['achieved'],d['clocks']['sm_mhz'])"
  done
done
