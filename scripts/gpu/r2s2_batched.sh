#!/bin/bash
# multi-host attention launch: parity, then bench A/B (ordered + side stream vs batched)
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python -m pytest tests/test_gpu.py -q -x -k "hosts or end_to_end or paired or parity" 2>&1 | tail -3
for cfg in llama8b-128k llama8b-32k; do
for rep in 1 2; do
  for mode in default batched; do
    extra=""; [ $mode = batched ] && extra="--batched"
    timeout 300 python bench.py --config $cfg --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-breakdown $extra > gpurun_out/bt.json 2>gpurun_out/bt.err || tail -5 gpurun_out/bt.err
    python -c "import json;d=json.load(open('gpurun_out/bt.json'));print('$cfg $mode',round(d['value']),d['ms_per_step'],d['roofline']['frac'],d['roofline']['achieved'],d['clocks']['sm_mhz'])"
  done
done
done
