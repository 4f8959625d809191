#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python -m pytest tests/test_gpu.py -q -x -k "hosts or end_to_end or retain or select" 2>&1 | tail -3
timeout 300 python -m pytest tests/test_gpu_peers.py tests/test_gpu_variants.py -q -x 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for rep in 1 2; do for mode in batched per-host; do
timeout 300 python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --attn-launch $mode > gpurun_out/bb.json 2>gpurun_out/bb.err || tail -5 gpurun_out/bb.err
python -c "import json;d=json.load(open('gpurun_out/bb.json'));b=d['breakdown'];print('$mode',round(d['value']),d['ms_per_step'],d['roofline']['frac'],d['clocks']['sm_mhz'],{k:(v['ms_per_step'],v['launches']) for k,v in b.items() if k!='bounds'})"
done; done
