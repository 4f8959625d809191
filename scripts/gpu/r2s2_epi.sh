#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python -m pytest tests/test_gpu.py -q -x 2>&1 | tail -2
for h in 1 7; do timeout 120 python scripts/attn_profile.py --host $h --phase all --ctatimes --iters 2 2>&1 | grep -E "^per CTA|^ctas"; done
for rep in 1 2; do
timeout 300 python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ep.json 2>gpurun_out/ep.err || tail -5 gpurun_out/ep.err
python -c "import json;d=json.load(open('gpurun_out/ep.json'));b=d['breakdown'];print(round(d['value']),d['ms_per_step'],d['roofline']['frac'],d['clocks']['sm_mhz'],{k:(v['ms_per_step'],v['launches']) for k,v in b.items() if k!='bounds'})"
done
