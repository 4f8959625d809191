#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null
for rep in 1 2; do for v in base cur-pair cur-persist; do
  L=""; P=""; [ $v = base ] && L=$PWD/build_variants_base.so; [ $v = cur-persist ] && P=0
  APB_ATTN_PAIR=$P APB_LIB=$L timeout -k 10 300 python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ps.json 2>gpurun_out/ps.err || tail -5 gpurun_out/ps.err
  python -c "import json;d=json.load(open('gpurun_out/ps.json'));b=d['breakdown'];print('$v',round(d['value']),d['ms_per_step'],d['roofline']['frac'],d['clocks']['sm_mhz'],b['attn_all']['ms_per_step'])"
done; done
for cfg in llama8b-32k qwen14b-128k; do for v in base cur-persist; do
  L=""; P=""; [ $v = base ] && L=$PWD/build_variants_base.so; [ $v = cur-persist ] && P=0
  APB_ATTN_PAIR=$P APB_LIB=$L timeout -k 10 600 python bench.py --config $cfg --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-breakdown > gpurun_out/ps.json 2>gpurun_out/ps.err || tail -5 gpurun_out/ps.err
  python -c "import json;d=json.load(open('gpurun_out/ps.json'));print('$cfg $v',round(d['value']),d['ms_per_step'],d['roofline']['frac'],d['clocks']['sm_mhz'])"
done; done
