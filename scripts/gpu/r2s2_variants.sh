#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null
for rep in 1 2 3; do for v in cur r2; do
  L=""; [ $v != cur ] && L=$PWD/build_variants_$v.so
  APB_LIB=$L timeout -k 5 200 python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-breakdown 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('$v',round(d['value']),d['ms_per_step'],d['roofline']['frac'],d['clocks']['sm_mhz'])"
done; done
