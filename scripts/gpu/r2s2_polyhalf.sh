#!/bin/bash
# A/B: per-half placement of the FMA-pipe exponentials (3+1 and 1+3 pairs of 16 vs the default 2+2).
python -c "import __graft_entry__ as g; g.build()" > /dev/null
for v in p31 p13; do
APB_LIB=$PWD/build_variants_$v.so timeout -k 10 600 python -m pytest tests/test_gpu.py -m gpu -q -x -k "persist or steal or end_to_end" 2>&1 | tail -1
done
for rep in 1 2 3; do for v in cur p31 p13; do
  L=""; [ $v != cur ] && L=$PWD/build_variants_$v.so
  APB_LIB=$L timeout -k 5 200 python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-breakdown 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('$v',round(d['value']),d['ms_per_step'],d['roofline']['frac'],d['clocks']['sm_mhz'])"
done; done
