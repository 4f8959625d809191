#!/bin/bash
# A/B: row sum widened on the ALU pipe (PRMT + FADD2, identical sums) with 2/3/4 FMA-pipe exp pairs.
python -c "import __graft_entry__ as g; g.build()" > /dev/null
for v in rsalu rsalu3; do
APB_LIB=$PWD/build_variants_$v.so timeout -k 10 600 python -m pytest tests/test_gpu.py -m gpu -q -x -k "persist or steal or end_to_end" 2>&1 | tail -1
done
for rep in 1 2 3; do for v in cur rsalu rsalu3 rsalu4; do
  L=""; [ $v != cur ] && L=$PWD/build_variants_$v.so
  APB_LIB=$L timeout -k 5 200 python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-breakdown 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('$v',round(d['value']),d['ms_per_step'],d['roofline']['frac'],d['clocks']['sm_mhz'])"
done; done
