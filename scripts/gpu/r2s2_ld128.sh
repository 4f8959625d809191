#!/bin/bash
# A/B: S row read with one x128 TMEM load (APB_LD128=1) vs the default; parity first.
python -c "import __graft_entry__ as g; g.build()" > /dev/null
APB_LIB=$PWD/build_variants_ld128.so timeout -k 10 600 python -m pytest tests/test_gpu.py -m gpu -q -x -k "persist or steal or end_to_end or d64 or hosts" 2>&1 | tail -2
for rep in 1 2 3; do for v in cur ld128; do
  L=""; [ $v != cur ] && L=$PWD/build_variants_$v.so
  APB_LIB=$L timeout -k 5 200 python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline --no-breakdown 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('$v',round(d['value']),d['ms_per_step'],d['roofline']['frac'],d['clocks']['sm_mhz'])"
done; done
for v in cur ld128; do
  L=""; [ $v != cur ] && L=$PWD/build_variants_$v.so
  APB_LIB=$L timeout -k 5 300 python bench.py --dist D2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-breakdown 2>/dev/null | python -c "import json,sys;d=json.load(sys.stdin);print('D2 $v',round(d['value']),d['roofline']['frac'])"
done
