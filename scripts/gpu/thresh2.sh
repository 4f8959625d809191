#!/bin/bash
for v in th12 th16 th20 th12 th16 th20; do
  L=$PWD/build_variants_$v.so
  for dist in D1 D2; do
    APB_LIB=$L timeout 300 python bench.py --steps 3 --no-e2e --no-cpu-baseline --no-breakdown --dist $dist > gpurun_out/th.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/th.json'));print('$v $dist',round(d['value']),d['roofline']['frac'],d['clocks']['sm_mhz'])"
  done
done
