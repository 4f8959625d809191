#!/bin/bash
for v in base th12 th4 base th12; do
  if [ $v = base ]; then L=$PWD/paper_2502_12085_b200/libapb.so; else L=$PWD/build_variants_$v.so; fi
  for dist in D1 D2; do
    APB_LIB=$L timeout 300 python bench.py --steps 3 --no-e2e --no-cpu-baseline --no-breakdown --dist $dist > gpurun_out/th.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/th.json'));print('$v $dist',round(d['value']),d['roofline']['frac'],d['clocks']['sm_mhz'])"
  done
done
