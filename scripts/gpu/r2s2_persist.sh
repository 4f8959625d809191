#!/bin/bash
# persistent (CLC work-stealing) attention: parity first (with a hard timeout), then A/B vs the
# non-persistent build (build_variants_base.so)
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout -k 10 600 python -m pytest tests/test_gpu.py -q -x -k "attention or hosts or end_to_end" 2>&1 | tail -3
rc=$?
timeout -k 10 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for h in 1 7; do
  for lib in base cur; do
    L=""; [ $lib = base ] && L=$PWD/build_variants_base.so
    echo "$lib host $h: $(APB_ATTN_PAIR=0 APB_LIB=$L timeout -k 5 120 python scripts/attn_profile.py --host $h --phase all --iters 3 --queued 5 2>&1 | tail -1)"
  done
done
for rep in 1 2; do for lib in base cur; do
  L=""; [ $lib = base ] && L=$PWD/build_variants_base.so
  APB_LIB=$L timeout -k 10 300 python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ps.json 2>gpurun_out/ps.err || tail -5 gpurun_out/ps.err
  python -c "import json;d=json.load(open('gpurun_out/ps.json'));b=d['breakdown'];print('$lib',round(d['value']),d['ms_per_step'],d['roofline']['frac'],d['clocks']['sm_mhz'],b['attn_all']['ms_per_step'])"
done; done
