#!/bin/bash
# decode variants: whole-step profile + ncu duration / DRAM of the per-host partial kernel
for v in "$@"; do
  echo "== $v"
  APB_LIB=$PWD/build_variants_$v.so timeout -k 5 120 python scripts/decode_profile.py 2>&1 | tail -1
  APB_LIB=$PWD/build_variants_$v.so timeout -k 5 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"decode_mma|decode_stream|merge_kernel" -c 2 python scripts/decode_profile.py --iters 1 2>&1 | grep -E "duration|warps"
done
