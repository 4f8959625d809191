#!/bin/bash
# DRAM bytes + duration of one attention launch per variant (critical host, attn_profile default)
for v in "$@"; do
  echo "== $v"
  APB_LIB=$PWD/build_variants_$v.so timeout -k 5 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:apb_attention -s 2 -c 1 python scripts/attn_profile.py --iters 3 2>&1 | grep -E "duration|dram__|hit_rate"
done
