#!/bin/bash
# compare attention build variants with a few ncu counters (one launch each)
M=gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_elapsed,sm__issue_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_active.avg,smsp__warps_active.avg.pct_of_peak_sustained_active
for v in "$@"; do
  echo "== $v"
  APB_LIB=$PWD/build_variants_$v.so timeout -k 5 300 ncu --metrics $M --clock-control none -k regex:apb_attention -s 2 -c 1 python scripts/attn_profile.py --iters 3 2>&1 | grep -E "duration|per_second|pct|cycles_active"
done
