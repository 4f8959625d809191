#!/bin/bash
# time attention variants with SM clock / power sampled during the run
for v in "$@"; do
  L=$PWD/build_variants_$v.so
  nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv,noheader,nounits -lms 50 > gpurun_out/clk_$v.txt &
  P=$!
  APB_LIB=$L timeout -k 5 60 python scripts/attn_profile.py --iters 12 | tail -1
  kill $P
  echo "== $v clocks/power (median of samples under load):"
  python - "$v" <<'PY'
import sys, statistics
rows = [l.split(",") for l in open(f"gpurun_out/clk_{sys.argv[1]}.txt") if l.strip()]
load = [(float(a), float(b)) for a, b in rows if float(b) > 400]
if load:
    print("  sm_mhz", statistics.median(x[0] for x in load), "power_w", statistics.median(x[1] for x in load), "n", len(load))
PY
done
