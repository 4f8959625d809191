#!/bin/bash
for dbg in 0 1; do echo "select dbg=$dbg"; APB_SELECT_DBG=$dbg timeout 60 python scripts/attn_profile.py --select --iters 3 --queued 50 | tail -1; done
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"select|gather" -c 6 python scripts/attn_profile.py --select --iters 3 2>&1 | grep -E "select_fast|gather_kernel|duration" | head -12
