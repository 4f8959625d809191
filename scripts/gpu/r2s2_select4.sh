#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python -m pytest tests/test_gpu.py tests/test_gpu_peers.py -q -x -k "select or end_to_end or peer" 2>&1 | tail -3
for cfg in llama8b-128k llama8b-512k llama8b-1m; do for env in "" reg; do echo "$cfg APB_SELECT=$env"; APB_SELECT=$env timeout 60 python scripts/attn_profile.py --config $cfg --select --iters 3 --queued 50 | tail -1; done; done
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"select|gather" -c 6 python scripts/attn_profile.py --config llama8b-1m --select --iters 3 2>&1 | grep -E "duration" | head -12
