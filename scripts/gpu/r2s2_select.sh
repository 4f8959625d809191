#!/bin/bash
# cluster select + gather: parity, queued device time vs the register select + PDL gather, ncu durations
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python -m pytest tests/test_gpu.py -q -x -k "select or end_to_end" 2>&1 | tail -3
timeout 300 python -m pytest tests/test_gpu_peers.py tests/test_gpu_variants.py -q -x 2>&1 | tail -2
for env in "" reg "" reg; do echo "APB_SELECT=$env"; APB_SELECT=$env timeout 60 python scripts/attn_profile.py --select --iters 3 --queued 50 | tail -1; done
for cfg in llama8b-32k yi34b-200k llama8b-1m; do for env in "" reg; do echo "$cfg APB_SELECT=$env"; APB_SELECT=$env timeout 60 python scripts/attn_profile.py --config $cfg --select --iters 3 --queued 50 | tail -1; done; done
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"select|gather" -c 6 python scripts/attn_profile.py --select --iters 3 2>&1 | grep -E "select_|gather_kernel|duration" | head -12
