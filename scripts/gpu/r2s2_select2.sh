#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null
for st in 1 2 3 4 5 0; do echo "STOP=$st"; APB_SELECT_STOP=$st timeout 60 python scripts/attn_profile.py --select --iters 3 --queued 50 | tail -1; done
