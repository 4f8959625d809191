#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null
for var in 0 3 4; do for st in 2 3 4 5; do echo "VAR=$var STOP=$st"; APB_SELECT_VAR=$var APB_SELECT_STOP=$st timeout 60 python scripts/attn_profile.py --select --iters 3 --queued 50 | tail -1; done; done
