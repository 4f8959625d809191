#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null
for c in llama8b-128k llama8b-512k; do
for dbg in 0 1; do for grp in "" m1 m4 m16 n1 n2 n4; do
echo "$c dbg=$dbg group=$grp $(APB_SCORE_DBG=$dbg APB_GEMM_GROUP=$grp timeout 120 python scripts/attn_profile.py --config $c --score --iters 3 --queued 10 | tail -1)"
done; done; done
