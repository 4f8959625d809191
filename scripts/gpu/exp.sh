#!/bin/bash
for f in 0 1 2 3; do echo "skip=$f"; APB_DEBUG_SKIP=$f python scripts/attn_profile.py --iters 4 | tail -2; done
