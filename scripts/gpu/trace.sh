#!/bin/bash
python scripts/attn_profile.py --iters 2 --trace 0 2>&1 | sed -n 3,16p
APB_DEBUG_SKIP=3 python scripts/attn_profile.py --iters 2 --trace 0 2>&1 | sed -n 1,16p
