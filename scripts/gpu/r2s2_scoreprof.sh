#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 60 python scripts/attn_profile.py --score --iters 3 --queued 20 | tail -1
ncu --set full --import-source on --clock-control none -k regex:"gemm_kernel" -s 2 -c 1 -o gpurun_out/score_full -f python scripts/attn_profile.py --score --iters 3 > gpurun_out/score_ncu.log 2>&1
ncu -i gpurun_out/score_full.ncu-rep --page raw --csv > gpurun_out/score_raw.csv 2>/dev/null
ncu -i gpurun_out/score_full.ncu-rep --page source --csv > gpurun_out/score_source.csv 2>/dev/null
ncu -i gpurun_out/score_full.ncu-rep --page details > gpurun_out/score_details.txt 2>/dev/null
ls -la gpurun_out/score_*
