#!/bin/bash
mkdir -p gpurun_out
timeout -k 10 600 python bench.py --workload model --steps 3 --warmup 3 > gpurun_out/model_bench.json 2> gpurun_out/model_bench.err; echo "MODEL $?"; tail -2 gpurun_out/model_bench.err
python -c "import json;d=json.load(open('gpurun_out/model_bench.json'));print('tok/s',round(d['value']),'roofline',json.dumps(d['roofline'])[:600]);print('e2e',d.get('e2e',{}).get('value'))"
timeout -k 10 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/model_launches.csv python bench.py --workload model --steps 1 --warmup 1 --layers 2 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "NCU $?"
python scripts/ncu_summary.py launches gpurun_out/model_launches.csv | head -20
