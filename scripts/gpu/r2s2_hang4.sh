#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > /dev/null
run() { echo "== $*"; timeout -k 5 240 "$@" > gpurun_out/h.json 2>gpurun_out/h.err; echo "rc $?"; grep "^bench \[" gpurun_out/h.err | tail -3; }
run python bench.py
run python bench.py
run python bench.py --no-breakdown
run python bench.py --no-cpu-baseline
