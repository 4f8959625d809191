#!/bin/bash
mkdir -p gpurun_out
timeout -k 10 1500 python -m pytest tests/ -q -m gpu --durations=12 > gpurun_out/b2_tests.log 2>&1; echo "TESTS $?"; tail -16 gpurun_out/b2_tests.log
timeout -k 10 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/b2_smoke.log 2>&1; echo "SMOKE $?"; tail -1 gpurun_out/b2_smoke.log
bash scripts/gpu/multirank.sh
