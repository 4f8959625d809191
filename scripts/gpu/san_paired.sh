#!/bin/bash
# compute-sanitizer over the paired (2-CTA cluster, multicast K/V) attention kernel's parity tests.
mkdir -p gpurun_out
for t in memcheck synccheck racecheck; do
  timeout -k 10 900 compute-sanitizer --tool $t --print-limit 20 python -m pytest tests/test_gpu.py -q -x -k "paired_matches_single_cta and (gqa8-d128 or d128-sink or gqa3)" > gpurun_out/san_paired_$t.txt 2>&1; echo "SAN $t $?"; tail -2 gpurun_out/san_paired_$t.txt
done
