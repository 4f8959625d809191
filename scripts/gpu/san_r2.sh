#!/bin/bash
# compute-sanitizer over the round-2 kernels' GPU tests: the CTA-pair GEMM (all epilogues incl. the
# scoring epilogue + finalize), the register radix select + PDL gather, the attention row sum.
mkdir -p gpurun_out
SEL='test_gemm or swiglu_epilogue or rope_epilogue or residual_in_place'
for t in memcheck synccheck racecheck; do
  timeout -k 10 1200 compute-sanitizer --tool $t --print-limit 20 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_model.py -q -x -k "($SEL) and not 14336 and not 1000" > gpurun_out/san2_gemm_$t.txt 2>&1; echo "GEMM $t $?"; tail -2 gpurun_out/san2_gemm_$t.txt
  timeout -k 10 1200 compute-sanitizer --tool $t --print-limit 20 python -m pytest tests/test_gpu.py -q -x -k "(retain_score_parity and toy) or (select_compact_bit_exact and not ties) or (select_sizes and (300 or 1000)) or (attention_parity and toy)" > gpurun_out/san2_hot_$t.txt 2>&1; echo "HOT $t $?"; tail -2 gpurun_out/san2_hot_$t.txt
done
