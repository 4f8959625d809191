#!/bin/bash
# 2-rank torchrun of bench.py on one GPU (--same-device: both ranks on cuda:0, gloo process group),
# the N > 1 LOCAL/PASSING schedule with the peer-memory exchange (CUDA IPC, the AllGather fused into
# the compaction: a real exchange between the two processes), both host layouts.
mkdir -p gpurun_out
for lay in cyclic block; do
  timeout -k 10 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus 2 --steps 2 --warmup 3 --layers 4 --same-device --host-layout $lay --no-e2e \
    > gpurun_out/mr_$lay.json 2> gpurun_out/mr_$lay.err; echo "MR $lay $?"; grep '^{' gpurun_out/mr_$lay.json | head -c 400; echo
done
