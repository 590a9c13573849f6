#!/bin/bash
# validate the N>1 bench path on a 1-GPU box: 2 ranks on cuda:0, gloo, sharded hash == whole-key hash
mkdir -p gpurun_out
for C in C4 C2; do
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 2 --steps 5 --warmup 3 --dist-backend gloo --same-device --verify --config $C --no-cpu-baseline \
  > gpurun_out/mr_$C.json 2> gpurun_out/mr_$C.err; echo "mr $C rc=$?"
tail -c 600 gpurun_out/mr_$C.json; tail -5 gpurun_out/mr_$C.err
done
