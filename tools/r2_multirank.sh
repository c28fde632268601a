#!/bin/bash
# FUNCTIONAL check of bench.py's multi-rank path on one GPU (ranks share the device; gloo
# collectives on host copies; no kernel waits on another rank): cuts, shard plans, planned shard
# kernels, record exchange, combine, the bench's own verification asserts.  Not a bench number.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for N in 2 4; do
  timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
    --master-addr 127.0.0.1 --master-port $((29500 + N)) bench.py --gpus $N --size-mib 1024 \
    --steps 2 --warmup 1 --dist-backend gloo --no-e2e --no-cpu-baseline --no-per-op \
    --no-per-config > gpurun_out/multirank_$N.log 2>&1
  echo "N=$N rc=$?"; tail -c 600 gpurun_out/multirank_$N.log; echo
done
