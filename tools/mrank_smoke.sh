#!/bin/bash
# Multi-rank smoke run of bench.py on ONE GPU: N processes share device 0 and
# exchange through host-staged gloo collectives (exercises the torchrun path;
# the numbers are not measurements).
cd "$(dirname "$0")/.."
N=${1:-2}; shift
BH_DIST_BACKEND=gloo BH_SHARE_GPU=1 timeout 600 python -m torch.distributed.run --nnodes=1 \
  --nproc-per-node $N --master-addr 127.0.0.1 --master-port ${PORT:-29517} bench.py --gpus $N "$@"
