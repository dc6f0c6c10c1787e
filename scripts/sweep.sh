#!/bin/bash
# BASELINE config 5 sweep on N GPUs -> gpurun_out/sweep_gN.jsonl
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out
n=$1; shift
if [ "$n" = 1 ]; then
  timeout 2400 python bench_sweep.py "$@" > gpurun_out/sweep_g1.jsonl 2> gpurun_out/sweep_g1.err
else
  timeout 2400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29571 \
    bench_sweep.py --gpus $n "$@" > gpurun_out/sweep_g$n.jsonl 2> gpurun_out/sweep_g$n.err
fi
echo "sweep g$n rc=$? lines=$(wc -l < gpurun_out/sweep_g$n.jsonl)"
