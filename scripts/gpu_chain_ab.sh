# chain-fold pipelining A/B at 4 GPUs (BSP C2 = chain over 2 rows/GPU; C3/C4 DS odd = chain)
for v in base ch16k ch1k cta4 cta1; do
  if [ $v = base ]; then unset DSS_LIB_VARIANT; else export DSS_LIB_VARIANT=build/variants/libdssync_b200_$v.so; fi
  for c in c2 c3; do
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus 4 --config $c --steps 60 --warmup 3 --no-nccl --e2e-steps 3 > gpurun_out/chab_${v}_$c.log 2>&1
    echo "$v $c rc=$?"
  done
done
unset DSS_LIB_VARIANT
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29562 bench.py --gpus 4 --config c4 --steps 20 --warmup 3 --no-nccl --e2e-steps 3 > gpurun_out/chab_base_c4.log 2>&1; echo c4=$?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_chain.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_chain.log
