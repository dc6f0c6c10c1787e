timeout 900 python -m pytest tests/test_multi_gpu.py -x -q > gpurun_out/mgpu_ab3.log 2>&1; echo mgpu=$?; tail -1 gpurun_out/mgpu_ab3.log
for v in base c4k8 c8k8f c16k8; do
  if [ $v = base ]; then unset DSS_LIB_VARIANT; else export DSS_LIB_VARIANT=build/variants/libdssync_b200_$v.so; fi
  for c in c2 c3; do
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29581 bench.py --gpus 4 --config $c --steps 40 --warmup 3 --no-nccl --e2e-steps 3 > gpurun_out/chab3_${v}_$c.log 2>&1
    echo "$v $c rc=$?"
  done
done
unset DSS_LIB_VARIANT
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29582 bench.py --gpus 4 --config c4 --steps 30 --warmup 3 --e2e-steps 3 > gpurun_out/chab3_base_c4.log 2>&1; echo c4=$?
