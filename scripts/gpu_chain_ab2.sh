timeout 600 python -m pytest tests/test_multi_gpu.py -x -q > gpurun_out/mgpu_ab2.log 2>&1; echo mgpu=$?; tail -1 gpurun_out/mgpu_ab2.log
for v in c16k4 c16k8 c16k4nf c32k4nf c8k8nf c64k4; do
  export DSS_LIB_VARIANT=build/variants/libdssync_b200_$v.so
  for c in c2 c3; do
    timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus 4 --config $c --steps 40 --warmup 3 --no-nccl --e2e-steps 3 > gpurun_out/chab2_${v}_$c.log 2>&1
    echo "$v $c rc=$?"
  done
done
