# 2 GPUs: concurrent chain mean pass with backoff polling (A keeps 8 CTAs/SM), parity + A/B
export DSS_LIB_VARIANT=build/variants/libdssync_b200_conc1.so
timeout 600 python -m pytest tests/test_multi_gpu.py -x -q > gpurun_out/mgpu_3e.log 2>&1; echo mgpu_conc1=$?; tail -1 gpurun_out/mgpu_3e.log
unset DSS_LIB_VARIANT
for v in base conc1 conc2; do
  if [ $v = base ]; then unset DSS_LIB_VARIANT; else export DSS_LIB_VARIANT=build/variants/libdssync_b200_$v.so; fi
  for c in c2 c3; do
    timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29581 bench.py --gpus 2 --config $c --steps 60 --warmup 3 --no-nccl --e2e-steps 3 --no-cpu-baseline > gpurun_out/ch3e_${v}_$c.log 2>&1
    echo "$v $c rc=$? $(tail -1 gpurun_out/ch3e_${v}_$c.log | python3 -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['value'],1), 'bsp', round(d['bsp']['iters_s'],1), {k:round(v['ms_per_step'],4) for k,v in d['kernels'].items()})" 2>&1 | tail -1)"
  done
done
