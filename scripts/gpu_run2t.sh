# 2 GPUs: chain chunk / occupancy A/B at C2 and C3
for v in base c16k8 c32k8 c8k4 c16k4 c4k8; do
  if [ $v = base ]; then unset DSS_LIB_VARIANT; else export DSS_LIB_VARIANT=build/variants/libdssync_b200_$v.so; fi
  for c in c2; do
    timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29581 bench.py --gpus 2 --config $c --steps 60 --warmup 3 --no-nccl --e2e-steps 3 --no-cpu-baseline > gpurun_out/ch2t_${v}_$c.log 2>&1
    echo "$v $c rc=$? $(tail -1 gpurun_out/ch2t_${v}_$c.log | python3 -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['value'],1), 'bsp', round(d['bsp']['iters_s'],1), {k:round(v['ms_per_step'],4) for k,v in d['kernels'].items()}, {k:round(v['ms_per_step'],4) for k,v in d['bsp']['kernels'].items()})" 2>&1 | tail -1)"
  done
done
