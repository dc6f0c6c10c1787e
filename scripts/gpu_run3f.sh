# 4 GPUs: chain in-place mean delivery: parity at 2 and 4 GPUs, A/B at 2 GPUs (C2, C3) and 4 GPUs (C3)
timeout 900 python -m pytest tests/test_multi_gpu.py -q > gpurun_out/mgpu_3f.log 2>&1; echo mgpu=$?; tail -1 gpurun_out/mgpu_3f.log
for v in base noinplace; do
  if [ $v = base ]; then unset DSS_LIB_VARIANT; else export DSS_LIB_VARIANT=build/variants/libdssync_b200_$v.so; fi
  for c in c2 c3; do
    CUDA_VISIBLE_DEVICES=0,1 timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29581 bench.py --gpus 2 --config $c --steps 60 --warmup 3 --no-nccl --e2e-steps 3 --no-cpu-baseline > gpurun_out/ch3f_${v}_g2_$c.log 2>&1
    echo "$v g2 $c rc=$? $(tail -1 gpurun_out/ch3f_${v}_g2_$c.log | python3 -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['value'],1), 'bsp', round(d['bsp']['iters_s'],1), {k:round(v['ms_per_step'],4) for k,v in d['kernels'].items()})" 2>&1 | tail -1)"
  done
  timeout 120 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29582 bench.py --gpus 4 --config c3 --steps 40 --warmup 3 --no-nccl --e2e-steps 3 --no-cpu-baseline > gpurun_out/ch3f_${v}_g4_c3.log 2>&1
  echo "$v g4 c3 rc=$? $(tail -1 gpurun_out/ch3f_${v}_g4_c3.log | python3 -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['value'],1), 'bsp', round(d['bsp']['iters_s'],1), {k:round(v['ms_per_step'],4) for k,v in d['kernels'].items()})" 2>&1 | tail -1)"
done
