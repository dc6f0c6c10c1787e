# 4 GPUs: final C3 / C4 numbers (DS, BSP, NCCL baselines)
for c in c3 c4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29582 bench.py --gpus 4 --config $c --steps 20 --warmup 3 --e2e-steps 3 --no-cpu-baseline > gpurun_out/final_g4_$c.log 2>&1
  echo "$c rc=$? $(tail -1 gpurun_out/final_g4_$c.log | python3 -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['value'],2), 'bsp', round(d['bsp']['iters_s'],2), 'nccl', {k:round(v['iters_s'],2) for k,v in d.get('nccl_baselines',{}).items() if isinstance(v,dict)}, {k:round(v['ms_per_step'],3) for k,v in d['kernels'].items()})" 2>&1 | tail -1)"
done
