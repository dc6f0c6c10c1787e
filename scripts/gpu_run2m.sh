# 2 GPUs: chain partial vs mean pass split (C2, C3), DS and BSP
for c in c2 c3; do
  timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29581 bench.py --gpus 2 --config $c --steps 60 --warmup 3 --e2e-steps 3 --no-cpu-baseline > gpurun_out/bench_g2_${c}_2m.log 2>&1
  echo "$c rc=$? $(tail -1 gpurun_out/bench_g2_${c}_2m.log | python3 -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['value'],1), 'bsp', round(d['bsp']['iters_s'],1), {k:(round(v['ms_per_step'],4), v.get('nvlink_gbs')) for k,v in d['kernels'].items()}, {k:round(v['ms_per_step'],4) for k,v in d['bsp']['kernels'].items()}, d.get('nccl_baselines'))" 2>&1 | tail -1)"
done
