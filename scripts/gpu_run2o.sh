# 4 GPUs after the source split: whole GPU suite, smoke, benches at 1/2/4 GPUs
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_2o.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_2o.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_2o.log 2>&1; echo smoke=$?
timeout 300 python bench.py > gpurun_out/bench_g1_2o.log 2>&1; echo g1=$?; tail -1 gpurun_out/bench_g1_2o.log | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); print('g1', round(d['value'],1), 'bsp', round(d['bsp']['iters_s'],1), 'e2e', round(d['e2e']['value'],1), 'roof', round(d['roofline']['frac'],3), 'cpu', d['cpu_baseline']['value'])"
CUDA_VISIBLE_DEVICES=0,1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29581 bench.py --gpus 2 --steps 200 --warmup 5 > gpurun_out/bench_g2_2o.log 2>&1; echo g2=$?
tail -1 gpurun_out/bench_g2_2o.log | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); print('g2', round(d['value'],1), 'bsp', round(d['bsp']['iters_s'],1), 'e2e', round(d['e2e']['value'],1), d.get('nccl_baselines',{}).get('ds_split_allreduce'))"
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29582 bench.py --gpus 4 --steps 200 --warmup 5 > gpurun_out/bench_g4_2o.log 2>&1; echo g4=$?
tail -1 gpurun_out/bench_g4_2o.log | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); print('g4', round(d['value'],1), 'bsp', round(d['bsp']['iters_s'],1), 'e2e', round(d['e2e']['value'],1), d.get('nvlink',{}).get('frac'), d.get('nccl_baselines',{}).get('ds_split_allreduce'))"
