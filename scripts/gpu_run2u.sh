# 4 GPUs: whole GPU suite, smoke, C2 benches at 1/2/4 GPUs, ncu of the fused C1 kernel
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_2u.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_2u.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_2u.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke_2u.log
timeout 300 python bench.py > gpurun_out/bench_g1_2u.log 2>&1; echo g1=$?; tail -1 gpurun_out/bench_g1_2u.log | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); print('g1', round(d['value'],1), 'bsp', round(d['bsp']['iters_s'],1), 'e2e', round(d['e2e']['value'],1), 'roof', round(d['roofline']['frac'],3), 'cpu', d['cpu_baseline']['value'], d['clocks'])"
CUDA_VISIBLE_DEVICES=0,1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29581 bench.py --gpus 2 --steps 200 --warmup 5 > gpurun_out/bench_g2_2u.log 2>&1; echo g2=$?
tail -1 gpurun_out/bench_g2_2u.log | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); print('g2', round(d['value'],1), 'bsp', round(d['bsp']['iters_s'],1), 'e2e', round(d['e2e']['value'],1))"
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29582 bench.py --gpus 4 --steps 200 --warmup 5 > gpurun_out/bench_g4_2u.log 2>&1; echo g4=$?
tail -1 gpurun_out/bench_g4_2u.log | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); print('g4', round(d['value'],1), 'bsp', round(d['bsp']['iters_s'],1), 'e2e', round(d['e2e']['value'],1), d.get('nvlink',{}).get('frac'))"
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref_2u.log 2>&1; echo ref=$?; tail -1 gpurun_out/bench_ref_2u.log | cut -c1-200
python profiles/c1_logistic_run.py 300 > gpurun_out/c1run_2u.log 2>&1; echo plain=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:small_steps -c 1 -o gpurun_out/prof_c1_logistic_2u -f python profiles/c1_logistic_run.py 300 > gpurun_out/ncu_c1_2u.log 2>&1; echo ncu=$?
