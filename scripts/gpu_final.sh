# Final validation on 4 GPUs: whole GPU suite (incl. 8-process oversubscribed multi-GPU),
# smoke, C2 benches at 1/2/4 GPUs, C1, the reference arm, sweeps at 2/4 GPUs
DSS_TEST_OVERSUBSCRIBE=1 timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/final_pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/final_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/final_smoke.log
timeout 300 python bench.py > gpurun_out/final_g1.log 2>&1; echo g1=$?
CUDA_VISIBLE_DEVICES=0,1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29581 bench.py --gpus 2 --steps 200 --warmup 5 > gpurun_out/final_g2.log 2>&1; echo g2=$?
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29582 bench.py --gpus 4 --steps 200 --warmup 5 > gpurun_out/final_g4.log 2>&1; echo g4=$?
timeout 300 python bench.py --config c1 --steps 5000 --warmup 5 > gpurun_out/final_c1.log 2>&1; echo c1=$?
timeout 300 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/final_ref.log 2>&1; echo ref=$?
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29591 bench_sweep.py --gpus 4 > gpurun_out/final_sweep_g4.jsonl 2>gpurun_out/final_sweep_g4.err; echo sw4=$?
CUDA_VISIBLE_DEVICES=0,1 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29592 bench_sweep.py --gpus 2 > gpurun_out/final_sweep_g2.jsonl 2>gpurun_out/final_sweep_g2.err; echo sw2=$?
for f in final_g1 final_g2 final_g4 final_c1 final_ref; do tail -1 gpurun_out/$f.log | python3 -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$f', d.get('impl','ours'), round(d['value'],2), 'bsp', round(d.get('bsp',{}).get('iters_s',0),1), 'e2e', round(d['e2e']['value'],1), 'roof', (d.get('roofline') or {}).get('frac'), d.get('clocks'))"; done
