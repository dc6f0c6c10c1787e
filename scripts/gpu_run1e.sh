timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_1e.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_1e.log
timeout 400 python bench.py --steps 300 --warmup 5 > gpurun_out/bench_1e.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench_1e.log | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); print('value',d['value'],'e2e',d['e2e'],'cpu',d['cpu_baseline']['value'], 'roof', d['roofline']['frac'])"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29641 bench.py --gpus 2 --steps 100 --warmup 5 --no-nccl > gpurun_out/bench_2e.log 2>&1; echo bench2=$?; tail -1 gpurun_out/bench_2e.log | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); print('value',d['value'],'e2e',d['e2e'])"
