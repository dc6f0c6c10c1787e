timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_1f.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_1f.log
timeout 300 python bench.py --config c1 --steps 5000 --warmup 5 > gpurun_out/bench_c1f.log 2>&1; echo c1=$?; tail -1 gpurun_out/bench_c1f.log | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); print('value',d['value'],'bsp',d['bsp']['iters_s'],'e2e',d['e2e']['value'],'cpu',d['cpu_baseline']['value'], d['kernels'])"
timeout 900 python bench_sweep.py --gpus 1 --max-mb 1 > gpurun_out/sweep_g1f.jsonl 2>/dev/null; echo sweep=$?
