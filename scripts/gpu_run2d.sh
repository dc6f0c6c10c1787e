# 1 GPU: fused small-world logistic kernel parity + C1 bench
timeout 900 python -m pytest tests/test_gpu_logistic.py tests/test_gpu_cli.py -q > gpurun_out/pytest_2d.log 2>&1; echo logi=$?; tail -3 gpurun_out/pytest_2d.log
timeout 300 python bench.py --config c1 --steps 5000 --warmup 5 > gpurun_out/bench_c1_2d.log 2>&1; echo c1=$?; tail -1 gpurun_out/bench_c1_2d.log | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); print('value',d['value'],'bsp',d['bsp']['iters_s'],'e2e',d['e2e']['value'],'dev',d.get('device_gradient_run',{}).get('iters_s'))"
