# logistic device path: parity + C1 bench (with the device-gradient run) + C2 e2e fix
timeout 900 python -m pytest tests/test_gpu_logistic.py -x -q > gpurun_out/pytest_2a.log 2>&1; echo logistic=$?; tail -3 gpurun_out/pytest_2a.log
timeout 900 python -m pytest tests -m gpu -x -q -k "not multi" > gpurun_out/pytest_2a_all.log 2>&1; echo all=$?; tail -2 gpurun_out/pytest_2a_all.log
timeout 300 python bench.py --config c1 --steps 5000 --warmup 5 > gpurun_out/bench_c1_2a.log 2>&1; echo c1=$?; tail -1 gpurun_out/bench_c1_2a.log | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); print('value',d['value'],'bsp',d['bsp']['iters_s'],'e2e',d['e2e']['value'],'dev',d.get('device_gradient_run'))"
timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c2_2a.log 2>&1; echo c2=$?; tail -1 gpurun_out/bench_c2_2a.log | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); print('value',d['value'],'e2e',d['e2e']['value'],'roof',d['roofline']['frac'])"
