timeout 1200 python -m pytest tests -m gpu -q -k "not multi" > gpurun_out/pytest_3i.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_3i.log
timeout 300 python bench.py --config c1 --steps 3000 --warmup 5 > gpurun_out/bench_c1_3i.log 2>&1; echo c1=$?; tail -1 gpurun_out/bench_c1_3i.log | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); print('value',d['value'],'e2e',d['e2e']['value'],'dev',d.get('device_gradient_run'))"
