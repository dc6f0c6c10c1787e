# 1 GPU: restructured logistic kernels (parity), C1 bench, C2 default bench line, smoke
timeout 900 python -m pytest tests/test_gpu_logistic.py tests/test_gpu_cli.py -q > gpurun_out/pytest_2n.log 2>&1; echo logi=$?; tail -2 gpurun_out/pytest_2n.log
timeout 300 python bench.py --config c1 --steps 5000 --warmup 5 > gpurun_out/bench_c1_2n.log 2>&1; echo c1=$?; tail -1 gpurun_out/bench_c1_2n.log | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); print('value',d['value'],'bsp',d['bsp']['iters_s'],'e2e',d['e2e']['value'],'dev',d.get('device_gradient_run',{}).get('iters_s'))"
timeout 300 python bench.py > gpurun_out/bench_c2_2n.log 2>&1; echo c2=$?; tail -1 gpurun_out/bench_c2_2n.log | cut -c1-400
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_2n.log 2>&1; echo smoke=$?; tail -2 gpurun_out/smoke_2n.log
