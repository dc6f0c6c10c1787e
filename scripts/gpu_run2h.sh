# 1 GPU: logistic fast-finite change parity, C1 bench, ncu of the fused C1 kernel
timeout 1200 python -m pytest tests -m gpu -q -k "not multi" > gpurun_out/pytest_2h_all.log 2>&1; echo all=$?; tail -1 gpurun_out/pytest_2h_all.log
timeout 900 python -m pytest tests/test_gpu_logistic.py tests/test_gpu_cli.py -q > gpurun_out/pytest_2h.log 2>&1; echo logi=$?; tail -2 gpurun_out/pytest_2h.log
timeout 300 python bench.py --config c1 --steps 5000 --warmup 5 > gpurun_out/bench_c1_2h.log 2>&1; echo c1=$?; tail -1 gpurun_out/bench_c1_2h.log | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); print('value',d['value'],'bsp',d['bsp']['iters_s'],'e2e',d['e2e']['value'],'dev',d.get('device_gradient_run',{}).get('iters_s'))"
python profiles/c1_logistic_run.py 300 > gpurun_out/c1run.log 2>&1; echo plain=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:small_steps -c 1 -o gpurun_out/prof_c1_logistic -f python profiles/c1_logistic_run.py 300 > gpurun_out/ncu_c1.log 2>&1; echo ncu=$?
