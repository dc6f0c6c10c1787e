timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_logistic.py -q > gpurun_out/pytest_3b.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_3b.log
timeout 900 python bench_sweep.py > gpurun_out/sweep_3b_g1.jsonl 2>gpurun_out/sweep_3b.err; echo sweep=$?
python3 - <<'PY'
import json
for line in open("gpurun_out/sweep_3b_g1.jsonl"):
    try: d = json.loads(line)
    except Exception: continue
    if d["bytes_per_worker"] <= 1 << 22: print(d["N"], d["bytes_per_worker"], round(d["ds_iters_s"]), round(d["bsp_iters_s"]))
PY
timeout 300 python bench.py --config c1 --steps 5000 --warmup 5 > gpurun_out/bench_c1_3b.log 2>&1; echo c1=$?; tail -1 gpurun_out/bench_c1_3b.log | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); print('value',d['value'],'bsp',d['bsp']['iters_s'],'e2e',d['e2e']['value'],'dev',d.get('device_gradient_run',{}).get('iters_s'))"
