timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_logistic.py -q > gpurun_out/pytest_3a.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_3a.log
timeout 600 python bench_sweep.py --max-mb 1 --no-nccl > gpurun_out/sweep_3a.jsonl 2>gpurun_out/sweep_3a.err; echo sweep=$?
python3 - <<'PY'
import json
for line in open("gpurun_out/sweep_3a.jsonl"):
    try: d = json.loads(line)
    except Exception: continue
    print(d["N"], d["bytes_per_worker"], round(d["ds_iters_s"]), round(d["bsp_iters_s"]))
PY
