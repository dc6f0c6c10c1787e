# 1 GPU: persistent multi-CTA small-world kernel: parity (batched steps tests), sweep A/B up to 8 MB
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "batched or small or steps" > gpurun_out/pytest_2x.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_2x.log
for v in base nopersist; do
  if [ $v = base ]; then unset DSS_LIB_VARIANT; else export DSS_LIB_VARIANT=build/variants/libdssync_b200_$v.so; fi
  timeout 600 python bench_sweep.py --max-mb 8 > gpurun_out/sweep_2x_$v.jsonl 2>gpurun_out/sweep_2x_$v.err; echo sweep_$v=$?
done
python3 - <<'PY'
import json
rows = {}
for v in ("base", "nopersist"):
    for line in open(f"gpurun_out/sweep_2x_{v}.jsonl"):
        try: d = json.loads(line)
        except Exception: continue
        rows.setdefault((d["N"], d["bytes_per_worker"]), {})[v] = (round(d["ds_iters_s"]), round(d["bsp_iters_s"]))
for k in sorted(rows): print(k, rows[k])
PY
