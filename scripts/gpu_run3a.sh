# 1 GPU: resident-grid limits A/B after the load batching
for v in base relax relax4m; do
  if [ $v = base ]; then unset DSS_LIB_VARIANT; else export DSS_LIB_VARIANT=build/variants/libdssync_b200_$v.so; fi
  timeout 600 python bench_sweep.py --max-mb 4 > gpurun_out/sweep_3a_$v.jsonl 2>gpurun_out/sweep_3a_$v.err; echo sweep_$v=$?
done
python3 - <<'PY'
import json
rows = {}
for v in ("base", "relax", "relax4m"):
    for line in open(f"gpurun_out/sweep_3a_{v}.jsonl"):
        try: d = json.loads(line)
        except Exception: continue
        rows.setdefault((d["N"], d["bytes_per_worker"]), {})[v] = (round(d["ds_iters_s"]), round(d["bsp_iters_s"]))
for k in sorted(rows): print(k, rows[k])
PY
