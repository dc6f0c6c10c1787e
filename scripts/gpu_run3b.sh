timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_logistic.py tests/test_gpu_mlp.py -q > gpurun_out/pytest_3e.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_3e.log
for r in 1 2; do
for v in narrow wide; do
  if [ $v = narrow ]; then export DSS_LIB_VARIANT=$PWD/build/variants/libdssync_b200_base.so; else unset DSS_LIB_VARIANT; fi
  timeout 300 python bench_sweep.py --max-mb 1 --no-nccl > gpurun_out/sweep_3e_${v}_$r.jsonl 2>gpurun_out/sweep_3e_${v}_$r.err; echo $v$r=$?
done; done
python3 - <<'PY'
import json
rows = {}
for v in ("narrow", "wide"):
    for r in (1, 2):
        for line in open(f"gpurun_out/sweep_3e_{v}_{r}.jsonl"):
            try: d = json.loads(line)
            except Exception: continue
            rows.setdefault((d["N"], d["bytes_per_worker"]), {}).setdefault(v, []).append((round(d["ds_iters_s"]), round(d["bsp_iters_s"])))
for k, x in sorted(rows.items()):
    print(k, "narrow", x.get("narrow"), "wide", x.get("wide"))
PY
