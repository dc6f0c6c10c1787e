for v in base ackrelax; do
  if [ $v = base ]; then unset DSS_LIB_VARIANT; else export DSS_LIB_VARIANT=build/variants/libdssync_b200_$v.so; fi
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29591 bench_sweep.py --gpus 4 --max-mb 1 --no-nccl > gpurun_out/sweep_3n_$v.jsonl 2>gpurun_out/sweep_3n_$v.err; echo sweep_$v=$?
done
python3 - <<'PY'
import json
rows = {}
for v in ("base", "ackrelax"):
    for line in open(f"gpurun_out/sweep_3n_{v}.jsonl"):
        try: d = json.loads(line)
        except Exception: continue
        rows.setdefault((d["N"], d["bytes_per_worker"]), {})[v] = (round(d["ds_iters_s"]), round(d["bsp_iters_s"]))
for k in sorted(rows): print(k, rows[k])
PY
