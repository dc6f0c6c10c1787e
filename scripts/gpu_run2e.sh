# 2 GPUs: one-shot parity (all paths) + small-buffer sweep one-shot vs two-shot
timeout 900 python -m pytest tests/test_multi_gpu.py -x -q > gpurun_out/mgpu_2e.log 2>&1; echo mgpu=$?; tail -1 gpurun_out/mgpu_2e.log
for p in 0 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29591 bench_sweep.py --gpus 2 --max-mb 4 --path $p --no-nccl > gpurun_out/sweep_2e_p$p.jsonl 2>gpurun_out/sweep_2e_p$p.err; echo sweep$p=$?
done
python3 - <<'PY'
import json
rows = {}
for p in (0, 4):
    for line in open(f"gpurun_out/sweep_2e_p{p}.jsonl"):
        try: d = json.loads(line)
        except Exception: continue
        rows.setdefault((d["N"], d["bytes_per_worker"]), {})[p] = d["ds_iters_s"]
for k in sorted(rows): print(k, {p: round(v) for p, v in rows[k].items()})
PY
