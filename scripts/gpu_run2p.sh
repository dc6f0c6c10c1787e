# 4 GPUs: generalized one-shot (several members per GPU, small rows): parity, sweep vs path 4, C3 check
timeout 1200 python -m pytest tests/test_multi_gpu.py -x -q > gpurun_out/mgpu_2p.log 2>&1; echo mgpu=$?; tail -1 gpurun_out/mgpu_2p.log; grep -c MISMATCH gpurun_out/mgpu_2p.log
for p in 0 4; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29591 bench_sweep.py --gpus 4 --max-mb 4 --path $p --no-nccl > gpurun_out/sweep_2p_p$p.jsonl 2>gpurun_out/sweep_2p_p$p.err; echo sweep$p=$?
done
python3 - <<'PY'
import json
rows = {}
for p in (0, 4):
    try:
        for line in open(f"gpurun_out/sweep_2p_p{p}.jsonl"):
            try: d = json.loads(line)
            except Exception: continue
            rows.setdefault((d["N"], d["bytes_per_worker"]), {})[p] = d["ds_iters_s"]
    except FileNotFoundError: pass
for k in sorted(rows): print(k, {p: round(v) for p, v in rows[k].items()})
PY
timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29581 bench.py --gpus 4 --config c3 --steps 40 --warmup 3 --no-nccl --e2e-steps 3 --no-cpu-baseline > gpurun_out/bench_g4_c3_2p.log 2>&1; echo c3=$?
tail -1 gpurun_out/bench_g4_c3_2p.log | cut -c1-300
