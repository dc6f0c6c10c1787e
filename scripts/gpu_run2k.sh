# 4 GPUs: parity after the one-shot base-offset fix; 2-GPU style A/B of the merged chain at 4 GPUs (C3)
timeout 1200 python -m pytest tests/test_multi_gpu.py -x -q > gpurun_out/mgpu_2k.log 2>&1; echo mgpu=$?; tail -1 gpurun_out/mgpu_2k.log; grep -c MISMATCH gpurun_out/mgpu_2k.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29581 bench.py --gpus 4 --steps 100 --warmup 5 --e2e-steps 3 --no-cpu-baseline > gpurun_out/bench_g4_2k.log 2>&1; echo c2=$?
tail -1 gpurun_out/bench_g4_2k.log | python3 -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['value'],1), 'bsp', round(d['bsp']['iters_s'],1), {k:round(v['ms_per_step'],4) for k,v in d['kernels'].items()}, d.get('nvlink',{}).get('frac'))"
for p in 0 4; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29591 bench_sweep.py --gpus 4 --max-mb 4 --groups 2,4 --path $p --no-nccl > gpurun_out/sweep_2k_p$p.jsonl 2>gpurun_out/sweep_2k_p$p.err; echo sweep$p=$?
done
python3 - <<'PY'
import json
rows = {}
for p in (0, 4):
    try:
        for line in open(f"gpurun_out/sweep_2k_p{p}.jsonl"):
            try: d = json.loads(line)
            except Exception: continue
            rows.setdefault((d["N"], d["bytes_per_worker"]), {})[p] = d["ds_iters_s"]
    except FileNotFoundError: pass
for k in sorted(rows): print(k, {p: round(v) for p, v in rows[k].items()})
PY
