# 4 GPUs: parity for every path incl. one-shot; C2 bench; sweep one-shot vs two-shot (S=2,4,8)
timeout 1200 python -m pytest tests/test_multi_gpu.py -x -q > gpurun_out/mgpu_2g.log 2>&1; echo mgpu=$?; tail -1 gpurun_out/mgpu_2g.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29581 bench.py --gpus 4 --steps 100 --warmup 5 --e2e-steps 3 --no-cpu-baseline > gpurun_out/bench_g4_2g.log 2>&1; echo c2=$?
tail -1 gpurun_out/bench_g4_2g.log | python3 -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['value'],1), 'bsp', round(d['bsp']['iters_s'],1), {k:round(v['ms_per_step'],4) for k,v in d['kernels'].items()}, d.get('nvlink',{}).get('frac'), d.get('nccl_baselines',{}))"
for v in base os16m; do
  if [ $v = base ]; then unset DSS_LIB_VARIANT; else export DSS_LIB_VARIANT=build/variants/libdssync_b200_$v.so; fi
  for p in 0 4; do
    if [ $v = os16m ] && [ $p = 4 ]; then continue; fi
    timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29591 bench_sweep.py --gpus 4 --max-mb 16 --path $p --no-nccl > gpurun_out/sweep_2g_${v}_p$p.jsonl 2>gpurun_out/sweep_2g_${v}_p$p.err; echo sweep_${v}_$p=$?
  done
done
unset DSS_LIB_VARIANT
python3 - <<'PY'
import json
rows = {}
for tag in ("base_p0", "base_p4", "os16m_p0"):
    try:
        for line in open(f"gpurun_out/sweep_2g_{tag}.jsonl"):
            try: d = json.loads(line)
            except Exception: continue
            rows.setdefault((d["N"], d["bytes_per_worker"]), {})[tag] = d["ds_iters_s"]
    except FileNotFoundError: pass
for k in sorted(rows): print(k, {p: round(v) for p, v in rows[k].items()})
PY
