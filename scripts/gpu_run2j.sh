# 4 GPUs: parity (fixed one-shot, merged chain); C2/C3 merged vs two-kernel chain; sweep one-shot vs two-shot
timeout 1200 python -m pytest tests/test_multi_gpu.py -x -q > gpurun_out/mgpu_2j.log 2>&1; echo mgpu=$?; tail -1 gpurun_out/mgpu_2j.log; grep -c MISMATCH gpurun_out/mgpu_2j.log
for v in base nomerge; do
  if [ $v = base ]; then unset DSS_LIB_VARIANT; else export DSS_LIB_VARIANT=build/variants/libdssync_b200_$v.so; fi
  for c in c2 c3; do
    timeout 200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29581 bench.py --gpus 4 --config $c --steps 60 --warmup 3 --no-nccl --e2e-steps 3 --no-cpu-baseline > gpurun_out/ch2j_${v}_$c.log 2>&1
    echo "$v $c rc=$? $(tail -1 gpurun_out/ch2j_${v}_$c.log | python3 -c "
import json,sys
d=json.loads(sys.stdin.read()); print(round(d['value'],1), 'bsp', round(d['bsp']['iters_s'],1), {k:round(v['ms_per_step'],4) for k,v in d['kernels'].items()}, {k:round(v['ms_per_step'],4) for k,v in d['bsp']['kernels'].items()})" 2>&1 | tail -1)"
  done
done
unset DSS_LIB_VARIANT
for p in 0 4; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29591 bench_sweep.py --gpus 4 --max-mb 4 --groups 2,4 --path $p --no-nccl > gpurun_out/sweep_2j_p$p.jsonl 2>gpurun_out/sweep_2j_p$p.err; echo sweep$p=$?
done
python3 - <<'PY'
import json
rows = {}
for p in (0, 4):
    try:
        for line in open(f"gpurun_out/sweep_2j_p{p}.jsonl"):
            try: d = json.loads(line)
            except Exception: continue
            rows.setdefault((d["N"], d["bytes_per_worker"]), {})[p] = d["ds_iters_s"]
    except FileNotFoundError: pass
for k in sorted(rows): print(k, {p: round(v) for p, v in rows[k].items()})
PY
