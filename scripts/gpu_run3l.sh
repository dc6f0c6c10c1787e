# 4 GPUs: three one-shot buffers: parity at 2/4/8(oversubscribed); sweep vs two buffers
DSS_TEST_OVERSUBSCRIBE=1 timeout 1500 python -m pytest tests/test_multi_gpu.py -q -s > gpurun_out/mgpu_3l.log 2>&1; echo mgpu=$?; grep -E "MISMATCH|MGPU|passed|failed" gpurun_out/mgpu_3l.log | tail -8
for v in base buf2; do
  if [ $v = base ]; then unset DSS_LIB_VARIANT; else export DSS_LIB_VARIANT=build/variants/libdssync_b200_$v.so; fi
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29591 bench_sweep.py --gpus 4 --max-mb 1 --no-nccl > gpurun_out/sweep_3l_$v.jsonl 2>gpurun_out/sweep_3l_$v.err; echo sweep_$v=$?
done
python3 - <<'PY'
import json
rows = {}
for v in ("base", "buf2"):
    for line in open(f"gpurun_out/sweep_3l_{v}.jsonl"):
        try: d = json.loads(line)
        except Exception: continue
        rows.setdefault((d["N"], d["bytes_per_worker"]), {})[v] = (round(d["ds_iters_s"]), round(d["bsp_iters_s"]))
for k in sorted(rows): print(k, rows[k])
PY
