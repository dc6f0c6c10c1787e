# 4 GPUs: one-shot flow control -- parity at 2, 4 and 8 (oversubscribed) GPUs; small-row sweep at 4 GPUs
DSS_TEST_OVERSUBSCRIBE=1 timeout 1500 python -m pytest tests/test_multi_gpu.py -q -s > gpurun_out/mgpu_3k.log 2>&1; echo mgpu=$?; grep -E "MISMATCH|MGPU|passed|failed" gpurun_out/mgpu_3k.log | tail -12
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29591 bench_sweep.py --gpus 4 --max-mb 1 --no-nccl > gpurun_out/sweep_3k.jsonl 2>gpurun_out/sweep_3k.err; echo sweep=$?
python3 - <<'PY'
import json
for line in open("gpurun_out/sweep_3k.jsonl"):
    try: d = json.loads(line)
    except Exception: continue
    print(d["N"], d["bytes_per_worker"], round(d["ds_iters_s"]), round(d["bsp_iters_s"]))
PY
