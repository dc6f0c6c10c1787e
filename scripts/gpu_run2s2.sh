timeout 1200 python -m pytest tests/test_multi_gpu.py -q > gpurun_out/mgpu_2s.log 2>&1; echo mgpu=$?; tail -1 gpurun_out/mgpu_2s.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29591 bench_sweep.py --gpus 4 --max-mb 4 > gpurun_out/sweep_2s_g4.jsonl 2>gpurun_out/sweep_2s_g4.err; echo sweep=$?
python3 - <<'PY'
import json
for line in open("gpurun_out/sweep_2s_g4.jsonl"):
    try: d = json.loads(line)
    except Exception: continue
    print(d["N"], d["bytes_per_worker"], round(d["ds_iters_s"]), round(d["bsp_iters_s"]), round(d.get("nccl_bsp_iters_s", 0)))
PY
