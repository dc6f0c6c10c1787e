timeout 120 build/nvlink_probe 512 > gpurun_out/nvlink_probe_g4b.log 2>&1; echo probe=$?; grep -E "fold|readall" gpurun_out/nvlink_probe_g4b.log
timeout 600 python -m pytest tests/test_multi_gpu.py -x -q > gpurun_out/mgpu4b.log 2>&1; echo mgpu=$?; tail -2 gpurun_out/mgpu4b.log
for c in c2 c3; do timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 4 --config $c --steps 200 --warmup 5 > gpurun_out/b4b_$c.log 2>&1; echo g4_$c=$?; done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29532 bench_sweep.py --gpus 4 --max-mb 256 > gpurun_out/sweep_g4.jsonl 2> gpurun_out/sweep_g4.err; echo sweep=$?
