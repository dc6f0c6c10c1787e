set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu4.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu4.log
for c in c4slice c3 c2; do timeout 400 python bench.py --config $c --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/b1_$c.log 2>&1; echo $c=$?; done
for c in c2 c3; do timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 4 --config $c --steps 200 --warmup 5 > gpurun_out/b4_$c.log 2>&1; echo g4_$c=$?; done
