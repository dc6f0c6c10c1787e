CUDA_VISIBLE_DEVICES=0,1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29581 bench.py --gpus 2 --steps 200 --warmup 5 > gpurun_out/final_g2b.log 2>&1; echo g2=$?
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29582 bench.py --gpus 4 --steps 200 --warmup 5 > gpurun_out/final_g4b.log 2>&1; echo g4=$?
for f in final_g2b final_g4b; do tail -1 gpurun_out/$f.log | python3 -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$f', round(d['value'],2), 'roof', d['roofline']['frac'], d['roofline']['kernel'], 'nvlink', d.get('nvlink',{}).get('frac'))"; done
