#!/bin/bash
# 4-GPU A/B of the worker placement (contiguous vs tiled) on C2 / C3 / C4.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out
n=${1:-4}; out=gpurun_out/place_ab_g$n.jsonl; : > $out
for cfg in c3 c4 c2; do for pl in 0 1; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port 29521 bench.py --gpus $n --config $cfg --placement $pl --extras none --no-e2e --steps 20 --warmup 5 \
    >> $out 2> gpurun_out/place_ab_${cfg}_${pl}.err || echo "{\"config\": \"$cfg\", \"placement\": $pl, \"failed\": true}" >> $out
done; done
python - <<'PY'
import json
for ln in open("gpurun_out/place_ab_g%s.jsonl" % __import__("os").environ.get("N", "4")) if False else []:
    pass
PY
cat $out | python -c "
import json,sys
for ln in sys.stdin:
    try: d=json.loads(ln)
    except Exception: print(ln[:200]); continue
    if d.get('failed'): print(d); continue
    print(d['config']['workload'][:3], d.get('placement'), 'DS', round(d['value'],1), 'BSP', round(d['bsp']['iters_s'],1), 'nccl', {k: round(v['iters_s'],1) for k,v in d.get('nccl_baselines',{}).items() if isinstance(v,dict)}, 'roof', d['roofline']['kind'], round(d['roofline']['frac'],3))
"
