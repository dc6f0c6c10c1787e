#!/bin/bash
# sweep A/B: scripts/sweep_ab.sh N "base variant.so" [sweep args]
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out
n=$1; vars=$2; shift 2
for v in $vars; do
  if [ "$v" = base ]; then unset DSS_LIB_VARIANT; else export DSS_LIB_VARIANT=$PWD/$v; fi
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29581 \
    bench_sweep.py --gpus $n --no-nccl "$@" 2>/dev/null | grep '^{' | sed "s|^{|{\"variant\": \"$(basename $v)\", |"
done > gpurun_out/sweep_ab_g$n.jsonl
unset DSS_LIB_VARIANT
python - gpurun_out/sweep_ab_g$n.jsonl <<'PY'
import json, sys
rows = [json.loads(l) for l in open(sys.argv[1])]
for r in rows:
    print(r["variant"][:24], r["N"], r["bytes_per_worker"], "ds", round(r["ds_iters_s"], 1), "bsp", round(r["bsp_iters_s"], 1))
PY
