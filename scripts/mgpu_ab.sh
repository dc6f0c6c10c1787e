#!/bin/bash
# Multi-GPU A/B of library variants: scripts/mgpu_ab.sh N "base build/variants/x.so ..." "c2 c3 c4" [bench args]
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out
n=$1; vars=$2; cfgs=$3; shift 3
out=gpurun_out/mgpu_ab_g$n.jsonl; : > $out
for round in 1 2; do for cfg in $cfgs; do for v in $vars; do
  if [ "$v" = base ]; then unset DSS_LIB_VARIANT; else export DSS_LIB_VARIANT=$PWD/$v; fi
  line=$(timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port 29531 bench.py --gpus $n --config $cfg --extras none --no-e2e --no-nccl --steps 20 --warmup 5 "$@" \
    2> gpurun_out/mgpu_ab_last.err | tail -1)
  echo "{\"variant\": \"$v\", \"cfg\": \"$cfg\", \"line\": ${line:-null}}" >> $out
done; done; done
unset DSS_LIB_VARIANT
python - "$out" <<'PY'
import json, sys
for ln in open(sys.argv[1]):
    d = json.loads(ln); l = d["line"]
    if not l: print(d["variant"], d["cfg"], "FAILED"); continue
    k = {kk: round(v["ms_per_step"], 4) for kk, v in l["kernels"].items()}
    print(d["variant"].split("/")[-1], d["cfg"], "DS", round(l["value"], 1), "BSP", round(l["bsp"]["iters_s"], 1), k)
PY
