#!/bin/bash
# Clocks / throttle reasons and kernel rate of one config under library
# variants: scripts/power_ab.sh CONFIG "base build/variants/x.so" [bench args]
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out
cfg=$1; vars=$2; shift 2
out=gpurun_out/power_ab_$cfg.jsonl; : > $out
for round in 1 2; do for v in $vars; do
  if [ "$v" = base ]; then unset DSS_LIB_VARIANT; else export DSS_LIB_VARIANT=$PWD/$v; fi
  line=$(timeout 900 python bench.py --config $cfg --extras none --no-e2e --no-cpu-baseline "$@" 2>/dev/null | tail -1)
  echo "{\"variant\": \"$v\", \"line\": ${line:-null}}" >> $out
done; done
unset DSS_LIB_VARIANT
python - "$out" <<'PY'
import json, sys
for ln in open(sys.argv[1]):
    d = json.loads(ln); l = d["line"]
    if not l: print(d["variant"], "FAILED"); continue
    print(d["variant"].split("/")[-1], round(l["value"], 2), "frac", round(l["roofline"]["frac"], 4),
          "GB/s", round(l["roofline"]["achieved"]), l["clocks"], "bsp", round(l["bsp"]["iters_s"], 2))
PY
