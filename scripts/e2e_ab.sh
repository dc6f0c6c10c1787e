#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out
for round in 1 2; do for v in $1; do timeout 600 python profiles/tools/e2e_ab.py $v $2; done; done > gpurun_out/e2e_ab.jsonl 2>&1
cat gpurun_out/e2e_ab.jsonl
