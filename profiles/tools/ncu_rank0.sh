#!/bin/bash
# NVLink byte counters of one rank's cross-GPU kernels.  Ranks 1..G-1 run
# bench.py normally; rank 0 runs the same command under ncu, collecting only
# device-level counters (nvltx/nvlrx bytes + duration) of kernels matching
# REGEX.  Never wraps the whole multi-rank job in ncu.
#   profiles/tools/ncu_rank0.sh G REGEX OUT [bench args...]
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/../..}"; mkdir -p gpurun_out
G=$1; RE=$2; OUT=$3; shift 3
export MASTER_ADDR=127.0.0.1 MASTER_PORT=29561 WORLD_SIZE=$G
pids=()
for r in $(seq 1 $((G - 1))); do
  RANK=$r LOCAL_RANK=$r timeout 900 python bench.py --gpus $G "$@" > gpurun_out/${OUT}_rank$r.log 2>&1 &
  pids+=($!)
done
RANK=0 LOCAL_RANK=0 timeout 900 ncu --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -k "regex:$RE" -c 8 --csv --log-file gpurun_out/${OUT}.csv \
  python bench.py --gpus $G "$@" > gpurun_out/${OUT}_rank0.log 2>&1
rc=$?
for p in "${pids[@]}"; do wait $p; done
echo "ncu rank0 rc=$rc"; grep -h "PROF\|passes" gpurun_out/${OUT}_rank0.log | head -12
