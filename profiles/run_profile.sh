#!/usr/bin/env bash
# Profiling recipe for the DS-Sync hot kernels (run under gpurun on ONE B200;
# /opt/skills/guides/B200_PROFILING.md).  Every ncu run follows a plain run of
# the identical command line that exited 0.
#   usage: bash profiles/run_profile.sh <config> [kernel-regex]
set -euo pipefail
CFG=${1:-c2}
KRE=${2:-ds_group_kernel}
DOVR=${3:+--d $3}
OUT=gpurun_out
mkdir -p $OUT
CMD="python bench.py --config $CFG --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 3 $DOVR"

# 1) launch list: every kernel with its device time (cold-cache, serialised)
$CMD > $OUT/plain_$CFG.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/launches_$CFG.csv $CMD > $OUT/ncu_launches_$CFG.log 2>&1

# 2) full section set on the dominant kernel, source-correlated (-lineinfo)
$CMD > $OUT/plain2_$CFG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:$KRE -s 4 -c 2 \
    -o $OUT/prof_${CFG}_${KRE} -f $CMD > $OUT/ncu_full_${CFG}_${KRE}.log 2>&1
echo done
