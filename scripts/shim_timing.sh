#!/bin/bash
# Drop-in cost: the reference's run_training pure vs linked with the B200
# shim (DS W=16/N=4, momentum, isotropic quadratic, fp64), d = 1M and 4M,
# lockstep and parallel; final params compared bit for bit.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out
out=gpurun_out/shim_timing.jsonl; : > $out
for d in 1000000 4000000; do for mode in lockstep parallel; do
  T=$([ $d -gt 1000000 ] && echo 6 || echo 12)
  r=$(timeout 900 oracle/_ref/shim_bench $d $T 16 4 $mode /tmp/ref.bin)
  b=$(timeout 900 oracle/_ref/shim_bench_b200 $d $T 16 4 $mode /tmp/b200.bin)
  same=$(cmp -s /tmp/ref.bin /tmp/b200.bin && echo true || echo false)
  echo "{\"reference\": $r, \"b200_shim\": $b, \"final_params_bit_identical\": $same}" >> $out
done; done
cat $out
