# A/B of kernel tuning variants on one box (same GPU for every variant).
for v in base m8mb1 m8mb2 ad2 mb1; do
  if [ $v = base ]; then unset DSS_LIB_VARIANT; else export DSS_LIB_VARIANT=build/variants/libdssync_b200_$v.so; fi
  for c in c3 c4slice; do
    timeout 300 python bench.py --config $c --steps 60 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/ab_${v}_$c.log 2>&1
    echo "$v $c rc=$?"
  done
done
unset DSS_LIB_VARIANT
timeout 600 oracle/_ref/ref_unit_tests_b200 > gpurun_out/ref_unit_b200.log 2>&1; echo refunit=$?; tail -3 gpurun_out/ref_unit_b200.log
