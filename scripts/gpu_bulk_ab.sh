DSS_LIB_VARIANT=build/variants/libdssync_b200_bulk.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "f32_bit_exact or golden_traj" > gpurun_out/pytest_bulk.log 2>&1; echo pytest_bulk=$?; tail -1 gpurun_out/pytest_bulk.log
for v in base bulk bulk512; do
  if [ $v = base ]; then unset DSS_LIB_VARIANT; else export DSS_LIB_VARIANT=build/variants/libdssync_b200_$v.so; fi
  for c in c4slice c3; do
    timeout 400 python bench.py --config $c --steps 40 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/bulk_${v}_$c.log 2>&1; echo "$v $c rc=$?"
  done
done
