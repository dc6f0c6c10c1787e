# 1 GPU: L2 prefetch of the next member chunk (stateful groups of 8) A/B
for v in base nopf base nopf; do
  if [ $v = base ]; then unset DSS_LIB_VARIANT; else export DSS_LIB_VARIANT=build/variants/libdssync_b200_$v.so; fi
  for c in c4slice c3; do
    timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/pf_${v}_$c.log 2>&1
    tail -1 gpurun_out/pf_${v}_$c.log | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', '$c', round(d['value'],2), 'bsp', round(d['bsp']['iters_s'],2), 'roof', round(d['roofline']['frac'],3))"
  done
done
