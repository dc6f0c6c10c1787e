timeout 1500 python bench_sweep.py > gpurun_out/sweep_full_g1.jsonl 2>gpurun_out/sweep_full_g1.err; echo g1=$?; wc -l gpurun_out/sweep_full_g1.jsonl
for c in c3 c4slice; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${c}_2v.log 2>&1; echo $c=$?
  tail -1 gpurun_out/bench_${c}_2v.log | python3 -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'][:40], round(d['value'],2), 'bsp', round(d['bsp']['iters_s'],2), 'roof', round(d['roofline']['frac'],3))"
done
