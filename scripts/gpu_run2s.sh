timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_2s.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_2s.log
grep -E "stats=6|MGPU" gpurun_out/pytest_2s.log | head
timeout 300 python bench.py --steps 300 --warmup 5 > gpurun_out/bench_2s.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench_2s.log | cut -c1-300
