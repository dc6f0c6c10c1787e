timeout 1200 python -m pytest tests -m "gpu and not multigpu" -x -q > gpurun_out/pytest_1c.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_1c.log
timeout 900 python bench_sweep.py --gpus 1 --max-mb 1024 > gpurun_out/sweep_g1.jsonl 2> gpurun_out/sweep_g1.err; echo sweep1=$?
