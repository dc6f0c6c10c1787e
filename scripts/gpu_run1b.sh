timeout 900 python -m pytest tests -m "gpu and not multigpu" -x -q > gpurun_out/pytest_1b.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_1b.log
timeout 300 python bench.py --config c3 --steps 60 --warmup 3 --no-cpu-baseline --e2e-steps 3 > gpurun_out/b1b_c3.log 2>&1; echo c3=$?
timeout 300 python bench.py --config c1 --steps 2000 --warmup 5 --no-cpu-baseline > gpurun_out/b1b_c1.log 2>&1; echo c1=$?
timeout 600 bash profiles/run_profile.sh c4slice ds_group_kernel 40000000; echo prof1=$?
timeout 600 bash profiles/run_profile.sh c4slice bsp_kernel 40000000; echo prof2=$?
