# logistic + run-driver parity, then the whole single-GPU suite
timeout 900 python -m pytest tests/test_gpu_logistic.py tests/test_gpu_cli.py -q > gpurun_out/pytest_2b.log 2>&1; echo new=$?; tail -3 gpurun_out/pytest_2b.log
timeout 1200 python -m pytest tests -m gpu -q -k "not multi" > gpurun_out/pytest_2b_all.log 2>&1; echo all=$?; tail -2 gpurun_out/pytest_2b_all.log
