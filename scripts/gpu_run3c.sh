timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "edge or batched" > gpurun_out/pytest_3c.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_3c.log
