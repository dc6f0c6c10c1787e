# 4 GPUs: 8-process (2 per GPU) multi-GPU parity -- the G=8 plans, one-shot, push and chain tables
DSS_TEST_OVERSUBSCRIBE=1 timeout 1500 python -m pytest tests/test_multi_gpu.py -q -k "8" -s > gpurun_out/mgpu_3j.log 2>&1; echo mgpu8=$?; grep -E "case|MGPU|passed|failed|Error" gpurun_out/mgpu_3j.log | tail -60
