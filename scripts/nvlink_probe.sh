#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"; mkdir -p gpurun_out
{
nvidia-smi nvlink -h 2>&1 | head -80
echo ---- status; nvidia-smi nvlink -s -i 0 2>&1 | head -30
echo ---- gt d; nvidia-smi nvlink -gt d -i 0 2>&1 | head -40
echo ---- gt r; nvidia-smi nvlink -gt r -i 0 2>&1 | head -10
python - <<'PY'
import subprocess, torch, time
def ctr(dev):
    out = subprocess.run(["nvidia-smi", "nvlink", "-gt", "d", "-i", str(dev)], capture_output=True, text=True).stdout
    return out
a = torch.empty(1 << 28, dtype=torch.float32, device="cuda:0")  # 1 GiB
b = torch.empty(1 << 28, dtype=torch.float32, device="cuda:1")
b.copy_(a); torch.cuda.synchronize()
before0, before1 = ctr(0), ctr(1)
for _ in range(10):
    b.copy_(a)
torch.cuda.synchronize()
time.sleep(1.5)
after0, after1 = ctr(0), ctr(1)
print("==== gpu0 before"); print(before0[:3000]); print("==== gpu0 after"); print(after0[:3000])
print("==== gpu1 after"); print(after1[:1500])
PY
} > gpurun_out/nvlink_probe.log 2>&1
tail -30 gpurun_out/nvlink_probe.log
