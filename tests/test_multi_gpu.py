"""Multi-GPU parity: every cross-GPU path (one-shot, fused push two-shot,
ordered chain, unfused pull two-shot; one process per GPU) is bit-exact with
the fp32 oracle, and ranks with mismatched geometry refuse to attach.
Needs >= G GPUs (gpurun --gpus 2/4); skipped on single-GPU boxes.

These cases are NOT emulated by running G processes on one GPU: the
cross-GPU kernels spin on flags that other ranks' kernels release, and on
this driver such waiting kernels in separate processes on one device are
not guaranteed to run concurrently (the B200 profiling guide records
Xid 109 context-switch timeouts from exactly that).  On one GPU the same
plans are exercised as a single-process world (every other test), and the
multi-process host logic by the gloo tests in test_dist_cpu.py."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]


def _ngpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.parametrize("G", [2, 4, 8])
def test_two_shot_nvlink_bit_exact(G):
    if _ngpus() < G:
        pytest.skip(f"needs {G} GPUs (one process per GPU; see the module docstring)")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={G}",
           "--master-addr=127.0.0.1", f"--master-port={29600 + G}", os.path.join(ROOT, "tests", "mgpu_worker.py")]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    print(p.stdout)  # every case's line (the logs under profiles/ are this output)
    print(p.stderr[-4000:])
    assert p.returncode == 0 and "MGPU PASS" in p.stdout
