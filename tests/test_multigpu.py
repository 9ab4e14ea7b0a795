"""Multi-GPU ring over NVLink (symmetric-memory peer stores): parity on every rank,
including a remote restore.  Runs under torchrun when >= 2 GPUs are visible."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpu():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.parametrize("n,transport", [(2, "p2p"), (2, "nccl"), (2, "runsteps"), (2, "loop"),
                                         (2, "r9"), (2, "shared"),
                                         (4, "p2p"), (4, "nccl"), (4, "runsteps"), (4, "loop"),
                                         (4, "shared"),
                                         (8, "p2p")])
def test_ring_over_nvlink_parity(n, transport):
    """p2p: fused ring-put over NVLink; nccl: the comparison transport (bit-exact too);
    runsteps / loop: the native decode loops (kv_run_steps on two streams, the
    one-launch-per-step kv_loop) over
    NVLink; r9: a reader on the holder's GPU acquires seq while the predecessor keeps
    publishing and checks each observed step's table and newest tokens (reading R9);
    shared: NEXT-3 with every holder on another rank (mirrors, pulls over NVLink,
    evictions and drops, a failure restored from the remote-shared holder)."""
    if _ngpu() < n:
        pytest.skip(f"needs {n} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + n),
           os.path.join(ROOT, "tests", "mgpu_worker.py")]
    env = dict(os.environ, KV_TRANSPORT=transport)
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    out = r.stdout + r.stderr
    assert r.returncode == 0 and "MGPU_PARITY_OK" in out, out[-4000:]
