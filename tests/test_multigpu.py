"""Multi-GPU path (one process per GPU; APPP hops over NCCL send/recv or the P2P pull transport):
bit-identical to virtual tiles on one GPU.  Runs only where >= 2 GPUs are visible."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpu():
    import torch
    return torch.cuda.device_count()


@pytest.mark.parametrize("transport", ["nccl", "p2p"])
@pytest.mark.parametrize("world", [2, 4])
def test_multi_gpu_bit_identical(world, transport):
    if _ngpu() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + world), os.path.join(ROOT, "tests", "mgpu_check.py")]
    env = dict(os.environ, PTYCHO_APPP_TRANSPORT=transport)
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    print(out.stdout[-4000:], out.stderr[-4000:])
    assert out.returncode == 0
    assert "MGPU OK" in out.stdout
