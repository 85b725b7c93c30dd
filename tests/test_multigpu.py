"""Real multi-GPU EP (NCCL) parity: launches tests/mp_worker.py with
torch.distributed.run on 2 (and, when present, 4) GPUs.  Skipped on a box with
fewer than 2 GPUs; the host-side multi-rank logic is covered on CPU by
tests/test_abi_cpu.py::test_two_rank_gloo_count_exchange_and_layout."""

import os
import subprocess
import sys

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.parametrize("a2a", ["nccl", "p2p"])
@pytest.mark.parametrize("n", [2, 4])
def test_ep_over_real_ranks(n, a2a):
    if _ngpus() < n:
        pytest.skip(f"needs {n} GPUs")
    port = 29600 + n + (7 if a2a == "p2p" else 0) + os.getpid() % 500
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "tests", "mp_worker.py")]
    env = dict(os.environ, MOE_TEST_A2A=a2a)
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    for rank in range(n):
        assert f"RANK {rank} OK" in out, out[-4000:]
