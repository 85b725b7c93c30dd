"""Real multi-GPU EP (NCCL) parity: launches tests/mp_worker.py with
torch.distributed.run on 2 (and, when present, 4) GPUs.  Skipped on a box with
fewer than 2 GPUs; the host-side multi-rank logic is covered on CPU by
tests/test_abi_cpu.py::test_two_rank_gloo_count_exchange_and_layout."""

import os
import signal
import subprocess
import sys

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.parametrize("a2a", ["nccl", "p2p", "p2p_fused", "p2p_gather", "p2p_ce"])
@pytest.mark.parametrize("n", [2, 4])
def test_ep_over_real_ranks(n, a2a):
    if _ngpus() < n:
        pytest.skip(f"needs {n} GPUs")
    port = 29600 + n + {"nccl": 0, "p2p": 7, "p2p_fused": 13, "p2p_gather": 19, "p2p_ce": 25}[a2a] + os.getpid() % 500
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "tests", "mp_worker.py")]
    env = dict(os.environ, MOE_TEST_A2A=a2a.split("_")[0])
    if a2a == "p2p_fused":
        env["MOE_FUSED_COMBINE"] = "1"       # K6 epilogue returns rows over NVLink
    env["MOE_DISPATCH"] = "gather" if a2a == "p2p_gather" else "scatter"
    if a2a == "p2p_ce":                      # copy-engine data plane (256-row GEMM tiles)
        env["MOE_A2A_CE"] = "1"
        env["MOE_GEMM_CG"] = "2"
    # own process group, so a hung rank is killed together with the launcher
    p = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True, cwd=ROOT, env=env,
                         start_new_session=True)
    try:
        out, _ = p.communicate(timeout=300)
    except subprocess.TimeoutExpired:
        os.killpg(p.pid, signal.SIGKILL)
        out, _ = p.communicate()
        pytest.fail("multi-GPU worker timed out:\n" + out[-4000:])
    assert p.returncode == 0, out[-4000:]
    for rank in range(n):
        assert f"RANK {rank} OK" in out, out[-4000:]


@pytest.mark.parametrize("n,tp,fused", [(2, 2, 0), (2, 2, 1), (4, 2, 0), (4, 2, 1), (4, 4, 1)])
def test_tp_over_real_ranks(n, tp, fused):
    """Tensor parallelism inside the experts (reading G20) over real ranks, P2P."""
    if _ngpus() < n:
        pytest.skip(f"needs {n} GPUs")
    port = 29900 + 10 * n + tp + fused + os.getpid() % 400
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "tests", "mp_worker_tp.py")]
    env = dict(os.environ, MOE_TEST_TP=str(tp), MOE_FUSED_COMBINE=str(fused))
    p = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True, cwd=ROOT, env=env,
                         start_new_session=True)
    try:
        out, _ = p.communicate(timeout=300)
    except subprocess.TimeoutExpired:
        os.killpg(p.pid, signal.SIGKILL)
        out, _ = p.communicate()
        pytest.fail("multi-GPU TP worker timed out:\n" + out[-4000:])
    assert p.returncode == 0, out[-4000:]
    for rank in range(n):
        assert f"RANK {rank} OK" in out, out[-4000:]
