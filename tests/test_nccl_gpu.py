"""The NCCL data plane itself (ncclSend/Recv halo planes on the exchange
communicator, the in-place all-reduces of the LLG statistics, the
non-monotone continuation), one process per GPU under torchrun, bit for bit
against the reference goldens -- with the overlapped and the serialised
exchange.  Needs >= 2 GPUs (NCCL refuses two ranks on one device); on the
one-GPU pool the same plan runs through the in-process emulation
(tests/test_slab_gpu.py)."""

import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
CASES = ["mixed3d", "allmur3d", "zwall_magnet", "two_magnets", "bias3d", "cpw_small",
         "nonmono3d", "fail3d"]


def _gpus() -> int:
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


# nproc 1: the same driver (torchrun, process group, gather) on one GPU, so
# the host side of this test runs on the one-GPU pool too
@pytest.mark.parametrize("overlap", ["1", "0"])
@pytest.mark.parametrize("nproc", [1, 2, 3, 4])
def test_nccl_slabs_match_reference_goldens(nproc, overlap):
    if _gpus() < nproc:
        pytest.skip(f"needs {nproc} GPUs (NCCL: one rank per GPU)")
    env = dict(os.environ, MPB_OVERLAP=overlap, MPB_SWEEP_MINCHUNK="2")
    out = subprocess.run(
        [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
         f"--nproc-per-node={nproc}", "--master-addr=127.0.0.1", f"--master-port={_port()}",
         str(ROOT / "tests" / "nccl_worker.py")] + CASES,
        cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    for name in CASES:
        assert any(line.startswith(f"OK {name}") for line in out.stdout.splitlines()), name
