"""Multi-GPU domain decomposition on real GPUs (skipped with < 2 devices):
slab-decomposed forces / energies / pair counts against one GPU, with the
NVLink peer exchanges overlapped with the force kernel (nbx_dd_force), and
the overlapped, sequential-peer and NCCL paths bit-identical."""

import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
REPO = Path(__file__).resolve().parents[1]


def _ngpu():
    import torch

    return torch.cuda.device_count()


def _torchrun(n, script, *args, port):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(REPO / "tools" / script), *args]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=REPO, env=dict(os.environ))
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    return r.stdout


@pytest.mark.skipif(_ngpu() < 2, reason="needs 2 GPUs")
def test_dd_overlapped_p2p_matches_one_gpu():
    out = _torchrun(2, "dd_check.py", "--atoms", "96000", "--p2p", port=29571)
    assert "DD PARITY OK" in out, out


@pytest.mark.skipif(_ngpu() < 2, reason="needs 2 GPUs")
def test_dd_exchange_paths_bit_identical():
    out = _torchrun(2, "dd_p2p_check.py", "96000", port=29572)
    assert "bit-identical on every rank: True" in out and "timeouts: False" in out, out


@pytest.mark.skipif(_ngpu() < 2, reason="needs 2 GPUs")
def test_dd_migration_matches_allgather_assign():
    out = _torchrun(2, "dd_migrate_check.py", "96000", port=29573)
    assert "MIGRATE PARITY OK" in out, out
