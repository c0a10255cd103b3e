"""Row-block sharded solve across real ranks (
PAPER.md:1239-1247 on GS as a parallel step): torchrun with one GPU per rank, NCCL
halos and reduction partials, bit-identical to the oracle on the whole system —
with every rank holding the global matrix, and with each rank holding only its own
rows (local input, the weak-scaling layout); the reductions' shard values by
ncclAllGather or by device-initiated peer stores (peer_reduce, CUDA IPC over NVLink).  Needs >= 2 GPUs; skipped otherwise
(the host-side logic is covered over gloo in test_shard_host.py)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _gpus():
    torch = pytest.importorskip("torch")
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("local", [False, True])
@pytest.mark.parametrize("peer", [False, True])
def test_sharded_solve_across_ranks(world, local, peer):
    if _gpus() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29700 + world + 10 * local + 20 * peer),
           os.path.join(ROOT, "tools", "shard_rank.py"), "--N", "16"] + (["--local"] if local else []) + \
        (["--peer"] if peer else [])
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert '"equal": true' in r.stdout
