"""The layer x KV-head grid (70B "layer groups x KV-head groups"; BASELINE
configs[3] runs 4 x 2 on 8 GPUs): every rank of a grid on one GPU realigns its (layer,
head) block and delivers it to the consumer's full cache — fused into the realign
epilogue (IPC-mapped destination with the full cache's layer stride) or through the
targeted gather with staging + local permute — and the result equals the unsharded
run bit for bit (tests/grid_worker.py).  (-m gpu)"""
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.gpu
@pytest.mark.parametrize("wl,lg,hg,gather,match", [
    ("segment", 4, 2, "fused", "shard-match"),     # configs[3]'s 4 x 2 grid on 8 ranks
    ("segment", 4, 2, "nccl", "replicated"),
    ("segment", 1, 2, "fused", "replicated"),      # heads only
    ("five", 2, 2, "fused", "shard-match"),        # 5 consumers on 4 ranks
    ("five", 2, 2, "nccl", "shard-match"),
])
def test_grid_bit_exact(wl, lg, hg, gather, match):
    world = lg * hg
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.join(ROOT, "tests", "grid_worker.py"),
           wl, str(lg), str(hg), gather, match]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    n_agents = 5 if wl == "five" else 1
    for rank in range(world):
        hosted = sum(1 for m in range(1, n_agents + 1) if (m - 1) % world == rank)
        assert f"rank {rank}: {hosted} agents bit-exact" in r.stdout, r.stdout
