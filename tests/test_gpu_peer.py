"""The fused gather (include/kvcomm.h kvcomm_ipc_*, shard.PeerCaches): 2 ranks on one
GPU over gloo write their layer blocks into the consumer rank's IPC-shared caches; the
result equals the unsharded run bit for bit (tests/peer_worker.py)."""
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
@pytest.mark.parametrize("fmt,match,top_k,world,sim,scal,pipe", [
    ("bf16", "replicated", 0, 2, "l2", "frobenius", "no"), ("fp8", "replicated", 0, 2, "l2", "frobenius", "no"),
    ("bf16", "shard-match", 0, 2, "l2", "frobenius", "no"), ("fp8", "shard-match", 0, 2, "l2", "frobenius", "no"),
    ("bf16", "shard-match", 2, 2, "l2", "frobenius", "no"), ("bf16", "shard-match", 0, 3, "l2", "frobenius", "no"),
    ("bf16", "shard-match", 0, 2, "cosine", "frobenius", "no"), ("bf16", "shard-match", 0, 3, "l2", "mean_l2", "no"),
    ("bf16", "shard-match-emb", 0, 2, "l2", "frobenius", "no"), ("fp8", "shard-match-emb", 2, 3, "cosine", "frobenius", "no"),
    ("bf16", "shard-match-emb", 1, 4, "l2", "mean_l2", "no"),
    ("bf16", "shard-match", 0, 2, "l2", "frobenius", "pipe"), ("fp8", "shard-match-emb", 2, 3, "l2", "frobenius", "pipe")])
def test_fused_gather_multi_rank_bit_exact(fmt, match, top_k, world, sim, scal, pipe):
    """Also: sharded matching (kvcomm_plan_match_shard) gives weights, verdicts and
    caches bit-identical to the unsharded run (dense and top-k weights; 3 ranks split
    the 48 and 20 position blocks of the two sample lengths unevenly; the cosine
    variant's three partial sums and the mean-l2 scalar distance; pools that hold only
    their rank's embedding rows, shard-match-emb; "pipe": the bench's N > 1 schedule, every
    realign on a second stream and the runs issued back to back)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.join(ROOT, "tests", "peer_worker.py"),
           fmt, match, str(top_k), sim, scal, pipe]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    hosted = [sum(1 for m in range(1, 6) if (m - 1) % world == rank) for rank in range(world)]
    for rank in range(world):
        assert f"rank {rank}: {hosted[rank]} agents bit-exact" in r.stdout, r.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["shard-mismatch", "shard-mismatch-empty", "shard-mismatch-replace"])
def test_sharded_matching_detects_out_of_step_pools(mode):
    """Ranks whose pools differ (rank 1 evicted an anchor; or every anchor so that it has
    no job at all; or its full pool replaced the anchor in slot 0 by another of the same
    length, so the candidate slot ids still agree) must not blend with each other's weights: every job whose layout
    fingerprints differ is NewAnchor (SHARD_MISMATCH), no agent is realigned, and
    results() raises SHAPE_MISMATCH (rank 1 with empty pools: host verdicts EMPTY_POOL)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.join(ROOT, "tests", "peer_worker.py"),
           "bf16", mode, "0"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "rank 0: 3 agents untouched, mismatch reported" in r.stdout, r.stdout
    assert "rank 1: 2 agents untouched, mismatch reported" in r.stdout, r.stdout


@pytest.mark.gpu
def test_per_thread_store_path_equals_bulk_store():
    """KVCOMM_STORE_STG=1 forces the peer-destination store path (per-thread STG) for
    every segment; it must write exactly the bytes the TMA bulk-store path writes."""
    code = ("import sys, torch; sys.path.insert(0, %r); sys.path.insert(0, %r); import synth, harness; "
            "p = synth.make_problem(5, L=2, H=2, d=64, D_e=64, L_phi=150, anchor_lens=[150, 170, 190], "
            "prefix_lens=[20], target_start=30, pf_base_start=30, inv_freq=synth.llama3_inv_freq(64)); "
            "g = harness.run_gpu(p, gamma=1.0); torch.save((g['dst_k'], g['dst_v']), sys.argv[1])"
            % (ROOT, os.path.join(ROOT, "tests")))
    import tempfile
    import torch
    outs = []
    with tempfile.TemporaryDirectory() as td:
        for stg in ("0", "1"):
            f = os.path.join(td, f"out{stg}.pt")
            env = dict(os.environ, KVCOMM_STORE_STG=stg)
            r = subprocess.run([sys.executable, "-c", code, f], cwd=ROOT, env=env, capture_output=True, text=True,
                               timeout=600)
            assert r.returncode == 0, r.stderr[-3000:]
            outs.append(torch.load(f))
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])
