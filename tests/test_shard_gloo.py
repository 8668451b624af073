"""Multi-GPU path host logic on CPU (-m "not gpu"): layer sharding, consumer placement
and the targeted gather of realigned layer blocks, with world_size 2 over gloo.

The per-rank compute stand-in is the oracle applied to the rank's layer block (the
realignment is independent per layer); the gathered cache on each
consumer rank must equal the unsharded oracle result bit for bit (T2/T3 of SURVEY
§4)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2510_12872_b200 import shard

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_layer_shard_partitions_all_layers():
    for L in (1, 7, 32, 80):
        for G in (1, 2, 3, 4, 8):
            if G > L:
                continue
            blocks = [shard.layer_shard(L, r, G) for r in range(G)]
            assert blocks[0][0] == 0 and blocks[-1][1] == L
            assert all(a[1] == b[0] for a, b in zip(blocks, blocks[1:]))
            sizes = [e - b for b, e in blocks]
            assert max(sizes) - min(sizes) <= 1
    assert [shard.consumer_rank(m, 2) for m in range(1, 6)] == [0, 1, 0, 1, 0]
    assert [shard.consumer_rank(m, 8) for m in range(1, 6)] == [0, 1, 2, 3, 4]
    with pytest.raises(ValueError):
        shard.layer_shard(8, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_realign_layers(lb, le, seed):
    """Deterministic per-agent realigned caches of layers [lb, le) via the oracle."""
    import sys
    sys.path.insert(0, ROOT)
    from oracle import kvcomm_oracle as O
    import synth
    L, H, d, T, k = 4, 2, 16, 6, 3
    out = []
    for agent in (1, 2, 3):
        rng = np.random.default_rng(seed + agent)
        bk = rng.standard_normal((L, H, T, d))
        bv = rng.standard_normal((L, H, T, d))
        offs = [rng.standard_normal((L, H, T, d)) * 0.15 for _ in range(k)]
        W = O.position_weights(np.abs(rng.standard_normal((T, k))))[0]
        r = O.realign_segment(W, bk[lb:le], bv[lb:le], [o[lb:le] for o in offs], [o[lb:le] for o in offs], 0,
                              10 * agent, synth.plain_inv_freq(d))
        out.append((torch.from_numpy(r["k"]).to(torch.float32), torch.from_numpy(r["v"]).to(torch.float32)))
    return out


def _worker(rank, world, port, result_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    L = 4
    lb, le = shard.layer_shard(L, rank, world)
    mine = _oracle_realign_layers(lb, le, seed=7)
    agents = [1, 2, 3]
    full = []
    for a, (k, v) in zip(agents, mine):
        if shard.consumer_rank(a, world) == rank:
            full.append((torch.zeros((L,) + tuple(k.shape[1:])), torch.zeros((L,) + tuple(v.shape[1:]))))
        else:
            full.append((None, None))
    shard.gather_to_consumers(agents, [(k.contiguous(), v.contiguous()) for k, v in mine], full, L, rank, world)
    ref = _oracle_realign_layers(0, L, seed=7)
    ok = True
    for a, (fk, fv), (rk, rv) in zip(agents, full, ref):
        if shard.consumer_rank(a, world) == rank:
            ok &= torch.equal(fk, rk) and torch.equal(fv, rv)
    result_q.put((rank, ok))
    dist.barrier()
    dist.destroy_process_group()


def test_gather_to_consumers_world2_gloo_equals_unsharded():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    res = dict(q.get(timeout=5) for _ in range(2))
    assert all(p.exitcode == 0 for p in procs)
    assert res == {0: True, 1: True}
