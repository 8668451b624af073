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


def test_grid_shard_partitions_layers_and_heads():
    """70B runs layer groups x KV-head groups (4 x 2 on 8 GPUs)."""
    for L, H, lg, hg in ((80, 8, 4, 2), (32, 8, 8, 1), (4, 4, 1, 4), (5, 3, 2, 3)):
        cover = np.zeros((L, H), dtype=int)
        for r in range(lg * hg):
            (lb, le), (hb, he) = shard.grid_shard(L, H, r, lg, hg)
            cover[lb:le, hb:he] += 1
            assert (lb, le) == shard.layer_shard(L, r // hg, lg) and (hb, he) == shard.head_shard(H, r % hg, hg)
        assert (cover == 1).all()
    assert shard.grid_shard(80, 8, 5, 4, 2) == ((40, 60), (4, 8))
    with pytest.raises(ValueError):
        shard.grid_shard(8, 2, 0, 2, 3)


def _oracle_realign_block(lb, le, hb, he, seed):
    """Per-agent realigned caches of the (layer, head) block via the oracle."""
    return [(k[:, hb:he].contiguous(), v[:, hb:he].contiguous()) for k, v in _oracle_realign_layers(lb, le, seed)]


def _grid_worker(rank, world, hg, port, result_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    L, H = 4, 2
    (lb, le), (hb, he) = shard.grid_shard(L, H, rank, world // hg, hg)
    mine = _oracle_realign_block(lb, le, hb, he, seed=9)
    agents = [1, 2, 3]
    full = [(torch.zeros((L, H) + tuple(k.shape[2:])), torch.zeros((L, H) + tuple(k.shape[2:])))
            if shard.consumer_rank(a, world) == rank else (None, None) for a, (k, _) in zip(agents, mine)]
    shard.gather_to_consumers(agents, mine, full, L, rank, world, head_groups=hg)
    ref = _oracle_realign_layers(0, L, seed=9)
    ok = True
    for a, (fk, fv), (rk, rv) in zip(agents, full, ref):
        if shard.consumer_rank(a, world) == rank:
            ok &= torch.equal(fk, rk) and torch.equal(fv, rv)
    result_q.put((rank, ok))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,hg", [(2, 2), (4, 2)])
def test_gather_head_blocks_gloo_equals_unsharded(world, hg):
    """Head blocks are not contiguous in the consumer's [L, H, N, d] cache: they are
    received into staging buffers and permuted into place."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_grid_worker, args=(r, world, hg, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
    res = dict(q.get(timeout=5) for _ in range(world))
    assert all(p.exitcode == 0 for p in procs)
    assert res == {r: True for r in range(world)}


class _FakePlan:
    """Stands in for kvcomm.Plan in the host-logic test of shard.MatchShard."""

    def __init__(self, rank, size, fail_shard=False):
        self.rank, self.size, self.fail_shard = rank, size, fail_shard
        self.calls = []

    def match_handle(self):
        return bytes([self.rank]) * 64, self.size

    def match_shard(self, rank, world, handles=()):
        if self.fail_shard and world > 1:
            raise RuntimeError("cannot open peer buffers")
        self.calls.append(("shard", rank, world, [h[0] for h in handles]))

    def run_begin(self, queries, stream=None):
        self.calls.append(("begin",))

    def run_end(self, sync=False, stream=None):
        self.calls.append(("end",))


def _match_shard_worker(rank, world, port, case, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        size = 100 + (rank if case == "size" else 0)
        plan = _FakePlan(rank, size, fail_shard=(case == "fail" and rank == 1))
        try:
            ms = shard.MatchShard(plan, rank, world, device=0)
        except RuntimeError as e:
            q.put((rank, "raised", str(e), plan.calls))
            return
        orig = shard.stream_barrier
        shard.stream_barrier = lambda flag, group=None: (plan.calls.append(("barrier",)), dist.barrier(group=group))
        try:
            ms.run([None])
        finally:
            shard.stream_barrier = orig
        ms.close()
        q.put((rank, "ok", "", plan.calls))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", ["ok", "fail", "size"])
def test_match_shard_handshake_gloo(case):
    """shard.MatchShard: every rank receives the handles in rank order and its own rank /
    world; a failure on one rank (or plans of different layouts) raises on ALL ranks and
    leaves no rank sharded; a run is begin -> cross-rank barrier -> end."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_match_shard_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        r, status, msg, calls = q.get(timeout=120)
        out[r] = (status, msg, calls)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    if case == "ok":
        for r in range(world):
            status, _, calls = out[r]
            assert status == "ok"
            assert calls[0] == ("shard", r, world, [0, 1])
            assert calls[1:4] == [("begin",), ("barrier",), ("end",)]
            assert calls[4] == ("shard", 0, 1, [])
    else:
        for r in range(world):
            status, msg, calls = out[r]
            assert status == "raised", out
            assert "sharded matching unavailable" in msg
            sharded = [c for c in calls if c[0] == "shard" and c[2] > 1]
            unsharded_after = [c for c in calls if c[0] == "shard" and c[2] == 1]
            assert not sharded or unsharded_after, calls   # nobody left sharded
        if case == "size":
            assert "differ across ranks" in out[0][1]


def test_peer_destinations_of_a_head_block_keep_the_full_layer_stride():
    """PeerCaches.destinations(i, layer_range, head_range): the block's first row sits at
    ((l0 * H + h0) * N) * d of the consumer's full cache and its layers are H head
    blocks apart, which the binding passes to the plan as dst_heads = H."""
    from paper_2510_12872_b200 import kvcomm as K
    pc = shard.PeerCaches.__new__(shard.PeerCaches)
    pc.H, pc.d, pc.agents, pc.ptrs = 8, 128, [(1, 100)], [(1 << 20, 1 << 30)]
    dk, dv = pc.destinations(0, (20, 40), (4, 8))
    assert dk.data_ptr() == (1 << 20) + (20 * 8 + 4) * 100 * 128 * 2
    assert dv.data_ptr() == (1 << 30) + (20 * 8 + 4) * 100 * 128 * 2
    assert tuple(dk.shape) == (20, 4, 100, 128) and dk.stride() == (8 * 100 * 128, 100 * 128, 128, 1)
    assert K._dst_layout(dk, "dst") == (100, 8)
    full = pc.destinations(0, (0, 80))[0]
    assert full.stride() == (8 * 100 * 128, 100 * 128, 128, 1) and K._dst_layout(full, "dst") == (100, 8)
