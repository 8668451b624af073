"""Pool checkpoint (kvcomm_anchor_pool_save / kvcomm_anchor_pool_load; SURVEY §5 "pool
dump/load"): a reloaded pool holds the same slots, metadata and stored offsets bit for
bit, matches and realigns exactly like the saved one, and evicts the same anchor next
(LFU state restored) — bf16 and fp8 pools, device and host placement, and into a pool
whose row padding differs."""
import os

import pytest
import torch

import synth

pytestmark = pytest.mark.gpu

L, H, D, DE, CAP, MAXLEN, P = 3, 2, 64, 64, 5, 80, [6, 9]


def _pool(fmt, placement):
    from paper_2510_12872_b200 import kvcomm as K
    return K.AnchorPool(num_layers=L, num_kv_heads=H, head_dim=D, emb_dim=DE, capacity=CAP, max_anchor_len=MAXLEN,
                        prefix_len=P, inv_freq=synth.llama3_inv_freq(D), layer_range=(1, 3), offset_format=fmt,
                        placement=placement)


def _fill(pool, g):
    from paper_2510_12872_b200 import kvcomm as K
    rnd = lambda *s: (torch.randn(*s, generator=g, device="cuda") * 0.15).to(torch.bfloat16)
    Ls = pool.Ls
    lens = [80, 64, 77, 80]
    for i, n in enumerate(lens):
        emb = (torch.randn(n, DE, generator=g, device="cuda") / 8).to(torch.bfloat16)
        offs = [K.OffsetGiven(0, rnd(Ls, H, n, D), rnd(Ls, H, n, D), rnd(Ls, H, P[0], D), rnd(Ls, H, P[0], D))]
        if i != 2:   # slot 2 lacks consumer 1's offsets (presence mask bit clear)
            offs.append(K.OffsetGiven(1, rnd(Ls, H, n, D), rnd(Ls, H, n, D), rnd(Ls, H, P[1], D), rnd(Ls, H, P[1], D)))
        pool.insert(emb, offs)
    pool.record_access([0, 0, 3, 1])
    pool.evict(1)                     # a hole at slot 1
    return rnd


def _state(pool):
    out = []
    for s in range(CAP):
        info = pool.slot_info(s)
        rows = []
        if info["occupied"]:
            for c in range(2):
                if info["ph_present_mask"] >> c & 1:
                    rows.append(pool.read_offsets(s, c, "ph", info["length"]))
                if info["pf_present_mask"] >> c & 1:
                    rows.append(pool.read_offsets(s, c, "pf", P[c]))
        out.append((info, rows))
    return out


def _same(a, b):
    for (ia, ra), (ib, rb) in zip(a, b):
        assert ia == ib
        assert len(ra) == len(rb)
        for x, y in zip(ra, rb):
            for u, v in zip(x, y):
                assert torch.equal(u, v)


@pytest.mark.parametrize("fmt,placement,pad", [("bf16", "device", 0), ("fp8", "device", 0), ("bf16", "host", 0),
                                               ("bf16", "device", 8), ("fp8", "device", 8)])
def test_pool_checkpoint_round_trip(tmp_path, monkeypatch, fmt, placement, pad):
    from paper_2510_12872_b200 import kvcomm as K
    g = torch.Generator(device="cuda").manual_seed(11)
    a = _pool(fmt, placement)
    rnd = _fill(a, g)
    path = str(tmp_path / "pool.kvc")
    a.save(path)
    if pad:   # the loading process pads its rows differently: the file's dense layout still fits
        monkeypatch.setenv("KVCOMM_PH_PAD_ROWS", str(pad))
    b = K.AnchorPool.load(path, device=0)
    monkeypatch.delenv("KVCOMM_PH_PAD_ROWS", raising=False)
    assert (b.Ls, b.Hs, b.d, b.De, b.capacity, b.max_anchor_len, b.prefix_len, b.offset_format) == \
        (a.Ls, a.Hs, a.d, a.De, a.capacity, a.max_anchor_len, a.prefix_len, a.offset_format)
    _same(_state(a), _state(b))

    # matching and realignment through the reloaded pool are bit-identical
    q = (torch.randn(60, DE, generator=g, device="cuda") / 8).to(torch.bfloat16)
    ma, mb = a.match(q, consumer=0, gamma=1.0), b.match(q, consumer=0, gamma=1.0)
    assert ma.candidates == mb.candidates and ma.verdict == mb.verdict and ma.entropy == mb.entropy
    assert torch.equal(ma.W, mb.W) and torch.equal(ma.wbar, mb.wbar)
    base = [torch.randn(a.Ls, H, 60, D, generator=g, device="cuda").to(torch.bfloat16) for _ in range(2)]
    outs = []
    for pool, m in ((a, ma), (b, mb)):
        dk = torch.zeros(a.Ls, H, 90, D, dtype=torch.bfloat16, device="cuda")
        dv = torch.zeros_like(dk)
        K.realign_segment(K.Segment(pool, 0, K.PLACEHOLDER, m.W, m.candidates, base[0], base[1], 0, 20, dk, dv))
        outs.append((dk, dv))
    torch.cuda.synchronize()
    assert torch.equal(outs[0][0], outs[1][0]) and torch.equal(outs[0][1], outs[1][1])

    # LFU state: the next inserts fill the hole, then evict the same victim in both pools
    for _ in range(2):
        emb = (torch.randn(50, DE, generator=g, device="cuda") / 8).to(torch.bfloat16)
        offs = [K.OffsetGiven(0, rnd(a.Ls, H, 50, D), rnd(a.Ls, H, 50, D), rnd(a.Ls, H, P[0], D),
                              rnd(a.Ls, H, P[0], D))]
        assert a.insert(emb, offs) == b.insert(emb, offs)
    _same(_state(a), _state(b))
    a.destroy()
    b.destroy()


def test_pool_load_rejects_truncated_file(tmp_path):
    from paper_2510_12872_b200 import kvcomm as K
    from paper_2510_12872_b200._lib import KVCommError
    g = torch.Generator(device="cuda").manual_seed(5)
    a = _pool("bf16", "device")
    _fill(a, g)
    path = str(tmp_path / "pool.kvc")
    a.save(path)
    data = open(path, "rb").read()
    open(path, "wb").write(data[: len(data) // 2])
    with pytest.raises(KVCommError) as e:
        K.AnchorPool.load(path)
    assert e.value.status_name == "IO"
    open(path, "wb").write(data + b"x")
    with pytest.raises(KVCommError) as e:
        K.AnchorPool.load(path)
    assert e.value.status_name == "IO"
    a.destroy()


def test_embedding_sharded_pool(tmp_path):
    """A pool created with emb_shard=(rank, world) holds only its rank's embedding rows
    (fewer bytes), refuses unsharded matching, and checkpoints exactly (save -> load ->
    save gives the same file, the shard is kept)."""
    from paper_2510_12872_b200 import kvcomm as K
    from paper_2510_12872_b200._lib import KVCommError
    mk = lambda es: K.AnchorPool(num_layers=2, num_kv_heads=2, head_dim=64, emb_dim=64, capacity=3,
                                 max_anchor_len=81, prefix_len=[4], inv_freq=synth.llama3_inv_freq(64),
                                 emb_shard=es)
    dense, shard = mk(None), mk((1, 3))
    assert shard.nbytes() < dense.nbytes()
    g = torch.Generator(device="cuda").manual_seed(9)
    for n in (81, 77, 2):   # partial cycles: rank 1 of 3 holds rows 2-3 of every 6
        emb = torch.randn(n, 64, generator=g, device="cuda").to(torch.bfloat16)
        off = [K.OffsetGiven(0, *(torch.randn(2, 2, m, 64, generator=g, device="cuda").to(torch.bfloat16)
                                  for m in (n, n, 4, 4)))]
        shard.insert(emb, off)
    with pytest.raises(KVCommError) as e:
        shard.match(torch.zeros(10, 64, dtype=torch.bfloat16, device="cuda"))
    assert e.value.status_name == "INVALID_ARGUMENT" and "1/3 of the embedding rows" in str(e.value)
    p1, p2 = str(tmp_path / "a.kvc"), str(tmp_path / "b.kvc")
    shard.save(p1)
    back = K.AnchorPool.load(p1)
    assert back.emb_shard == (1, 3)
    back.save(p2)
    assert open(p1, "rb").read() == open(p2, "rb").read()
    with pytest.raises(KVCommError):
        mk((3, 3))
    dense.destroy(); shard.destroy(); back.destroy()


def test_pool_load_rejects_corrupt_slot_metadata(tmp_path):
    """A checkpoint whose LFU metadata no pool could have produced is an IO error: an
    insertion index at or past the counter, two slots sharing an index, or a presence
    bit at or above the consumer count (they would silently change the A17 tie-break)."""
    import struct
    from paper_2510_12872_b200 import kvcomm as K
    from paper_2510_12872_b200._lib import KVCommError
    g = torch.Generator(device="cuda").manual_seed(6)
    a = _pool("bf16", "device")
    _fill(a, g)
    path = str(tmp_path / "pool.kvc")
    a.save(path)
    a.destroy()
    data = bytearray(open(path, "rb").read())
    # header: magic 8 + version 4 + 16 config ints + emb shard 2 x int32 + prefix_len[C] + inv_freq[d/2]
    counter = 8 + 4 + 16 * 4 + 8 + 4 * len(P) + 8 * (D // 2)
    slot0 = counter + 8   # per slot: occupied i32, length i32, access i64, inserted i64, ph/pf masks u64
    next_index = struct.unpack_from("<q", data, counter)[0]
    assert next_index == 4 and struct.unpack_from("<i", data, slot0)[0] == 1
    back = K.AnchorPool.load(path)   # the unmodified file loads
    back.destroy()
    accepted = []
    for field, value in ((16, next_index), (16, 2), (24, 1 << len(P))):   # slot 2 holds index 2
        bad = bytearray(data)
        struct.pack_into("<q", bad, slot0 + field, value)
        open(path, "wb").write(bytes(bad))
        try:
            K.AnchorPool.load(path).destroy()
            accepted.append((field, value))
        except KVCommError as e:
            assert e.status_name == "IO" and "slot" in str(e), (field, value, str(e))
    assert not accepted, accepted
