"""BASELINE.json configs[3] at full per-GPU size: Llama-3-70B shape (80 layers, 8 KV
heads x 128, D_e 8192), a 3072-token shared segment (+ 32-token prefix), 256-anchor
pool, k = 256, layer + KV-head sharded 4 x 2 over 8 GPUs.  One GPU holds one shard
(layers [0,20), heads [0,4): 30 GiB of offsets + 12.9 GB of replicated embeddings);
this test realigns exactly that shard, in the plan's launch configuration, and
checks it against the oracle: all per-position distances of 4 anchors and of 8
sampled positions for all 256 anchors, w̄ / entropy / verdict over the whole sample,
and realigned K/V rows at sampled (token, layer, head) positions.  (-m gpu)
"""
import numpy as np
import pytest
import torch

import synth
from oracle import kvcomm_oracle as O
from synth.state import keyed_gen
from tests import harness

pytestmark = pytest.mark.gpu

L, H, D, DE = 80, 8, 128, 8192
LAYERS, HEADS = (0, 20), (0, 4)
T, P, M, N_VOCAB = 3072, 32, 256, 128256
SEED = 70


def _offset(slot, kind, plane):
    Ls, Hs = LAYERS[1] - LAYERS[0], HEADS[1] - HEADS[0]
    n = T if kind == "ph" else P
    g = keyed_gen(SEED, "c4off", slot, kind, plane)
    return (torch.randn(Ls, Hs, n, D, generator=g, device="cuda") * synth.OFFSET_STD).to(torch.bfloat16)


def _ids(slot):
    return torch.randint(0, N_VOCAB, (T,), generator=keyed_gen(SEED, "c4ids", slot), device="cuda")


@pytest.fixture(scope="module")
def c4():
    import paper_2510_12872_b200 as kv
    g = keyed_gen(SEED, "c4vocab")
    vocab = (torch.randn(N_VOCAB, DE, generator=g, device="cuda") / np.sqrt(DE)).to(torch.bfloat16)
    inv = synth.llama3_inv_freq(D)
    pool = kv.AnchorPool(num_layers=L, num_kv_heads=H, head_dim=D, emb_dim=DE, capacity=M, max_anchor_len=T,
                         prefix_len=[P], inv_freq=inv, layer_range=LAYERS, head_range=HEADS)
    for s in range(M):
        pool.insert(vocab[_ids(s)], [kv.OffsetGiven(0, _offset(s, "ph", 0), _offset(s, "ph", 1),
                                                    _offset(s, "pf", 0), _offset(s, "pf", 1))])
    gq = keyed_gen(SEED, "c4query")
    ids0 = _ids(0)
    swap = torch.rand(T, generator=gq, device="cuda") < 0.3
    q_ids = torch.where(swap, torch.randint(0, N_VOCAB, (T,), generator=gq, device="cuda"), ids0)
    query = vocab[q_ids].contiguous()
    Ls, Hs = LAYERS[1] - LAYERS[0], HEADS[1] - HEADS[0]
    gb = keyed_gen(SEED, "c4base")
    base = [torch.randn(Ls, Hs, T, D, generator=gb, device="cuda").to(torch.bfloat16) for _ in range(2)]
    pfb = [torch.randn(Ls, Hs, P, D, generator=gb, device="cuda").to(torch.bfloat16) for _ in range(2)]
    p0 = [torch.randn(Ls, Hs, 200, D, generator=gb, device="cuda").to(torch.bfloat16) for _ in range(2)]
    N = 200 + T + P
    dst = [torch.empty(Ls, Hs, N, D, dtype=torch.bfloat16, device="cuda") for _ in range(2)]
    segs = [kv.PlanSegment(0, 0, kv.PLACEHOLDER, 0, base[0], base[1], 0, 200),
            kv.PlanSegment(0, 0, kv.PREFIX, 0, pfb[0], pfb[1], 200, 200 + T),
            kv.PlanSegment(0, 0, kv.COPY, 0, p0[0], p0[1], 0, 0)]
    plan = kv.Plan([(pool, T, 0.3, 0)], segs, [(N, dst[0], dst[1])])
    m = pool.match(query, consumer=0, gamma=0.3, want_dist=True)      # exposes the distances
    plan.run([query], sync=True)
    ms, reused = plan.results()
    torch.cuda.synchronize()
    out = dict(vocab=vocab, query=query, ids=[None] * M, pool=pool, m=m, plan_match=ms[0], reused=reused,
               base=base, pfb=pfb, p0=p0, dst=dst, inv=inv)
    yield out
    plan.destroy()
    pool.destroy()
    torch.cuda.empty_cache()


_ORACLE = {}


def _oracle_columns(c4):
    """Oracle per-position distances of all 256 anchors (256 x 3072 fp64 = 6 MB, each
    computed from its own anchor) and the Frobenius d̄ (reading A4), cached."""
    if "dbar" not in _ORACLE:
        q = harness.f64(c4["query"])
        dbar_sq = np.zeros(M)
        cols = {}
        for s in range(M):
            col = O.distances(q, [harness.f64(c4["vocab"][_ids(s)])])[:, 0]
            dbar_sq[s] = np.sum(col * col)
            cols[s] = col
        _ORACLE["dbar"] = np.sqrt(dbar_sq)
        _ORACLE["cols"] = cols
    return _ORACLE


def test_config4_distances_weights_verdict(c4):
    m, pm = c4["m"], c4["plan_match"]
    assert m.candidates == pm.candidates == list(range(M))
    assert torch.equal(m.W, pm.W[:, : m.W.shape[1]]) and torch.equal(m.wbar, pm.wbar)
    gd = harness.f64(m.dist)
    orc = _oracle_columns(c4)
    # full columns for 4 anchors, all positions
    for s in (0, 1, 100, 255):
        np.testing.assert_allclose(gd[s, :T], orc["cols"][s], rtol=1e-6)
    # 8 sampled positions for all 256 anchors -> per-position weights
    pos = [0, 1, 777, 1500, 2048, 3000, 3070, 3071]
    d_pos = np.stack([orc["cols"][s][pos] for s in range(M)], axis=1)
    np.testing.assert_allclose(gd[:, pos].T, d_pos, rtol=1e-6)
    W_o = O.softmax_neg(d_pos, axis=1)
    gW = harness.f64(m.W)[:, pos].T
    assert np.all(np.abs(gW - W_o) <= 1e-5 * W_o + 1e-7)
    wbar = O.softmax_neg(orc["dbar"])
    assert np.all(np.abs(harness.f64(m.wbar) - wbar) <= 1e-5 * wbar + 1e-7)
    H_o = O.entropy(wbar)
    assert abs(m.entropy - H_o) <= 1e-6 * H_o + 1e-9
    assert m.shareable and c4["reused"] == [True]


@pytest.mark.parametrize("kind", ["ph", "pf"])
def test_config4_sampled_rows(c4, kind):
    m = c4["m"]
    rng = np.random.default_rng(4 if kind == "ph" else 5)
    n = T if kind == "ph" else P
    toks = sorted(set([0, n - 1] + [int(x) for x in rng.integers(0, n, size=4)]))
    lh = [(0, 0), (19, 3), (int(rng.integers(0, 20)), int(rng.integers(0, 4)))]
    orc = _oracle_columns(c4)
    if kind == "ph":
        d = np.stack([orc["cols"][s][toks] for s in range(M)], axis=1)
        wts = O.softmax_neg(d, axis=1)                    # Eq. 6 per-position weights
        base, bstart, tstart = c4["base"], 0, 200
    else:
        wts = np.tile(O.softmax_neg(orc["dbar"])[None, :], (len(toks), 1))   # Eq. 7: w̄ for every row
        base, bstart, tstart = c4["pfb"], 200, 200 + T
    bk = harness.f64(base[0][:, :, toks])
    bv = harness.f64(base[1][:, :, toks])
    dk = [harness.f64(_offset(s, kind, 0)[:, :, toks]) for s in range(M)]
    dv = [harness.f64(_offset(s, kind, 1)[:, :, toks]) for s in range(M)]
    ora = O.realign_segment(wts, bk, bv, dk, dv, bstart, tstart, c4["inv"])
    absk = O.blend_placeholder(wts, [np.abs(x) for x in dk])
    absv = O.blend_placeholder(wts, [np.abs(x) for x in dv])
    rows = [tstart + t for t in toks]
    gk = harness.f64(c4["dst"][0][:, :, rows])
    gv = harness.f64(c4["dst"][1][:, :, rows])
    for (l, h) in lh:
        harness.check_kv(gk[l, h], ora["k"][l, h], bk[l, h], absk[l, h], f"config4 {kind} K l{l} h{h}", n_terms=M)
        harness.check_kv(gv[l, h], ora["v"][l, h], bv[l, h], absv[l, h], f"config4 {kind} V l{l} h{h}", n_terms=M)


def test_config4_p0_copied(c4):
    assert torch.equal(c4["dst"][0][:, :, :200], c4["p0"][0])
    assert torch.equal(c4["dst"][1][:, :, :200], c4["p0"][1])
