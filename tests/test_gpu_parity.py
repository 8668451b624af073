"""CUDA path vs CPU oracle, element by element, through the C ABI (-m gpu).

Sizes are small enough for the oracle to finish in seconds yet span several
16 KiB tiles and a ragged tail; edge cases cover the degenerate inputs of the
method.  Full-size (BASELINE configs[1]) sampled parity lives in
test_gpu_fullsize.py.
"""
import numpy as np
import pytest
import torch

import synth
from oracle import kvcomm_oracle as O
from tests import harness

pytestmark = pytest.mark.gpu

K = None


def setup_module(module):
    global K
    assert torch.cuda.is_available(), "gpu tests need CUDA"
    from paper_2510_12872_b200 import kvcomm as _K
    module.K = _K


@pytest.mark.parametrize("seed", [0, 1, 2, 3, 4])
@pytest.mark.parametrize("gamma", [0.3, 0.9])
@pytest.mark.parametrize("scalar", ["frobenius", "mean_l2"])
def test_tiny_config_full_parity(seed, gamma, scalar):
    p = synth.tiny_problem(seed)
    gpu = harness.run_gpu(p, gamma=gamma, scalar=scalar)
    ora = harness.run_oracle(p, gamma=gamma, scalar=scalar)
    harness.compare(gpu, ora, p)


@pytest.mark.parametrize("d,De,L_phi,P", [(128, 256, 150, 37), (64, 64, 300, 5), (256, 128, 70, 64),
                                          (16, 32, 600, 3), (128, 4096, 64, 32)])
def test_medium_multi_tile_ragged(d, De, L_phi, P):
    g = np.random.default_rng(d + L_phi)
    lens = [L_phi + int(x) for x in g.integers(0, 65, size=6)]
    p = synth.make_problem(11, L=3, H=2, d=d, D_e=De, L_phi=L_phi, anchor_lens=lens, prefix_lens=[P],
                           target_start=77, pf_base_start=200, pf_target_start=[77 + L_phi],
                           inv_freq=synth.llama3_inv_freq(d))
    gpu = harness.run_gpu(p, gamma=1.0)
    ora = harness.run_oracle(p, gamma=1.0)
    harness.compare(gpu, ora, p)


def test_negative_delta_and_large_positions():
    p = synth.make_problem(5, L=2, H=2, d=128, D_e=64, L_phi=65, anchor_lens=[65, 80, 90], prefix_lens=[32],
                           target_start=8100, pf_base_start=9000, pf_target_start=[8165],
                           inv_freq=synth.llama3_inv_freq(128))
    gpu = harness.run_gpu(p, gamma=1.0)
    ora = harness.run_oracle(p, gamma=1.0)
    harness.compare(gpu, ora, p)


@pytest.mark.parametrize("top_k", [1, 3, 8])
def test_topk_indices_outside_tie_band(top_k):
    # query = anchor 0 with swaps: exact zero distances and ties between identical rows
    p = synth.make_problem(7, L=2, H=2, d=64, D_e=64, L_phi=100, anchor_lens=[100] * 10, prefix_lens=[16],
                           target_start=12, pf_base_start=12, inv_freq=synth.llama3_inv_freq(64), n_vocab=32)
    gpu = harness.run_gpu(p, gamma=1.0, top_k=top_k)
    ora = harness.run_oracle(p, gamma=1.0, top_k=top_k)
    stats = harness.compare(gpu, ora, p)
    # the small vocabulary makes many rows identical across anchors -> exact ties,
    # which the (distance, slot) order resolves identically on both sides
    assert "idx_tie_positions" in stats


def test_exact_single_anchor_returns_its_offset():
    p = synth.make_problem(3, L=2, H=2, d=128, D_e=64, L_phi=70, anchor_lens=[70], prefix_lens=[8],
                           target_start=30, pf_base_start=30, p_swap=0.0)
    gpu = harness.run_gpu(p, gamma=0.3)
    m = gpu["match"]
    assert m.shareable and m.candidates == [0] and m.entropy == 0.0
    assert torch.all(m.W[0, :70] == 1.0)
    # blended offset equals the stored offset exactly (weight exactly 1)
    assert torch.equal(gpu["dbg_k"], p.dk_ph[0][0].float())
    assert torch.equal(gpu["dbg_v"], p.dv_ph[0][0].float())
    ora = harness.run_oracle(p, gamma=0.3)
    harness.compare(gpu, ora, p)


def test_unchanged_prefix_reproduces_identical_cache():
    dev = torch.device("cuda", 0)
    L_, H, d, De, T = 2, 2, 128, 64, 100
    g = synth.make_gen(9)
    pool = K.AnchorPool(num_layers=L_, num_kv_heads=H, head_dim=d, emb_dim=De, capacity=3, max_anchor_len=T,
                        prefix_len=[0], inv_freq=synth.llama3_inv_freq(d))
    z = torch.zeros(L_, H, T, d, dtype=torch.bfloat16, device=dev)
    emb = [synth.randn_bf16((T, De), g).to(dev) for _ in range(3)]
    for e in emb:
        pool.insert(e, [K.OffsetGiven(0, z, z, z[:, :, :0], z[:, :, :0])])
    m = pool.match(emb[1], consumer=0, gamma=1.0)
    base_k = synth.randn_bf16((L_, H, T, d), g).to(dev)
    base_v = synth.randn_bf16((L_, H, T, d), g).to(dev)
    dk = torch.empty_like(base_k)
    dv = torch.empty_like(base_v)
    K.realign_segment(K.Segment(pool, 0, K.PLACEHOLDER, m.W, m.candidates, base_k, base_v, 0, 0, dk, dv))
    torch.cuda.synchronize()
    assert torch.equal(dk, base_k) and torch.equal(dv, base_v)


@pytest.mark.parametrize("layout", ["half", "interleaved"])
def test_measure_insert_matches_oracle(layout):
    dev = torch.device("cuda", 0)
    L_, H, d, De, T, P = 2, 3, 128, 64, 90, 20
    inv = synth.llama3_inv_freq(d)
    g = synth.make_gen(21)
    t = lambda n: synth.randn_bf16((L_, H, n, d), g)
    kr, vr, kb, vb = t(T), t(T), t(T), t(T)
    pkr, pvr, pkb, pvb = t(P), t(P), t(P), t(P)
    pool = K.AnchorPool(num_layers=L_, num_kv_heads=H, head_dim=d, emb_dim=De, capacity=2, max_anchor_len=T + 5,
                        prefix_len=[P], inv_freq=inv, rope_layout=layout)
    off = K.OffsetMeasure(0, ph_real=(kr.to(dev), vr.to(dev), 731), ph_base=(kb.to(dev), vb.to(dev), 0),
                          pf_real=(pkr.to(dev), pvr.to(dev), 731 + T), pf_base=(pkb.to(dev), pvb.to(dev), 40))
    slot, ev = pool.insert(synth.randn_bf16((T, De), g).to(dev), [off])
    torch.cuda.synchronize()
    for which, (a, b, c_, d_, sr, sb, n) in {"ph": (kr, vr, kb, vb, 731, 0, T),
                                             "pf": (pkr, pvr, pkb, pvb, 731 + T, 40, P)}.items():
        gk, gv = pool.offset_view(slot, 0, which, rows=n)
        odk, odv = O.measure_offset(harness.f64(a), harness.f64(b), sr, harness.f64(c_), harness.f64(d_), sb, inv,
                                    layout)
        harness.check_kv(harness.f64(gk), O.bf16_round(odk), np.zeros_like(odk),
                         np.abs(harness.f64(a)) + np.abs(harness.f64(c_)), f"measured ΔK {which}", layout)
        # ΔV: a difference of two bf16 values, rounded once -> bit-exact
        assert np.array_equal(harness.f64(gv), O.bf16_round(odv)), which


def test_error_contracts():
    dev = torch.device("cuda", 0)
    p = synth.tiny_problem(1)
    pool = K.AnchorPool(num_layers=p.L, num_kv_heads=p.H, head_dim=p.d, emb_dim=p.D_e, capacity=4,
                        max_anchor_len=48, prefix_len=[4, 4], inv_freq=p.inv_freq)
    q = p.emb_query.to(dev)
    assert pool.match(q, gamma=0.3).reason == "EMPTY_POOL"
    # anchor 0 has offsets for consumer 0 only
    s0, _ = pool.insert(p.emb_anchor[0].to(dev), [K.OffsetGiven(0, p.dk_ph[0][0].to(dev), p.dv_ph[0][0].to(dev),
                                                                p.dk_pf[0][0].to(dev), p.dv_pf[0][0].to(dev))])
    assert pool.match(q, consumer=1, gamma=0.3).reason == "NO_CANDIDATES"
    assert pool.match(q, consumer=K.ALL_CONSUMERS, gamma=0.3).reason == "NO_CANDIDATES"
    m = pool.match(q, consumer=0, gamma=0.3)
    assert m.candidates == [s0] and m.shareable
    long_q = torch.cat([q, q], 0)
    assert pool.match(long_q, consumer=0, gamma=0.3).reason == "TOO_LONG"
    with pytest.raises(K.KVCommError, match="INVALID_ARGUMENT"):
        pool.match(q, consumer=0, gamma=1.5)
    dst = torch.zeros(p.L, p.H, 64, p.d, dtype=torch.bfloat16, device=dev)
    bk, bv = p.base_k.to(dev), p.base_v.to(dev)
    with pytest.raises(K.KVCommError, match="MISSING_OFFSET"):
        K.realign_segment(K.Segment(pool, 1, K.PLACEHOLDER, m.W, [s0], bk, bv, 0, 8, dst, dst.clone()))
    with pytest.raises(K.KVCommError, match="NO_CANDIDATES"):
        K.realign_segment(K.Segment(pool, 0, K.PLACEHOLDER, m.W, [], bk, bv, 0, 8, dst, dst.clone()))
    with pytest.raises(K.KVCommError, match="SHAPE_MISMATCH"):   # prefix length must equal prefix_len
        K.realign_segment(K.Segment(pool, 0, K.PREFIX, m.wbar, [s0], bk, bv, 8, 40, dst, dst.clone()))
    with pytest.raises(K.KVCommError, match="SHAPE_MISMATCH"):   # rows past the destination
        K.realign_segment(K.Segment(pool, 0, K.PLACEHOLDER, m.W, [s0], bk, bv, 0, 40, dst, dst.clone()))
    with pytest.raises(K.KVCommError, match="NOT_FOUND"):
        pool.evict(3)
    # a zero-length segment is a no-op
    before = dst.clone()
    K.realign_segment(K.Segment(pool, 0, K.PLACEHOLDER, m.W, [s0], bk, bv, 0, 8, dst, dst.clone(), L_seg=0))
    torch.cuda.synchronize()
    assert torch.equal(dst, before)


def test_lfu_eviction_matches_oracle_model():
    dev = torch.device("cuda", 0)
    rng = np.random.default_rng(0)
    pool = K.AnchorPool(num_layers=1, num_kv_heads=1, head_dim=16, emb_dim=8, capacity=5, max_anchor_len=8,
                        prefix_len=[1], inv_freq=synth.plain_inv_freq(16))
    model = O.PoolModel(5)
    emb = torch.zeros(4, 8, dtype=torch.bfloat16, device=dev)
    for step in range(60):
        s_gpu, ev_gpu = pool.insert(emb, [])
        s_ora, ev_ora = model.insert(4)
        assert (s_gpu, ev_gpu) == (s_ora, ev_ora), step
        acc = [int(x) for x in rng.choice(sorted(model.slot_len), size=int(rng.integers(0, 4)))]
        pool.record_access(acc)
        model.record_access(acc)
        if step % 17 == 16:
            victim = sorted(model.slot_len)[0]
            pool.evict(victim)
            model.evict(victim)
    for s in range(5):
        info = pool.slot_info(s)
        assert info["occupied"] == (s in model.slot_len)
        if info["occupied"]:
            assert info["access_count"] == model.access[s]


def test_determinism_and_batch_equals_single_and_layer_sharding():
    """T2: realigning layer shards separately gives the unsharded result bitwise;
    one batched launch equals per-segment launches; repeated runs are identical."""
    dev = torch.device("cuda", 0)
    p = synth.make_problem(13, L=4, H=2, d=128, D_e=128, L_phi=130, anchor_lens=[130, 140, 150, 190],
                           prefix_lens=[32], target_start=50, pf_base_start=50, inv_freq=synth.llama3_inv_freq(128))
    full1 = harness.run_gpu(p, gamma=1.0)
    full2 = harness.run_gpu(p, gamma=1.0)
    assert torch.equal(full1["dst_k"], full2["dst_k"]) and torch.equal(full1["dst_v"], full2["dst_v"])
    assert full1["match"].entropy == full2["match"].entropy
    # layer shards [0,2) and [2,4) as separate pools
    for lb, le in [(0, 2), (2, 4)]:
        pool = K.AnchorPool(num_layers=4, num_kv_heads=2, head_dim=128, emb_dim=128, capacity=4,
                            max_anchor_len=190, prefix_len=[32], inv_freq=p.inv_freq, layer_range=(lb, le))
        for j in range(4):
            pool.insert(p.emb_anchor[j].to(dev), [K.OffsetGiven(0, p.dk_ph[0][j][lb:le].to(dev),
                                                                p.dv_ph[0][j][lb:le].to(dev),
                                                                p.dk_pf[0][j][lb:le].to(dev),
                                                                p.dv_pf[0][j][lb:le].to(dev))])
        m = pool.match(p.emb_query.to(dev), consumer=0, gamma=1.0)
        assert torch.equal(m.W.cpu(), full1["match"].W.cpu())
        N = full1["N"]
        dk = torch.zeros(le - lb, 2, N, 128, dtype=torch.bfloat16, device=dev)
        dv = torch.zeros_like(dk)
        segs = [K.Segment(pool, 0, K.PLACEHOLDER, m.W, m.candidates, p.base_k[lb:le].to(dev),
                          p.base_v[lb:le].to(dev), 0, 50, dk, dv),
                K.Segment(pool, 0, K.PREFIX, m.wbar, m.candidates, p.pf_base_k[0][lb:le].to(dev),
                          p.pf_base_v[0][lb:le].to(dev), 50, 180, dk, dv)]
        for s in segs:   # one launch per segment
            K.realign_segment(s)
        torch.cuda.synchronize()
        assert torch.equal(dk[:, :, 50:].cpu(), full1["dst_k"][lb:le, :, 50:])
        assert torch.equal(dv[:, :, 50:].cpu(), full1["dst_v"][lb:le, :, 50:])
    # layer x KV-head shards (config 4's 70B partitioning): [0,2)x[0,1), [2,4)x[1,2), ...
    for (lb, le), (hb, he) in [((0, 2), (0, 1)), ((0, 2), (1, 2)), ((2, 4), (0, 1)), ((2, 4), (1, 2))]:
        pool = K.AnchorPool(num_layers=4, num_kv_heads=2, head_dim=128, emb_dim=128, capacity=4,
                            max_anchor_len=190, prefix_len=[32], inv_freq=p.inv_freq, layer_range=(lb, le),
                            head_range=(hb, he))
        sl = lambda t: t[lb:le, hb:he].contiguous().to(dev)
        for j in range(4):
            pool.insert(p.emb_anchor[j].to(dev), [K.OffsetGiven(0, sl(p.dk_ph[0][j]), sl(p.dv_ph[0][j]),
                                                                sl(p.dk_pf[0][j]), sl(p.dv_pf[0][j]))])
        m = pool.match(p.emb_query.to(dev), consumer=0, gamma=1.0)
        N = full1["N"]
        dk = torch.zeros(le - lb, he - hb, N, 128, dtype=torch.bfloat16, device=dev)
        dv = torch.zeros_like(dk)
        K.realign_segments([K.Segment(pool, 0, K.PLACEHOLDER, m.W, m.candidates, sl(p.base_k), sl(p.base_v), 0, 50,
                                      dk, dv),
                            K.Segment(pool, 0, K.PREFIX, m.wbar, m.candidates, sl(p.pf_base_k[0]), sl(p.pf_base_v[0]),
                                      50, 180, dk, dv)])
        torch.cuda.synchronize()
        assert torch.equal(dk[:, :, 50:].cpu(), full1["dst_k"][lb:le, hb:he, 50:])
        assert torch.equal(dv[:, :, 50:].cpu(), full1["dst_v"][lb:le, hb:he, 50:])


def test_copy_segments_are_bit_exact_for_any_bit_pattern():
    dev = torch.device("cuda", 0)
    g = torch.Generator().manual_seed(3)
    pool = K.AnchorPool(num_layers=3, num_kv_heads=2, head_dim=128, emb_dim=16, capacity=1, max_anchor_len=8,
                        prefix_len=[0], inv_freq=synth.llama3_inv_freq(128))
    bits = torch.randint(-32768, 32767, (2, 3, 2, 150, 128), generator=g, dtype=torch.int16)
    bits[0, 0, 0, 0, :4] = torch.tensor([-32768, 0x7fc0, 0x7f80, -0x0080], dtype=torch.int16)  # -0, NaN, inf, -inf
    src_k = bits[0].view(torch.bfloat16).to(dev)
    src_v = bits[1].view(torch.bfloat16).to(dev)
    dk = torch.zeros(3, 2, 170, 128, dtype=torch.bfloat16, device=dev)
    dv = torch.zeros_like(dk)
    K.realign_segment(K.Segment(pool, 0, K.COPY, None, [], src_k, src_v, 0, 20, dk, dv))
    torch.cuda.synchronize()
    assert torch.equal(dk[:, :, 20:].view(torch.int16).cpu(), bits[0])
    assert torch.equal(dv[:, :, 20:].view(torch.int16).cpu(), bits[1])
    assert torch.all(dk[:, :, :20].view(torch.int16) == 0)
    # concat uses the same path
    ek = torch.zeros(3, 2, 150, 128, dtype=torch.bfloat16, device=dev)
    ev = torch.zeros_like(ek)
    K.concat_prefill_cache([(0, 150, src_k, src_v)], 150, ek, ev)
    torch.cuda.synchronize()
    assert torch.equal(ek.view(torch.int16).cpu(), bits[0]) and torch.equal(ev.view(torch.int16).cpu(), bits[1])


def test_match_many_equals_individual_matches():
    dev = torch.device("cuda", 0)
    probs = [synth.make_problem(40 + i, L=2, H=2, d=64, D_e=128, L_phi=L, anchor_lens=[L, L + 9, L + 30],
                                prefix_lens=[8], target_start=4, pf_base_start=4)
             for i, L in enumerate([33, 70, 129])]
    pools = []
    for p in probs:
        pool = K.AnchorPool(num_layers=2, num_kv_heads=2, head_dim=64, emb_dim=128, capacity=3,
                            max_anchor_len=max(p.anchor_lens), prefix_len=[8], inv_freq=p.inv_freq)
        for j in range(3):
            pool.insert(p.emb_anchor[j].to(dev), [K.OffsetGiven(0, p.dk_ph[0][j].to(dev), p.dv_ph[0][j].to(dev),
                                                                p.dk_pf[0][j].to(dev), p.dv_pf[0][j].to(dev))])
        pools.append(pool)
    qs = [p.emb_query.to(dev) for p in probs]
    many = K.match_many(list(zip(pools, qs)), gamma=0.5, want_dist=True)
    for pool, q, m in zip(pools, qs, many):
        one = pool.match(q, gamma=0.5, want_dist=True)
        assert m.candidates == one.candidates and m.verdict == one.verdict and m.entropy == one.entropy
        assert torch.equal(m.W, one.W) and torch.equal(m.wbar, one.wbar) and torch.equal(m.dist, one.dist)
    with pytest.raises(K.KVCommError, match="twice"):
        K.match_many([(pools[0], qs[0]), (pools[0], qs[0])])


@pytest.mark.parametrize("seed", [0, 1, 2])
@pytest.mark.parametrize("top_k", [0, 2])
def test_cosine_similarity_variant(seed, top_k):
    """Table A.4's cosine-similarity weighting on the device vs the oracle."""
    p = synth.make_problem(60 + seed, L=2, H=2, d=64, D_e=256, L_phi=90, anchor_lens=[90, 100, 95, 130, 90],
                           prefix_lens=[12], target_start=20, pf_base_start=20, inv_freq=synth.llama3_inv_freq(64))
    gpu = harness.run_gpu(p, gamma=1.0, top_k=top_k, similarity="cosine")
    ora = harness.run_oracle(p, gamma=1.0, top_k=top_k, similarity="cosine")
    harness.compare(gpu, ora, p)


def _fp8_codes(q: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(q.astype(np.float32)).to(torch.float8_e4m3fn).view(torch.uint8)


@pytest.mark.parametrize("d,L_phi,P", [(128, 150, 37), (64, 200, 5), (256, 70, 32), (80, 100, 7), (96, 90, 11),
                                        (192, 50, 40)])
def test_fp8_offsets_codes_and_realign(d, L_phi, P):
    """f3: e4m3 offset storage.  GIVEN offsets are quantised on the device to the same
    codes and scales as the oracle's quantiser (bit-exact), and the realignment from
    the fp8 pool matches the oracle run on the dequantised offsets."""
    p = synth.make_problem(31, L=2, H=2, d=d, D_e=64, L_phi=L_phi, anchor_lens=[L_phi, L_phi + 9, L_phi + 40],
                           prefix_lens=[P], target_start=25, pf_base_start=25, inv_freq=synth.llama3_inv_freq(d))
    gpu = harness.run_gpu(p, gamma=1.0, offset_format="fp8")
    pool = gpu["pool"]
    for j, s in enumerate(gpu["slots"]):
        for which, src in (("ph", p.dk_ph[0][j]), ("pf", p.dk_pf[0][j])):
            rows = src.shape[2]
            gk, _, sk, _ = pool.read_offsets(s, 0, which, rows)
            q, sc = O.quantize_rows_fp8(harness.f64(src))
            assert torch.equal(gk.cpu(), _fp8_codes(q)), (j, which)
            assert torch.equal(sk.cpu(), torch.from_numpy(sc)), (j, which)
    ora = harness.run_oracle(p, gamma=1.0, fp8=True)
    harness.compare(gpu, ora, p)


def _e4m3_hard_rows(d):
    """Rows on which x * fl(1/scale) and the IEEE quotient x / scale round to DIFFERENT
    e4m3 codes: for row maxima whose fp32 reciprocal scale is inexact enough, every
    positive bf16 x <= amax is tried and the ones that flip are kept (with their
    negatives), found with the oracle's own rounding.  Returns (rows, flips)."""
    allb = torch.arange(1, 0x7f80, dtype=torch.int32).to(torch.int16).view(torch.bfloat16).float().numpy()
    rows, flips = [], 0
    for amax in (2.15625, 1.296875, 2.84375, 1.2734375, 0.98046875, 3.328125, 0.021240234375):
        sc = np.float32(amax) / np.float32(448)
        xs = allb[allb <= amax].astype(np.float32)
        exact = O.e4m3_round((xs / sc).astype(np.float32).astype(np.float64))
        recip = O.e4m3_round((xs * (np.float32(1) / sc)).astype(np.float32).astype(np.float64))
        hard = xs[exact != recip]
        flips += len(hard)
        vals = [v for h in hard for v in (float(h), -float(h))]
        for i in range(0, max(len(vals), 1), d - 1):
            chunk = vals[i:i + d - 1]
            rows.append([amax] + chunk + [0.0] * (d - 1 - len(chunk)))
    return torch.tensor(rows, dtype=torch.float32).to(torch.bfloat16), flips


def test_fp8_quantiser_exact_on_rounding_ties():
    """The device quantiser gives the codes of an IEEE division exactly, also on the
    elements where a reciprocal multiply would round to a different e4m3 code."""
    d = 128
    rows, flips = _e4m3_hard_rows(d)
    assert flips >= 20          # a plain reciprocal multiply would get these codes wrong
    n = rows.shape[0]
    x = rows.view(1, 1, n, d).expand(2, 2, n, d).contiguous()
    dev = torch.device("cuda", 0)
    pool = K.AnchorPool(num_layers=2, num_kv_heads=2, head_dim=d, emb_dim=64, capacity=1, max_anchor_len=n,
                        prefix_len=[n], inv_freq=synth.llama3_inv_freq(d), offset_format="fp8")
    xd = x.to(dev)
    xn = torch.where(x == 0, x, -x)     # negatives; the zero padding stays +0
    slot, _ = pool.insert(torch.zeros(n, 64, dtype=torch.bfloat16, device=dev),
                          [K.OffsetGiven(0, xd, xn.to(dev), xd, xd)])
    q, sc = O.quantize_rows_fp8(harness.f64(x))
    qn, _ = O.quantize_rows_fp8(harness.f64(xn))
    for which in ("ph", "pf"):
        gk, gv, sk, sv = pool.read_offsets(slot, 0, which, n)
        assert torch.equal(gk.cpu(), _fp8_codes(q)), which
        assert torch.equal(sk.cpu(), torch.from_numpy(sc)), which
        if which == "ph":
            assert torch.equal(gv.cpu(), _fp8_codes(qn))
    pool.destroy()


def test_fp8_measure_insert_close_to_oracle():
    dev = torch.device("cuda", 0)
    L_, H, d, T, P = 2, 2, 128, 70, 8
    inv = synth.llama3_inv_freq(d)
    g = synth.make_gen(22)
    t = lambda n: synth.randn_bf16((L_, H, n, d), g)
    kr, vr, kb, vb, pkr, pvr, pkb, pvb = t(T), t(T), t(T), t(T), t(P), t(P), t(P), t(P)
    pool = K.AnchorPool(num_layers=L_, num_kv_heads=H, head_dim=d, emb_dim=64, capacity=1, max_anchor_len=T,
                        prefix_len=[P], inv_freq=inv, offset_format="fp8")
    off = K.OffsetMeasure(0, ph_real=(kr.to(dev), vr.to(dev), 300), ph_base=(kb.to(dev), vb.to(dev), 0),
                          pf_real=(pkr.to(dev), pvr.to(dev), 300 + T), pf_base=(pkb.to(dev), pvb.to(dev), 40))
    slot, _ = pool.insert(synth.randn_bf16((T, 64), g).to(dev), [off])
    torch.cuda.synchronize()
    f64 = harness.f64
    for which, (a, b, c_, d_, sr, sb, n) in {"ph": (kr, vr, kb, vb, 300, 0, T),
                                             "pf": (pkr, pvr, pkb, pvb, 300 + T, 40, P)}.items():
        ck, cv, sk, sv = pool.read_offsets(slot, 0, which, n)
        codes, scales = (ck, cv), (sk, sv)
        odk, odv = O.measure_offset(f64(a), f64(b), sr, f64(c_), f64(d_), sb, inv)
        for code, sc, ref in zip(codes, scales, (odk, odv)):
            got = code.cpu().view(torch.float8_e4m3fn).double().numpy() * f64(sc)[..., None]
            amax = np.max(np.abs(ref), axis=-1, keepdims=True)
            # one e4m3 step at the value's magnitude (fp32 vs fp64 measurement can flip a rounding)
            assert np.all(np.abs(got - ref) <= 2.0 ** -3 * np.abs(ref) + 2.0 ** -9 * amax / 448 + 1e-6), which


@pytest.mark.parametrize("fmt", ["bf16", "fp8"])
def test_host_resident_pool(fmt):
    """f4: offset slabs in pinned host memory (A.4.4 CPU offload) streamed
    by the same kernels; results identical to the device-resident pool."""
    p = synth.make_problem(8, L=2, H=2, d=128, D_e=64, L_phi=100, anchor_lens=[100, 120, 140], prefix_lens=[16],
                           target_start=30, pf_base_start=30, inv_freq=synth.llama3_inv_freq(128))
    dev = harness.run_gpu(p, gamma=1.0, offset_format=fmt)
    host = harness.run_gpu(p, gamma=1.0, offset_format=fmt, placement="host")
    assert torch.equal(dev["dst_k"], host["dst_k"]) and torch.equal(dev["dst_v"], host["dst_v"])
    ora = harness.run_oracle(p, gamma=1.0, fp8=(fmt == "fp8"))
    harness.compare(host, ora, p)


@pytest.mark.parametrize("fmt,d,n_anchor", [("bf16", 128, 40), ("fp8", 64, 20), ("fp8", 128, 3)])
def test_weight_block_fallback(fmt, d, n_anchor):
    """Units whose weight block [n_cand][rows] exceeds the kernel's unit buffer take the
    per-anchor weight-slice path; both paths agree with the oracle."""
    lens = [60 + 7 * (j % 5) for j in range(n_anchor)]
    p = synth.make_problem(40 + n_anchor, L=2, H=2, d=d, D_e=64, L_phi=60, anchor_lens=lens, prefix_lens=[11],
                           target_start=9, pf_base_start=9, inv_freq=synth.llama3_inv_freq(d))
    gpu = harness.run_gpu(p, gamma=1.0, offset_format=fmt)
    ora = harness.run_oracle(p, gamma=1.0, fp8=(fmt == "fp8"))
    harness.compare(gpu, ora, p)


def test_fp8_large_row_scale():
    """Offsets of very large magnitude (row scales amax/448 far above 1) quantise and
    realign like any other rows: no overflow in weight x row scale or the decode."""
    d = 128
    p = synth.make_problem(77, L=2, H=2, d=d, D_e=64, L_phi=90, anchor_lens=[90, 95, 130], prefix_lens=[20],
                           target_start=5, pf_base_start=5, inv_freq=synth.llama3_inv_freq(d))
    for lst in (p.dk_ph, p.dv_ph, p.dk_pf, p.dv_pf):
        lst[0][1] = (lst[0][1].float() * 4e6).to(torch.bfloat16)
    gpu = harness.run_gpu(p, gamma=1.0, offset_format="fp8")
    ora = harness.run_oracle(p, gamma=1.0, fp8=True)
    harness.compare(gpu, ora, p)


@pytest.mark.parametrize("n_anchor", [8, 9, 17])
def test_weight_chunk_boundaries(n_anchor):
    """d = 16: a 512-row tile takes 2 KiB of weights per anchor, so a 16 KiB weight chunk
    holds 8 anchors; n_cand = 8, 9, 17 hit the exact-fit, one-over and multi-chunk cases."""
    lens = [40 + 3 * (j % 4) for j in range(n_anchor)]
    p = synth.make_problem(60 + n_anchor, L=2, H=2, d=16, D_e=32, L_phi=40, anchor_lens=lens, prefix_lens=[6],
                           target_start=8, pf_base_start=4)
    gpu = harness.run_gpu(p, gamma=1.0)
    ora = harness.run_oracle(p, gamma=1.0)
    harness.compare(gpu, ora, p)


@pytest.mark.parametrize("fmt,top_k", [("bf16", 0), ("bf16", 32), ("fp8", 0)])
def test_maximum_capacity_1024_anchors(fmt, top_k):
    """KVCOMM_MAX_CAPACITY = 1024 candidates (config 5's largest pool) through match,
    weights (dense and the maximum top-k of 32) and realign (128 weight chunks at d=16;
    64 at d=64 fp8), against the oracle."""
    d = 16 if fmt == "bf16" else 64
    n = 1024
    lens = [24 + (j % 3) for j in range(n)]
    p = synth.make_problem(1024 + top_k, L=1, H=1, d=d, D_e=32, L_phi=24, anchor_lens=lens, prefix_lens=[4],
                           target_start=3, pf_base_start=2, inv_freq=synth.llama3_inv_freq(d), n_vocab=64)
    gpu = harness.run_gpu(p, gamma=1.0, top_k=top_k, offset_format=fmt)
    ora = harness.run_oracle(p, gamma=1.0, top_k=top_k, fp8=(fmt == "fp8"))
    harness.compare(gpu, ora, p)


@pytest.mark.parametrize("kind", ["placeholder", "prefix"])
def test_dyadic_inputs_are_bit_exact(kind):
    """with dyadic weights (1/2, 1/4, 1/4 permuted per position), dyadic
    offsets and bases and δ = 0, every product and partial sum is exact in fp32, so
    the single RNE rounding to bf16 must give the oracle's bf16 result bit for bit."""
    dev = torch.device("cuda", 0)
    L_, H, d, T, P = 2, 2, 64, 40, 8
    g = torch.Generator().manual_seed(11)
    dy = lambda shape, den, lim: (torch.randint(-lim, lim + 1, shape, generator=g).double() / den).to(torch.bfloat16)
    n = 3
    dk = [dy((L_, H, T, d), 16, 16) for _ in range(n)]
    dv = [dy((L_, H, T, d), 16, 16) for _ in range(n)]
    pk = [dy((L_, H, P, d), 16, 16) for _ in range(n)]
    pv = [dy((L_, H, P, d), 16, 16) for _ in range(n)]
    inv = synth.llama3_inv_freq(d)
    pool = K.AnchorPool(num_layers=L_, num_kv_heads=H, head_dim=d, emb_dim=64, capacity=n, max_anchor_len=T,
                        prefix_len=[P], inv_freq=inv)
    for j in range(n):
        pool.insert(torch.zeros(T, 64, dtype=torch.bfloat16, device=dev),
                    [K.OffsetGiven(0, dk[j].to(dev), dv[j].to(dev), pk[j].to(dev), pv[j].to(dev))])
    rows = T if kind == "placeholder" else P
    base_k, base_v = dy((L_, H, rows, d), 8, 32), dy((L_, H, rows, d), 8, 32)
    perms = [(0.5, 0.25, 0.25), (0.25, 0.5, 0.25), (0.25, 0.25, 0.5)]
    if kind == "placeholder":
        Wt = np.array([perms[i % 3] for i in range(T)])                      # [T, n]
        weights = torch.zeros(n, T, dtype=torch.float32)
        weights[:, :] = torch.from_numpy(Wt.T)
        ora = O.realign_segment(Wt, harness.f64(base_k), harness.f64(base_v), [harness.f64(x) for x in dk],
                                [harness.f64(x) for x in dv], 5, 5, inv, "placeholder")
        kkind = K.PLACEHOLDER
    else:
        wb = np.array(perms[1])
        weights = torch.from_numpy(wb).float()
        ora = O.realign_segment(wb, harness.f64(base_k), harness.f64(base_v), [harness.f64(x) for x in pk],
                                [harness.f64(x) for x in pv], 5, 5, inv, "prefix")
        kkind = K.PREFIX
    dst_k = torch.zeros(L_, H, rows + 5, d, dtype=torch.bfloat16, device=dev)
    dst_v = torch.zeros_like(dst_k)
    seg = K.Segment(pool, 0, kkind, weights.to(dev), [0, 1, 2], base_k.to(dev), base_v.to(dev), 5, 5, dst_k, dst_v)
    K.realign_segment(seg)
    torch.cuda.synchronize()
    gk = dst_k[:, :, 5:].cpu().view(torch.int16)
    gv = dst_v[:, :, 5:].cpu().view(torch.int16)
    ok = torch.from_numpy(ora["k"]).to(torch.bfloat16).view(torch.int16)
    ov = torch.from_numpy(ora["v"]).to(torch.bfloat16).view(torch.int16)
    assert torch.equal(gk, ok) and torch.equal(gv, ov)
    pool.destroy()


@pytest.mark.parametrize("fmt,d", [("bf16", 16), ("bf16", 128), ("bf16", 80), ("fp8", 128), ("fp8", 64)])
def test_interleaved_rope_layout(fmt, d):
    """rope_layout = INTERLEAVED (GPT-J pairs (2f, 2f+1)): realign with
    δ != 0 on placeholder and prefix against the oracle's interleaved rotation."""
    p = synth.make_problem(90 + d, L=2, H=2, d=d, D_e=64, L_phi=70, anchor_lens=[70, 80, 95], prefix_lens=[9],
                           target_start=37, pf_base_start=21, inv_freq=synth.llama3_inv_freq(d))
    gpu = harness.run_gpu(p, gamma=1.0, offset_format=fmt, rope_layout="interleaved")
    ora = harness.run_oracle(p, gamma=1.0, fp8=(fmt == "fp8"), rope_layout="interleaved")
    harness.compare(gpu, ora, p)


def test_fp8_measure_interleaved_close_to_oracle():
    dev = torch.device("cuda", 0)
    L_, H, d, T = 2, 2, 128, 40
    inv = synth.llama3_inv_freq(d)
    g = synth.make_gen(23)
    t = lambda n: synth.randn_bf16((L_, H, n, d), g)
    kr, vr, kb, vb = t(T), t(T), t(T), t(T)
    pool = K.AnchorPool(num_layers=L_, num_kv_heads=H, head_dim=d, emb_dim=64, capacity=1, max_anchor_len=T,
                        prefix_len=[0], inv_freq=inv, offset_format="fp8", rope_layout="interleaved")
    off = K.OffsetMeasure(0, ph_real=(kr.to(dev), vr.to(dev), 500), ph_base=(kb.to(dev), vb.to(dev), 0))
    slot, _ = pool.insert(synth.randn_bf16((T, 64), g).to(dev), [off])
    torch.cuda.synchronize()
    ck, cv, sk, sv = pool.read_offsets(slot, 0, "ph", T)
    odk, _ = O.measure_offset(harness.f64(kr), harness.f64(vr), 500, harness.f64(kb), harness.f64(vb), 0, inv,
                              O.INTERLEAVED)
    got = ck.cpu().view(torch.float8_e4m3fn).double().numpy() * harness.f64(sk)[..., None]
    amax = np.max(np.abs(odk), axis=-1, keepdims=True)
    assert np.all(np.abs(got - odk) <= 2.0 ** -3 * np.abs(odk) + 2.0 ** -9 * amax / 448 + 1e-6)


@pytest.mark.gpu
@pytest.mark.parametrize("variant", ["1", "2"])
@pytest.mark.parametrize("De,L_phi", [(64, 33), (8192, 9)])
def test_match_tma_variant_matches_oracle(De, L_phi, variant):
    """The TMA-fed distance kernels (KVCOMM_MATCH_TMA=1: 16 KiB tiles shared by all warps,
    a measured-slower measurement variant; =2: one ring stage per anchor row)
    must match the oracle: a small D_e (many anchor tiles per stage) and D_e = 8192 (each
    anchor tile split in two 16 KiB chunks), an odd L_φ (a one-position last block)."""
    import subprocess
    import sys
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys; sys.path.insert(0, %r); import synth; from tests import harness; "
            "p = synth.make_problem(11, L=1, H=1, d=16, D_e=%d, L_phi=%d, anchor_lens=[%d, %d, %d], prefix_lens=[2], "
            "target_start=3, pf_base_start=3); g = harness.run_gpu(p, gamma=0.9); o = harness.run_oracle(p, gamma=0.9); "
            "harness.compare(g, o, p); print('ok')" % (root, De, L_phi, L_phi, L_phi + 4, L_phi + 1))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=dict(os.environ, KVCOMM_MATCH_TMA=variant),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-3000:]


@pytest.mark.gpu
@pytest.mark.parametrize("top_k", [0, 3])
def test_match_ring_kernel_bitwise_equals_register_kernel(top_k, tmp_path):
    """The row-ring distance kernel reduces every anchor row in the register kernel's order
    (same lanes, groups of 8, fp64 accumulation, butterfly), so W, w̄, the distances and the
    entropy are bit-identical: D_e 4096 (config 2's width), 20 anchors of mixed lengths
    (truncation), an odd L_φ, dense and top-k weights."""
    import subprocess
    import sys
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys, torch; sys.path.insert(0, %r); import synth; from tests import harness; "
            "p = synth.make_problem(21, L=1, H=1, d=16, D_e=4096, L_phi=37, anchor_lens=[37 + (j %% 5) for j in range(20)], "
            "prefix_lens=[2], target_start=3, pf_base_start=3); g = harness.run_gpu(p, gamma=0.9, top_k=%d); m = g['match']; "
            "torch.save({'W': m.W.cpu(), 'wbar': m.wbar.cpu(), 'dist': m.dist.cpu(), 'H': m.entropy}, sys.argv[1]); print('ok')"
            % (root, top_k))
    outs = {}
    for v in ("0", "2"):
        f = str(tmp_path / f"m{v}.pt")
        r = subprocess.run([sys.executable, "-c", code, f], cwd=root, env=dict(os.environ, KVCOMM_MATCH_TMA=v),
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-3000:]
        outs[v] = torch.load(f)
    a, b = outs["0"], outs["2"]
    assert torch.equal(a["W"], b["W"]) and torch.equal(a["wbar"], b["wbar"]) and torch.equal(a["dist"], b["dist"])
    assert a["H"] == b["H"]
