"""Parity harness: run one synthetic Problem through the CUDA path (C ABI via the
binding) and through the CPU oracle, and compare them with the north-star tolerances.

Used by tests/test_gpu_parity.py and __graft_entry__.smoke().  The product package
never imports this file.

Tolerances (BASELINE.json north_star):
  * anchor-selection indices bit-exact outside the 1e-6 relative distance-tie band;
    verdict equal unless |H - γ log|𝒜|| <= 1e-6 · γ log|𝒜| (oracle side);
  * fp32 blended offsets: |g - o| <= 1e-4 · (|o| + Σ_j w_j |Δ_j|);
  * bf16 K/V: |g - o| <= max(1e-2 |o|, 2^-7 · 2^floor(log2 |o|)) + δ, where
    δ = (n + 8) · 2^-24 · M is the forward-error bound of the kernel's fp32 pipeline
    (n FMA roundings of Σ_j w_j Δ_j, the fp32 weight (and fp8 scale
    product), the base add, the rotation's two products, its sum and its fp32 cos/sin),
    M = |base| + Σ_j w_j |Δ_j| summed over the element and its RoPE partner, n = the
    number of blended anchors.  The north-star bound alone is reported next to it:
    check_kv counts the elements that pass only because of δ (outputs that cancel to
    ~0, where one bf16 ulp of o is below the fp32 pipeline's rounding error);
  * distances: relative 1e-6; weights W, w̄: |g - o| <= 1e-5 |o| + 1e-7.
"""
from __future__ import annotations

import math
from typing import Dict, Optional

import numpy as np
import torch

from oracle import kvcomm_oracle as O
import synth

TIE_REL = 1e-6


def f64(t: torch.Tensor) -> np.ndarray:
    return t.detach().to("cpu", torch.float64).numpy()


# --------------------------------------------------------------------------- GPU

def run_gpu(p: synth.Problem, gamma: float = 0.3, top_k: int = 0, capacity: Optional[int] = None,
            measure: bool = False, consumer: int = 0, device: int = 0, scalar: str = "frobenius",
            similarity: str = "l2", offset_format: str = "bf16", placement: str = "device",
            rope_layout: str = "half") -> Dict:
    """Insert p's anchors, match p's query, realign its placeholder + prefix for
    `consumer`, copy a synthetic p_(m,0) and check the ledger.  Returns CPU tensors."""
    from paper_2510_12872_b200 import kvcomm as K
    dev = torch.device("cuda", device)
    cap = capacity or len(p.anchor_lens)
    pool = K.AnchorPool(num_layers=p.L, num_kv_heads=p.H, head_dim=p.d, emb_dim=p.D_e, capacity=cap,
                        max_anchor_len=max(p.anchor_lens), prefix_len=p.prefix_lens, inv_freq=p.inv_freq,
                        device=device, scalar_distance=scalar, similarity=similarity,
                        offset_format=offset_format, placement=placement, rope_layout=rope_layout)
    slots = []
    for j, Lj in enumerate(p.anchor_lens):
        offs = []
        for c in range(len(p.prefix_lens)):
            offs.append(K.OffsetGiven(c, p.dk_ph[c][j].to(dev), p.dv_ph[c][j].to(dev),
                                      p.dk_pf[c][j].to(dev), p.dv_pf[c][j].to(dev)))
        s, ev = pool.insert(p.emb_anchor[j].to(dev), offs)
        slots.append(s)
    m = pool.match(p.emb_query.to(dev), consumer=consumer, gamma=gamma, top_k=top_k, want_dist=True)
    out = {"pool": pool, "slots": slots, "match": m, "rope_layout": rope_layout, "consumer": consumer}
    if not m.candidates:
        return out
    c = consumer
    P = p.prefix_lens[c]
    p0 = p.target_start
    N = p0 + p.L_phi + P
    dst_k = torch.full((p.L, p.H, N, p.d), float("nan"), dtype=torch.bfloat16, device=dev)
    dst_v = torch.full_like(dst_k, float("nan"))
    dbg = [torch.zeros(p.L, p.H, p.L_phi, p.d, dtype=torch.float32, device=dev) for _ in range(2)]
    dbgp = [torch.zeros(p.L, p.H, P, p.d, dtype=torch.float32, device=dev) for _ in range(2)]
    segs = [K.Segment(pool, c, K.PLACEHOLDER, m.W, m.candidates, p.base_k.to(dev), p.base_v.to(dev), 0,
                      p.target_start, dst_k, dst_v, debug_k=dbg[0], debug_v=dbg[1])]
    if P > 0:
        segs.append(K.Segment(pool, c, K.PREFIX, m.wbar, m.candidates, p.pf_base_k[c].to(dev),
                              p.pf_base_v[c].to(dev), p.pf_base_start, p.pf_target_start[c], dst_k, dst_v,
                              debug_k=dbgp[0], debug_v=dbgp[1]))
    K.realign_segments(segs)
    # p_(m,0): a synthetic system-prompt cache copied verbatim (reading A20)
    g = synth.make_gen(p.seed + 999)
    p0k = synth.randn_bf16((p.L, p.H, p0, p.d), g).to(dev)
    p0v = synth.randn_bf16((p.L, p.H, p0, p.d), g).to(dev)
    K.concat_prefill_cache([(0, p0, p0k, p0v), (p0, p.L_phi, None, None), (p0 + p.L_phi, P, None, None)], N,
                           dst_k, dst_v)   # copies p_(m,0) through the realign kernel's TMA ring
    torch.cuda.synchronize()
    out.update(dst_k=dst_k.cpu(), dst_v=dst_v.cpu(), dbg_k=dbg[0].cpu(), dbg_v=dbg[1].cpu(),
               dbgp_k=dbgp[0].cpu(), dbgp_v=dbgp[1].cpu(), p0k=p0k.cpu(), p0v=p0v.cpu(), N=N)
    return out


# ------------------------------------------------------------------------ oracle

def run_oracle(p: synth.Problem, gamma: float = 0.3, top_k: int = 0, consumer: int = 0,
               slots=None, scalar: str = "frobenius", similarity: str = "l2", fp8: bool = False,
               rope_layout: str = "half") -> Dict:
    """fp8=True: the offsets the blend sees are the e4m3-quantised ones (oracle's own
    quantiser, O.quantize_rows_fp8), as stored by an fp8 pool."""
    store = (lambda x: O.dequantize_rows_fp8(*O.quantize_rows_fp8(x))) if fp8 else (lambda x: x)
    slots = slots or list(range(len(p.anchor_lens)))
    lens = {s: L for s, L in zip(slots, p.anchor_lens)}
    embs = {s: f64(e) for s, e in zip(slots, p.emb_anchor)}
    present = {s: True for s in slots}
    r = O.predict(f64(p.emb_query), lens, embs, present, gamma, top_k, scalar, similarity)
    out = {"match": r}
    if not r.candidates:
        return out
    c = consumer
    j_of = {s: j for j, s in enumerate(slots)}
    js = [j_of[s] for s in r.candidates]
    dk = [store(f64(p.dk_ph[c][j])) for j in js]
    dv = [store(f64(p.dv_ph[c][j])) for j in js]
    ph = O.realign_segment(r.W, f64(p.base_k), f64(p.base_v), dk, dv, 0, p.target_start, p.inv_freq,
                           layout=rope_layout)
    ph["absk"] = O.blend_placeholder(r.W, [np.abs(x) for x in dk])
    ph["absv"] = O.blend_placeholder(r.W, [np.abs(x) for x in dv])
    out["ph"] = ph
    if p.prefix_lens[c] > 0:
        pk = [store(f64(p.dk_pf[c][j])) for j in js]
        pv = [store(f64(p.dv_pf[c][j])) for j in js]
        pf = O.realign_segment(r.wbar, f64(p.pf_base_k[c]), f64(p.pf_base_v[c]), pk, pv, p.pf_base_start,
                               p.pf_target_start[c], p.inv_freq, kind="prefix", layout=rope_layout)
        pf["absk"] = O.blend_prefix(r.wbar, [np.abs(x) for x in pk])
        pf["absv"] = O.blend_prefix(r.wbar, [np.abs(x) for x in pv])
        out["pf"] = pf
    return out


# ------------------------------------------------------------------------ compare

def _partner(x: np.ndarray, layout: str = "half") -> np.ndarray:
    """The RoPE partner of every element: f <-> f + d/2 (half) or 2f <-> 2f + 1."""
    d = x.shape[-1]
    if layout == "interleaved":
        y = np.empty_like(x)
        y[..., 0::2], y[..., 1::2] = x[..., 1::2], x[..., 0::2]
        return y
    return np.concatenate([x[..., d // 2:], x[..., : d // 2]], axis=-1)


def check_offsets(g: np.ndarray, o: np.ndarray, absblend: np.ndarray, what: str) -> float:
    err = np.abs(g - o)
    tol = 1e-4 * (np.abs(o) + absblend)
    bad = err > tol
    if bad.any():
        i = np.argwhere(bad)[0]
        raise AssertionError(f"{what}: {bad.sum()} elements off, first {tuple(i)} gpu={g[tuple(i)]} "
                             f"oracle={o[tuple(i)]} tol={tol[tuple(i)]}")
    return float((err / np.maximum(np.abs(o) + absblend, 1e-30)).max()) if err.size else 0.0


U32 = 2.0 ** -24          # unit roundoff of fp32 (round to nearest)


def kv_tolerance(o: np.ndarray, base: np.ndarray, absblend: np.ndarray, n_terms: int, layout: str = "half"):
    """(north-star bound, north-star bound + δ) per element (module docstring)."""
    ao = np.abs(o)
    with np.errstate(divide="ignore"):
        ulp = np.where(ao > 0, 2.0 ** (np.floor(np.log2(np.where(ao > 0, ao, 1.0))) - 7), 0.0)
    north = np.maximum(1e-2 * ao, ulp)
    M = np.abs(base) + absblend
    M = M + _partner(M, layout)
    return north, north + (int(n_terms) + 8) * U32 * M


def check_kv(g: np.ndarray, o: np.ndarray, base: np.ndarray, absblend: np.ndarray, what: str,
             layout: str = "half", n_terms: int = 1) -> Dict:
    """Raises unless every element is within the bound; returns counts: elements
    compared, bit-equal, and how many pass only through the fp32-pipeline term δ."""
    north, tol = kv_tolerance(o, base, absblend, n_terms, layout)
    err = np.abs(g - o)
    bad = ~(err <= tol)
    if bad.any():
        i = np.argwhere(bad)[0]
        raise AssertionError(f"{what}: {bad.sum()} elements off, first {tuple(i)} gpu={g[tuple(i)]} "
                             f"oracle={o[tuple(i)]} tol={tol[tuple(i)]}")
    return {"n": int(g.size), "equal": int((g == o).sum()), "delta_only": int((err > north).sum())}


def merge_counts(acc: Dict, c: Dict) -> Dict:
    for k, v in c.items():
        acc[k] = acc.get(k, 0) + v
    return acc


def distance_tie_positions(dist: np.ndarray, cands, k: int) -> np.ndarray:
    """Positions where the oracle's (distance, slot) order at ranks <= k has a
    relative gap <= TIE_REL between neighbours (the reported tie band)."""
    n = dist.shape[1]
    tie = np.zeros(dist.shape[0], dtype=bool)
    for i in range(dist.shape[0]):
        order = sorted(range(n), key=lambda j: (dist[i, j], cands[j]))
        ds = [dist[i, j] for j in order[: min(k + 1, n)]]
        for a, b in zip(ds, ds[1:]):
            if b - a <= TIE_REL * max(b, 1e-300):
                tie[i] = True
    return tie


def compare(gpu: Dict, ora: Dict, p: synth.Problem, check_values: bool = True) -> Dict:
    gm, om = gpu["match"], ora["match"]
    slots = gpu["slots"]
    stats = {}
    names = ["OK", "EMPTY_POOL", "TOO_LONG", "NO_CANDIDATES", "HIGH_ENTROPY"]
    if not om.candidates:
        assert gm.reason == names[om.reason] and gm.verdict == om.verdict, (gm.reason, om.reason)
        return stats
    assert gm.candidates == om.candidates, (gm.candidates, om.candidates)
    # distances and weights
    gd = f64(gm.dist)[om.candidates][:, : p.L_phi].T
    np.testing.assert_allclose(gd, om.dist, rtol=TIE_REL, atol=0)
    gW = f64(gm.W)[:, : p.L_phi]
    oW = np.zeros_like(gW)
    oW[om.candidates] = om.W.T
    assert np.all(np.abs(gW - oW) <= 1e-5 * np.abs(oW) + 1e-7), np.abs(gW - oW).max()
    gwb = f64(gm.wbar)
    owb = np.zeros_like(gwb)
    owb[om.candidates] = om.wbar
    assert np.all(np.abs(gwb - owb) <= 1e-5 * np.abs(owb) + 1e-7)
    assert abs(gm.entropy - om.H) <= 1e-6 * abs(om.H) + 1e-9, (gm.entropy, om.H)
    assert abs(gm.threshold - om.threshold) <= 1e-6 * om.threshold + 1e-12, (gm.threshold, om.threshold)
    in_band = len(om.candidates) > 1 and abs(om.H - om.threshold) <= TIE_REL * om.threshold
    if not in_band:
        assert gm.verdict == om.verdict and gm.reason == names[om.reason], (gm.reason, om.reason)
    stats["verdict_in_band"] = in_band
    if om.idx is not None:
        tie = distance_tie_positions(om.dist, om.candidates, om.idx.shape[1])
        gi = gm.idx.cpu().numpy()
        mism = np.any(gi != om.idx, axis=1)
        assert not np.any(mism & ~tie), np.argwhere(mism & ~tie)[:5]
        stats["idx_tie_positions"] = int(tie.sum())
        stats["gpu_tie_band_count"] = gm.tie_band_count
    if not check_values or "dst_k" not in gpu:
        return stats
    ph = ora["ph"]
    lay = gpu.get("rope_layout", "half")
    stats["ph_dk_rel"] = check_offsets(f64(gpu["dbg_k"]), ph["dk_hat"], ph["absk"], "placeholder ΔK̂")
    stats["ph_dv_rel"] = check_offsets(f64(gpu["dbg_v"]), ph["dv_hat"], ph["absv"], "placeholder ΔV̂")
    t0, t1 = p.target_start, p.target_start + p.L_phi
    n = len(om.candidates)
    stats["ph_k"] = check_kv(f64(gpu["dst_k"])[:, :, t0:t1], ph["k"], f64(p.base_k), ph["absk"], "K̂ placeholder",
                             lay, n)
    stats["ph_v"] = check_kv(f64(gpu["dst_v"])[:, :, t0:t1], ph["v"], f64(p.base_v), ph["absv"], "V̂ placeholder",
                             lay, n)
    if "pf" in ora:
        pf = ora["pf"]
        c = gpu.get("consumer", 0)
        stats["pf_dk_rel"] = check_offsets(f64(gpu["dbgp_k"]), pf["dk_hat"], pf["absk"], "prefix ΔK̂")
        stats["pf_dv_rel"] = check_offsets(f64(gpu["dbgp_v"]), pf["dv_hat"], pf["absv"], "prefix ΔV̂")
        s0 = p.pf_target_start[c]
        s1 = s0 + p.prefix_lens[c]
        stats["pf_k"] = check_kv(f64(gpu["dst_k"])[:, :, s0:s1], pf["k"], f64(p.pf_base_k[c]), pf["absk"],
                                 "K̂ prefix", lay, n)
        stats["pf_v"] = check_kv(f64(gpu["dst_v"])[:, :, s0:s1], pf["v"], f64(p.pf_base_v[c]), pf["absv"],
                                 "V̂ prefix", lay, n)
    # p_(m,0) copied verbatim (bit-exact)
    assert torch.equal(gpu["dst_k"][:, :, : p.target_start], gpu["p0k"])
    assert torch.equal(gpu["dst_v"][:, :, : p.target_start], gpu["p0v"])
    return stats
