"""Element-by-element oracle check of a whole multi-agent request — the launch that
bench.py times (ReuseRequest.plan: one batched match over every pool, ONE gated
realign launch over every agent's placeholder, prefix and p_(m,0) segments, with the
consumers of one sample grouped on a shared base).

Test infrastructure.  Every oracle input is regenerated from its keyed seed
(synth.state.StateInputs), never read back from the CUDA path; the oracle
(`oracle/kvcomm_oracle.py`) computes each segment step by step (Eq. 5 match per pool,
Eq. 6 / Eq. 7 blend, R_δ, add, bf16 RNE) on host threads, one (segment, layer)
block per task (NumPy releases the GIL inside its array loops), and every output
element is compared with harness.check_kv.  The counts returned say how many
elements were compared, how many are bit-equal, and how many pass only through the
fp32-pipeline term δ of the tolerance.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
from typing import Dict, Iterable, Optional

import numpy as np
import torch

from oracle import kvcomm_oracle as O
from tests import harness

f64 = harness.f64


def _np64(t: torch.Tensor) -> np.ndarray:
    return t.numpy().astype(np.float64) if t.dtype != torch.bfloat16 else t.float().numpy().astype(np.float64)


def oracle_match(st, name: str, query: Optional[torch.Tensor] = None, gamma: Optional[float] = None,
                 top_k: int = 0, scalar: str = "frobenius", similarity: str = "l2") -> O.MatchResult:
    """Eq. 5 for pool `name`: anchors' embeddings regenerated from their token ids; the
    query is the state's input sample unless another input tensor is given."""
    inp = st.inputs
    vocab = inp.vocab()
    q = f64(query if query is not None else vocab[inp.query_ids(name)])
    lens, embs, pres = {}, {}, {}
    for s in range(st.w.capacity):
        embs[s] = f64(vocab[inp.anchor_ids(name, s)])
        lens[s] = embs[s].shape[0]
        pres[s] = True
    del vocab
    return O.predict(q, lens, embs, pres, st.request.gamma if gamma is None else gamma, top_k, scalar, similarity)


def _segment_layer(l, wts, kind, base, offs, dst, seg, inv, fp8):
    """Oracle for layer l of one segment, compared with the device's rows."""
    store = (lambda x: O.dequantize_rows_fp8(*O.quantize_rows_fp8(x))) if fp8 else (lambda x: x)
    L = seg.length
    bk = _np64(base[0][l:l + 1])
    bv = _np64(base[1][l:l + 1])
    dk = [store(_np64(o[l:l + 1, :, :L])) for o in offs[0]]
    dv = [store(_np64(o[l:l + 1, :, :L])) for o in offs[1]]
    ora = O.realign_segment(wts, bk, bv, dk, dv, seg.base_start, seg.target_start, inv,
                            kind="placeholder" if kind == "ph" else "prefix")
    if kind == "ph":
        absk = O.blend_placeholder(wts, [np.abs(x) for x in dk])
        absv = O.blend_placeholder(wts, [np.abs(x) for x in dv])
    else:
        absk = O.blend_prefix(wts, [np.abs(x) for x in dk])
        absv = O.blend_prefix(wts, [np.abs(x) for x in dv])
    t0 = seg.target_start
    gk = _np64(dst[0][l:l + 1, :, t0:t0 + L])
    gv = _np64(dst[1][l:l + 1, :, t0:t0 + L])
    n = len(offs[0])
    what = f"agent {seg.agent} {kind} {seg.pool} layer {l}"
    ck = harness.check_kv(gk, ora["k"], bk, absk, what + " K", n_terms=n)
    cv = harness.check_kv(gv, ora["v"], bv, absv, what + " V", n_terms=n)
    return harness.merge_counts(ck, cv)


def check_request(st, matches: Dict[str, O.MatchResult], reused: Iterable[int], fp8: bool = False,
                  workers: Optional[int] = None) -> Dict:
    """Compares every realigned and copied element of every reused agent's prompt cache
    with the oracle.  Returns element counts (see module docstring)."""
    inp = st.inputs
    w = st.w
    reused = set(reused)
    workers = workers or os.cpu_count() or 4
    counts: Dict[str, int] = {"segments": 0, "copied_equal": 0}
    with cf.ThreadPoolExecutor(max_workers=workers) as ex:
        for a_spec, a_dev in zip(w.agents, st.agents):
            if a_spec.agent not in reused:
                continue
            dst = (a_dev.dst_k.cpu(), a_dev.dst_v.cpu())
            for plane in range(2):   # p_(m,0) copied verbatim (reading A20)
                p0 = inp.p0(a_spec.agent, plane).cpu()
                assert torch.equal(dst[plane][:, :, :a_spec.p0], p0), f"agent {a_spec.agent} p0 plane {plane}"
                counts["copied_equal"] += p0.numel()
            for seg in a_spec.segments:
                if seg.kind == "p0":
                    continue
                m = matches[seg.pool]
                assert m.verdict == O.SHAREABLE, (seg.pool, m.reason)
                kind = "ph" if seg.kind == "placeholder" else "pf"
                if kind == "ph":
                    wts = m.W
                    base = (inp.base(seg.pool, 0).cpu(), inp.base(seg.pool, 1).cpu())
                else:
                    wts = m.wbar
                    base = (inp.prefix_base(seg.pool, seg.consumer, 0).cpu(),
                            inp.prefix_base(seg.pool, seg.consumer, 1).cpu())
                offs = tuple([inp.offset(seg.pool, s, seg.consumer, kind, plane)[:, :, :seg.length].cpu()
                              for s in m.candidates] for plane in range(2))
                futs = [ex.submit(_segment_layer, l, wts, kind, base, offs, dst, seg, st.inv_freq, fp8)
                        for l in range(inp.Ls)]
                for f in futs:
                    harness.merge_counts(counts, f.result())
                counts["segments"] += 1
                del offs
    return counts


def report(name: str, counts: Dict) -> None:
    """Prints the counts (pytest -s) and appends them to $KVCOMM_PARITY_REPORT if set."""
    import json
    line = json.dumps({"case": name, **counts})
    print(line)
    path = os.environ.get("KVCOMM_PARITY_REPORT")
    if path:
        with open(path, "a") as f:
            f.write(line + "\n")
