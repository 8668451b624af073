"""Online anchor-pool maintenance over a request stream (Algorithm 1, PAPER.md
P:745-801) for one placeholder pool shared by several consumers.

step(): match the sample against the pool (Eq. 5, one launch pair); if Shareable,
realign the placeholder (Eq. 6) and its neighbouring prefix (Eq. 7) for every
consumer in one launch and count an access for every candidate (reading A18);
otherwise take the dense caches from the caller's prefill (the model),
copy them into the consumers' prompts, and insert the sample as a new anchor whose
placeholder and prefix offsets are MEASURED on the device against the bases
 with LFU pruning when the pool is full (reading A17).

Host bookkeeping only; every step runs in libkvcomm's kernels.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, List, Optional, Sequence, Tuple

import torch

from . import kvcomm as K


@dataclass
class ConsumerSlot:
    """Consumer c's prompt around the placeholder: p_(c,0) | φ | p_(c,1) | ..."""
    t0: int                       # placeholder target start (|p_(c,0)|)
    pf_base_k: torch.Tensor       # prefix base [Ls, Hs, P_c, d] at base position pf_base_start
    pf_base_v: torch.Tensor
    pf_base_start: int
    dst_k: torch.Tensor           # [Ls, Hs, N_c, d] prompt cache (rows t0 .. t0+L+P_c written)
    dst_v: torch.Tensor


@dataclass
class StepResult:
    verdict: int
    reason: str
    candidates: List[int]
    slot: int = -1                # fallback: slot the sample was inserted into
    evicted: int = -1             # fallback: slot pruned to make room (-1: none)
    entropy: float = 0.0


class OnlinePool:
    def __init__(self, pool: K.AnchorPool, consumers: Sequence[ConsumerSlot], gamma: float = 0.3,
                 top_k: int = 0):
        if len(consumers) != len(pool.prefix_len):
            raise ValueError("one ConsumerSlot per pool consumer")
        self.pool, self.consumers, self.gamma, self.top_k = pool, list(consumers), gamma, top_k
        self.requests = 0
        self.reused = 0

    @property
    def reuse_rate(self) -> float:
        return self.reused / self.requests if self.requests else 0.0

    def step(self, emb: torch.Tensor, base_k: torch.Tensor, base_v: torch.Tensor,
             prefill: Callable[[int], Tuple[torch.Tensor, torch.Tensor, torch.Tensor, torch.Tensor]],
             stream=None) -> StepResult:
        """prefill(c) -> (K_ph, V_ph, K_pf, V_pf) device bf16: the dense in-context caches of
        consumer c (called only on the fallback branch)."""
        L = emb.shape[0]
        self.requests += 1
        m = self.pool.match(emb, consumer=K.ALL_CONSUMERS, gamma=self.gamma, top_k=self.top_k, stream=stream)
        if m.shareable:                                   # reuse branch
            segs = []
            for c, cs in enumerate(self.consumers):
                segs.append(K.Segment(self.pool, c, K.PLACEHOLDER, m.W, m.candidates, base_k, base_v, 0, cs.t0,
                                      cs.dst_k, cs.dst_v))
                segs.append(K.Segment(self.pool, c, K.PREFIX, m.wbar, m.candidates, cs.pf_base_k, cs.pf_base_v,
                                      cs.pf_base_start, cs.t0 + L, cs.dst_k, cs.dst_v))
            K.realign_segments(segs, stream=stream)
            self.pool.record_access(m.candidates)
            self.reused += 1
            return StepResult(m.verdict, m.reason, m.candidates, entropy=m.entropy)
        # fallback branch: dense caches, measured offsets, new anchor
        offs, copies = [], []
        for c, cs in enumerate(self.consumers):
            kph, vph, kpf, vpf = prefill(c)
            offs.append(K.OffsetMeasure(c, ph_real=(kph, vph, cs.t0), ph_base=(base_k, base_v, 0),
                                        pf_real=(kpf, vpf, cs.t0 + L),
                                        pf_base=(cs.pf_base_k, cs.pf_base_v, cs.pf_base_start)))
            copies.append(K.Segment(self.pool, c, K.COPY, None, [], kph, vph, 0, cs.t0, cs.dst_k, cs.dst_v))
            copies.append(K.Segment(self.pool, c, K.COPY, None, [], kpf, vpf, 0, cs.t0 + L, cs.dst_k, cs.dst_v))
        slot, ev = self.pool.insert(emb, offs, stream=stream)
        K.realign_segments(copies, stream=stream)         # the dense caches serve this request
        return StepResult(m.verdict, m.reason, m.candidates, slot, ev, m.entropy)
