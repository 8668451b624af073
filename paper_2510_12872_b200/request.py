"""Algorithm 1's reuse branch for all agents of one request.

Every placeholder pool's sample is matched once (weights depend only on the sample
and the pool, reading A21; Alg. 1 evaluates Eq. 5 for every placeholder before
branching).  Every agent whose placeholders are all Shareable gets all its
placeholder and prefix segments realigned and its p_(m,0) rows copied.  Agents
with any NewAnchor verdict take the dense fallback, which needs the model
and is outside this library: they are reported, not processed.

Two equivalent executions:
  run()          the native plan (kvcomm_plan_*): ONE batched match launch and ONE
                 realign launch per request, the branch taken on the device, no
                 host synchronisation needed (this is what bench.py times);
  run_unfused()  the individual C-ABI calls (match_many with one host sync, host
                 branch, realign_segments with COPY segments, ledger check).

Host bookkeeping only; all arithmetic runs in libkvcomm's kernels.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, List, Optional

import torch

from . import kvcomm as K


@dataclass
class SegmentLayout:
    kind: int                    # K.PLACEHOLDER | K.PREFIX
    pool: str                    # placeholder (pool) name this segment belongs to
    consumer: int                # consumer index of this (agent, slot) in the pool
    base_k: torch.Tensor         # [Ls, Hs, L_seg, d]
    base_v: torch.Tensor
    base_start: int
    target_start: int


@dataclass
class AgentLayout:
    agent: int
    N: int                       # prompt length
    p0_k: torch.Tensor           # [Ls, Hs, |p_(m,0)|, d]  system prompt cache (copied verbatim)
    p0_v: torch.Tensor
    segments: List[SegmentLayout]
    dst_k: torch.Tensor          # [Ls, Hs, N, d]
    dst_v: torch.Tensor


@dataclass
class RequestResult:
    matches: Dict[str, K.Match]
    reused_agents: List[int]
    fallback_agents: List[int]
    realigned_tokens: int
    blended_rows: int            # Σ_segments n_candidates * L_seg (for the byte model)
    copied_tokens: int


class ReuseRequest:
    """run() executes the request through the native plan (kvcomm_plan_*: one match
    launch + one gated realign launch, device-side branch); run_unfused() does the
    same through the individual calls (match_many, realign_segments, concat) with
    the branch taken on the host — both produce identical caches."""

    def __init__(self, pools: Dict[str, K.AnchorPool], agents: List[AgentLayout], gamma: float = 0.3,
                 top_k: int = 0):
        self.pools, self.agents, self.gamma, self.top_k = pools, agents, gamma, top_k
        self._match_out: Dict[str, Optional[K.Match]] = {n: None for n in pools}
        self.names = list(pools)
        self._plan: Optional[K.Plan] = None

    @property
    def plan(self) -> K.Plan:
        if self._plan is None:
            idx = {n: i for i, n in enumerate(self.names)}
            L_phi = {}
            segs = []
            for ai, a in enumerate(self.agents):
                for s in a.segments:
                    if s.kind == K.PLACEHOLDER:
                        L_phi[s.pool] = s.base_k.shape[2]
                    segs.append(K.PlanSegment(ai, idx[s.pool], s.kind, s.consumer, s.base_k, s.base_v, s.base_start,
                                              s.target_start))
                if a.p0_k.shape[2] > 0:
                    segs.append(K.PlanSegment(ai, 0, K.COPY, 0, a.p0_k, a.p0_v, 0, 0))
            matches = [(self.pools[n], L_phi[n], self.gamma, self.top_k) for n in self.names]
            self._plan = K.Plan(matches, segs, [(a.N, a.dst_k, a.dst_v) for a in self.agents])
        return self._plan

    def shard_matching(self, rank: int, world: int, device: int, group=None) -> None:
        """Layer-sharded request on `world` ranks: compute 1/world of the match positions
        here and exchange them (shard.MatchShard) instead of recomputing every distance."""
        from .shard import MatchShard
        self._mshard = MatchShard(self.plan, rank, world, device, group) if world > 1 else None

    def run(self, queries: Dict[str, torch.Tensor], stream=None, sync: bool = True) -> Optional["RequestResult"]:
        """Plan path.  sync=False only enqueues (collect with results())."""
        self.launch([queries[n] for n in self.names], stream=stream, sync=sync)
        return self.results() if sync else None

    def launch(self, qlist: List[torch.Tensor], stream=None, sync: bool = False) -> None:
        """Enqueue one run of the plan (queries in self.names order); sharded matching
        when shard_matching() was called."""
        if getattr(self, "_mshard", None) is not None:
            self._mshard.run(qlist, stream=stream, sync=sync)
        else:
            self.plan.run(qlist, sync=sync, stream=stream)

    def results(self) -> "RequestResult":
        ms, reused_flags = self.plan.results()
        matches = dict(zip(self.names, ms))
        reused = [a.agent for a, f in zip(self.agents, reused_flags) if f]
        fallback = [a.agent for a, f in zip(self.agents, reused_flags) if not f]
        toks = rows = copied = 0
        for a in self.agents:
            if a.agent not in reused:
                continue
            for s in a.segments:
                toks += s.base_k.shape[2]
                rows += s.base_k.shape[2] * len(matches[s.pool].candidates)
            copied += a.p0_k.shape[2]
        for name, m in matches.items():            # reading A18: +1 per Shareable turn
            if m.shareable:
                self.pools[name].record_access(m.candidates)
        return RequestResult(matches, reused, fallback, toks, rows, copied)

    def match(self, queries: Dict[str, torch.Tensor], stream=None) -> Dict[str, K.Match]:
        names = list(queries)
        ms = K.match_many([(self.pools[n], queries[n]) for n in names], consumer=K.ALL_CONSUMERS,
                          gamma=self.gamma, top_k=self.top_k, outs=[self._match_out[n] for n in names],
                          stream=stream)
        out = dict(zip(names, ms))
        self._match_out.update(out)
        return out

    def segments(self, matches: Dict[str, K.Match]):
        segs, reused, fallback, toks, rows, copied = [], [], [], 0, 0, 0
        for a in self.agents:
            names = {s.pool for s in a.segments}
            if not all(matches[n].shareable for n in names):
                fallback.append(a.agent)
                continue
            reused.append(a.agent)
            for s in a.segments:
                m = matches[s.pool]
                w = m.W if s.kind == K.PLACEHOLDER else m.wbar
                segs.append(K.Segment(self.pools[s.pool], s.consumer, s.kind, w, m.candidates, s.base_k, s.base_v,
                                      s.base_start, s.target_start, a.dst_k, a.dst_v))
                toks += s.base_k.shape[2]
                rows += s.base_k.shape[2] * len(m.candidates)
            if a.p0_k.shape[2] > 0:   # p_(m,0) copied verbatim in the same launch (reading A20)
                segs.append(K.Segment(self.pools[a.segments[0].pool], 0, K.COPY, None, [], a.p0_k, a.p0_v, 0, 0,
                                      a.dst_k, a.dst_v))
                copied += a.p0_k.shape[2]
        return segs, reused, fallback, toks, rows, copied

    def realign(self, segs, stream=None) -> None:
        K.realign_segments(segs, stream=stream)

    def check_ledger(self, reused: List[int], stream=None) -> None:
        for a in self.agents:
            if a.agent not in reused:
                continue
            parts = [(0, a.p0_k.shape[2], None, None)]
            for s in sorted(a.segments, key=lambda s: s.target_start):
                parts.append((s.target_start, s.base_k.shape[2], None, None))
            K.concat_prefill_cache(parts, a.N, a.dst_k, a.dst_v, stream=stream)

    def run_unfused(self, queries: Dict[str, torch.Tensor], stream=None) -> RequestResult:
        matches = self.match(queries, stream)
        segs, reused, fallback, toks, rows, copied = self.segments(matches)
        self.check_ledger(reused, stream)      # host-only: raises before any launch on a bad layout
        if segs:
            self.realign(segs, stream)
        for name, m in matches.items():            # reading A18: +1 per Shareable turn
            if m.shareable:
                self.pools[name].record_access(m.candidates)
        return RequestResult(matches, reused, fallback, toks, rows, copied)
