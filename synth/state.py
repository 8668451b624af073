"""Device-resident synthetic state for the paper's multi-agent workload
(BASELINE.json configs[1]): anchor pools filled through the public API, per-request
query embeddings, base caches, system-prompt caches and destination caches.

Every random tensor comes from its own keyed, seeded CUDA generator, so a test can
regenerate exactly the bytes of any single input (e.g. one anchor's offsets for one
consumer) to feed the oracle without reading anything back from the CUDA path.
No method arithmetic here.
"""
from __future__ import annotations

import hashlib
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

import numpy as np
import torch

from . import OFFSET_STD, Workload, llama3_inv_freq, five_agent_workload

N_VOCAB = 128256  # Llama-3 vocabulary size


def keyed_gen(seed: int, *keys, device="cuda") -> torch.Generator:
    h = hashlib.sha256(repr((seed,) + keys).encode()).digest()
    g = torch.Generator(device=device)
    g.manual_seed(int.from_bytes(h[:8], "little") & ((1 << 63) - 1))
    return g


def randn_bf16_dev(shape, seed, *keys, std=1.0, device="cuda") -> torch.Tensor:
    g = keyed_gen(seed, *keys, device=device)
    x = torch.randn(*shape, generator=g, device=device, dtype=torch.float32)
    if std != 1.0:
        x.mul_(std)
    return x.to(torch.bfloat16)


@dataclass
class StateInputs:
    """Regenerates any input of the state from (seed, keys)."""
    w: Workload
    seed: int
    layer_range: Tuple[int, int]
    device: str
    anchor_extra: int = 0
    head_range: Optional[Tuple[int, int]] = None

    @property
    def Ls(self):
        return self.layer_range[1] - self.layer_range[0]

    @property
    def Hs(self):
        hb, he = self.head_range or (0, self.w.H)
        return he - hb

    def _layers(self, t):  # generate full-L/H tensors so (layer, head) shards slice identical bytes
        lb, le = self.layer_range
        hb, he = self.head_range or (0, self.w.H)
        if (lb, le) == (0, self.w.L) and (hb, he) == (0, self.w.H):
            return t
        return t[lb:le, hb:he].contiguous()

    def vocab(self) -> torch.Tensor:
        g = keyed_gen(self.seed, "vocab", device=self.device)
        return (torch.randn(N_VOCAB, self.w.D_e, generator=g, device=self.device) *
                (1.0 / np.sqrt(self.w.D_e))).to(torch.bfloat16)

    def anchor_len(self, pool: str, slot: int) -> int:
        return self.w.pools[pool].L_phi + (self.anchor_extra if slot % 2 else 0)

    def anchor_ids(self, pool: str, slot: int) -> torch.Tensor:
        g = keyed_gen(self.seed, "ids", pool, slot, device=self.device)
        return torch.randint(0, N_VOCAB, (self.anchor_len(pool, slot),), generator=g, device=self.device)

    def query_ids(self, pool: str, request: int = 0) -> torch.Tensor:
        L = self.w.pools[pool].L_phi
        base = self.anchor_ids(pool, 0)[:L]
        g = keyed_gen(self.seed, "query", pool, request, device=self.device)
        swap = torch.rand(L, generator=g, device=self.device) < 0.3
        repl = torch.randint(0, N_VOCAB, (L,), generator=g, device=self.device)
        return torch.where(swap, repl, base)

    def offset(self, pool: str, slot: int, consumer: int, kind: str, plane: int) -> torch.Tensor:
        w = self.w
        L = self.anchor_len(pool, slot) if kind == "ph" else w.pools[pool].prefix_len[consumer]
        return self._layers(randn_bf16_dev((w.L, w.H, L, w.d), self.seed, "off", pool, slot, consumer, kind, plane,
                                           std=OFFSET_STD, device=self.device))

    def base(self, pool: str, plane: int, request: int = 0) -> torch.Tensor:
        w = self.w
        return self._layers(randn_bf16_dev((w.L, w.H, w.pools[pool].L_phi, w.d), self.seed, "base", pool, plane,
                                           request, device=self.device))

    def prefix_base(self, pool: str, consumer: int, plane: int) -> torch.Tensor:
        w = self.w
        P = w.pools[pool].prefix_len[consumer]
        return self._layers(randn_bf16_dev((w.L, w.H, P, w.d), self.seed, "pfbase", pool, consumer, plane,
                                           device=self.device))

    def p0(self, agent: int, plane: int) -> torch.Tensor:
        w = self.w
        a = w.agents[agent - 1]
        return self._layers(randn_bf16_dev((w.L, w.H, a.p0, w.d), self.seed, "p0", agent, plane,
                                           device=self.device))


@dataclass
class FiveAgentState:
    inputs: StateInputs
    pools: dict
    queries: Dict[str, torch.Tensor]
    request: object            # paper_2510_12872_b200.request.ReuseRequest
    agents: list
    inv_freq: np.ndarray

    @property
    def w(self) -> Workload:
        return self.inputs.w


def build_five_agent_state(w: Optional[Workload] = None, seed: int = 0, device: int = 0, gamma: float = 0.3,
                           layer_range: Optional[Tuple[int, int]] = None, anchor_extra: int = 0,
                           top_k: int = 0, offset_format: str = "bf16", similarity: str = "l2",
                           scalar_distance: str = "frobenius",
                           emb_shard: Optional[Tuple[int, int]] = None,
                           head_range: Optional[Tuple[int, int]] = None) -> FiveAgentState:
    from paper_2510_12872_b200 import kvcomm as K
    from paper_2510_12872_b200.request import AgentLayout, ReuseRequest, SegmentLayout
    w = w or five_agent_workload()
    dev = f"cuda:{device}"
    lr = layer_range or (0, w.L)
    inp = StateInputs(w, seed, lr, dev, anchor_extra, head_range)
    inv = llama3_inv_freq(w.d)
    vocab = inp.vocab()
    pools = {}
    for name, ps in w.pools.items():
        pool = K.AnchorPool(num_layers=w.L, num_kv_heads=w.H, head_dim=w.d, emb_dim=w.D_e, capacity=w.capacity,
                            max_anchor_len=ps.L_phi + anchor_extra, prefix_len=ps.prefix_len, inv_freq=inv,
                            device=device, layer_range=lr, head_range=head_range, offset_format=offset_format,
                            similarity=similarity,
                            scalar_distance=scalar_distance, emb_shard=emb_shard)
        for slot in range(w.capacity):
            emb = vocab[inp.anchor_ids(name, slot)]
            offs = [K.OffsetGiven(c, inp.offset(name, slot, c, "ph", 0), inp.offset(name, slot, c, "ph", 1),
                                  inp.offset(name, slot, c, "pf", 0), inp.offset(name, slot, c, "pf", 1))
                    for c in range(len(ps.consumers))]
            s, ev = pool.insert(emb, offs)
            assert s == slot and ev == -1
            del offs
        pools[name] = pool
    queries = {name: vocab[inp.query_ids(name)].contiguous() for name in w.pools}
    del vocab
    bases = {name: (inp.base(name, 0), inp.base(name, 1)) for name in w.pools}
    agents = []
    for a in w.agents:
        segs = []
        for s in a.segments:
            if s.kind == "p0":
                continue
            if s.kind == "placeholder":
                bk, bv = bases[s.pool]
                kind = K.PLACEHOLDER
            else:
                bk, bv = inp.prefix_base(s.pool, s.consumer, 0), inp.prefix_base(s.pool, s.consumer, 1)
                kind = K.PREFIX
            segs.append(SegmentLayout(kind, s.pool, s.consumer, bk, bv, s.base_start, s.target_start))
        dst_k = torch.zeros(inp.Ls, inp.Hs, a.N, w.d, dtype=torch.bfloat16, device=dev)
        dst_v = torch.zeros_like(dst_k)
        agents.append(AgentLayout(a.agent, a.N, inp.p0(a.agent, 0), inp.p0(a.agent, 1), segs, dst_k, dst_v))
    req = ReuseRequest(pools, agents, gamma=gamma, top_k=top_k)
    torch.cuda.synchronize()
    return FiveAgentState(inp, pools, queries, req, agents, inv)
