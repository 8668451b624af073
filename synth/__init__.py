"""Seeded synthetic inputs and workload layouts shared by tests, bench.py and smoke().

This module holds NONE of the KVComm method's arithmetic (no distances, softmax,
blending, rotation or offset measurement).  It only draws random tensors and
describes where segments sit in each agent's prompt, so that the oracle
(`oracle/`) and the CUDA path (`paper_2510_12872_b200/`) can be fed identical
bytes without sharing any code.

Input recipe:
  * base K/V            ~ N(0, 1)            rounded to bf16
  * ΔK / ΔV offsets     ~ N(0, 0.148²)       rounded to bf16  (≈50% of |x| < 0.1, PAPER.md A.4.5 P:1518)
  * token embeddings    rows of a vocabulary table ~ N(0, 1/D_e) (‖row‖ ≈ 1), bf16
  * anchor samples      uniform token ids; the query sample is anchor 0's ids with
                        each position re-drawn with probability 0.3 (exact ties,
                        near and far anchors all occur)
  * RoPE frequencies    Llama-3.1 (θ=500000, llama3 scaling ×8, low 1, high 4,
                        original context 8192) for the 8B/70B shapes; θ=10000 plain
                        for the tiny config.  These are model constants handed to
                        both sides as inputs.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Tuple

import numpy as np
import torch

# ----------------------------------------------------------------------------
# Model constants (inputs, not method arithmetic)
# ----------------------------------------------------------------------------


def plain_inv_freq(d: int, theta: float = 10000.0) -> np.ndarray:
    """inv_freq[f] = theta^(-2f/d), f < d/2, as float64 (standard RoPE schedule)."""
    f = np.arange(0, d, 2, dtype=np.float64)
    return 1.0 / (theta ** (f / d))


def llama3_inv_freq(d: int = 128, theta: float = 500000.0, factor: float = 8.0,
                    low_freq_factor: float = 1.0, high_freq_factor: float = 4.0,
                    original_max_position: int = 8192) -> np.ndarray:
    """Llama-3.1 'llama3' RoPE scaling of the plain schedule (model constant)."""
    inv = plain_inv_freq(d, theta)
    low_wl = original_max_position / low_freq_factor
    high_wl = original_max_position / high_freq_factor
    wl = 2.0 * math.pi / inv
    out = np.where(wl > low_wl, inv / factor, inv)
    smooth = (original_max_position / wl - low_freq_factor) / (high_freq_factor - low_freq_factor)
    smoothed = (1.0 - smooth) * out / factor + smooth * out
    medium = (wl >= high_wl) & (wl <= low_wl)
    return np.where(medium, smoothed, out).astype(np.float64)


# ----------------------------------------------------------------------------
# Random tensors
# ----------------------------------------------------------------------------

OFFSET_STD = 0.148


def make_gen(seed: int, device: str | torch.device = "cpu") -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return g


def randn_bf16(shape, gen: torch.Generator, std: float = 1.0,
               device: str | torch.device = "cpu") -> torch.Tensor:
    x = torch.randn(*shape, generator=gen, device=device, dtype=torch.float32)
    if std != 1.0:
        x.mul_(std)
    return x.to(torch.bfloat16)


def vocab_table(n_vocab: int, d_e: int, gen: torch.Generator,
                device: str | torch.device = "cpu") -> torch.Tensor:
    """[n_vocab, D_e] bf16 with rows ~ N(0, 1/D_e)."""
    return randn_bf16((n_vocab, d_e), gen, std=1.0 / math.sqrt(d_e), device=device)


def anchor_token_ids(n_anchors: int, lengths: List[int], n_vocab: int,
                     gen: torch.Generator) -> List[torch.Tensor]:
    """Uniform token ids per anchor (CPU int64)."""
    return [torch.randint(0, n_vocab, (L,), generator=gen) for L in lengths[:n_anchors]]


def query_token_ids(anchor0_ids: torch.Tensor, L_phi: int, n_vocab: int,
                    gen: torch.Generator, p_swap: float = 0.3) -> torch.Tensor:
    """Anchor 0's first L_phi ids with each position re-drawn w.p. p_swap."""
    base = anchor0_ids[:L_phi].clone()
    if base.numel() < L_phi:
        extra = torch.randint(0, n_vocab, (L_phi - base.numel(),), generator=gen)
        base = torch.cat([base, extra])
    swap = torch.rand(L_phi, generator=gen) < p_swap
    repl = torch.randint(0, n_vocab, (L_phi,), generator=gen)
    return torch.where(swap, repl, base)


# ----------------------------------------------------------------------------
# Small self-contained problem (configs[0] and parity cases)
# ----------------------------------------------------------------------------


@dataclass
class Problem:
    """One pool + one placeholder segment (+ optional prefix) for one or more consumers.

    Shapes (all bf16 unless noted, CPU tensors):
      emb_anchor[j]   [L_psi_j, D_e]
      emb_query       [L_phi, D_e]
      dk_ph[c][j], dv_ph[c][j]   [L, H, L_psi_j, d]     (base frame)
      dk_pf[c][j], dv_pf[c][j]   [L, H, P_c, d]
      base_k, base_v             [L, H, L_phi, d]       placeholder base at position 0
      pf_base_k, pf_base_v [c]   [L, H, P_c, d]         prefix base at position pf_base_start
    """
    L: int
    H: int
    d: int
    D_e: int
    inv_freq: np.ndarray
    L_phi: int
    anchor_lens: List[int]
    prefix_lens: List[int]
    emb_anchor: List[torch.Tensor]
    emb_query: torch.Tensor
    dk_ph: List[List[torch.Tensor]]
    dv_ph: List[List[torch.Tensor]]
    dk_pf: List[List[torch.Tensor]]
    dv_pf: List[List[torch.Tensor]]
    base_k: torch.Tensor
    base_v: torch.Tensor
    pf_base_k: List[torch.Tensor]
    pf_base_v: List[torch.Tensor]
    target_start: int
    pf_base_start: int
    pf_target_start: List[int]
    seed: int


def make_problem(seed: int, L: int, H: int, d: int, D_e: int, L_phi: int,
                 anchor_lens: List[int], prefix_lens: List[int], target_start: int,
                 pf_base_start: int = 0, pf_target_start: Optional[List[int]] = None,
                 inv_freq: Optional[np.ndarray] = None, n_vocab: int = 512,
                 p_swap: float = 0.3) -> Problem:
    g = make_gen(seed)
    table = vocab_table(n_vocab, D_e, g)
    ids = anchor_token_ids(len(anchor_lens), anchor_lens, n_vocab, g)
    emb_anchor = [table[i] for i in ids]
    qids = query_token_ids(ids[0] if ids else torch.zeros(0, dtype=torch.long), L_phi, n_vocab, g, p_swap)
    emb_query = table[qids]
    n_cons = len(prefix_lens)
    dk_ph, dv_ph, dk_pf, dv_pf = [], [], [], []
    for c in range(n_cons):
        dk_ph.append([randn_bf16((L, H, Lj, d), g, OFFSET_STD) for Lj in anchor_lens])
        dv_ph.append([randn_bf16((L, H, Lj, d), g, OFFSET_STD) for Lj in anchor_lens])
        dk_pf.append([randn_bf16((L, H, prefix_lens[c], d), g, OFFSET_STD) for _ in anchor_lens])
        dv_pf.append([randn_bf16((L, H, prefix_lens[c], d), g, OFFSET_STD) for _ in anchor_lens])
    base_k = randn_bf16((L, H, L_phi, d), g)
    base_v = randn_bf16((L, H, L_phi, d), g)
    pf_base_k = [randn_bf16((L, H, P, d), g) for P in prefix_lens]
    pf_base_v = [randn_bf16((L, H, P, d), g) for P in prefix_lens]
    if pf_target_start is None:
        pf_target_start = [target_start + L_phi] * n_cons
    if inv_freq is None:
        inv_freq = plain_inv_freq(d)
    return Problem(L, H, d, D_e, inv_freq, L_phi, list(anchor_lens), list(prefix_lens),
                   emb_anchor, emb_query, dk_ph, dv_ph, dk_pf, dv_pf, base_k, base_v,
                   pf_base_k, pf_base_v, target_start, pf_base_start, list(pf_target_start), seed)


def tiny_problem(seed: int = 0) -> Problem:
    """BASELINE.json configs[0]: 2 layers, 2 KV heads, head_dim 16, 4 anchors, one
    32-token shared segment re-prefixed by 8 tokens (δ=+8), θ=10000, D_e=32,
    anchor lengths {32,32,40,48}, one consumer with a 4-token prefix."""
    return make_problem(seed, L=2, H=2, d=16, D_e=32, L_phi=32, anchor_lens=[32, 32, 40, 48],
                        prefix_lens=[4], target_start=8, pf_base_start=8,
                        pf_target_start=[8 + 32], inv_freq=plain_inv_freq(16), n_vocab=64)


# ----------------------------------------------------------------------------
# The paper's 5-agent fully-connected workload (BASELINE.json configs[1])
# ----------------------------------------------------------------------------


@dataclass
class PoolSpec:
    name: str
    L_phi: int                     # sample length (= anchor length for timing)
    consumers: List[int]           # agent ids (1-based) consuming this pool, consumer index = position
    prefix_len: List[int]          # |p_(m,i)| of the prefix following this placeholder, per consumer


@dataclass
class SegmentSpec:
    agent: int
    kind: str                      # "placeholder" | "prefix" | "p0"
    pool: Optional[str]
    consumer: int                  # index into PoolSpec.consumers (-1 for p0)
    length: int
    base_start: int
    target_start: int


@dataclass
class AgentSpec:
    agent: int
    N: int                          # instantiated prompt length
    p0: int
    segments: List[SegmentSpec] = field(default_factory=list)


@dataclass
class Workload:
    name: str
    L: int
    H: int
    d: int
    D_e: int
    capacity: int
    pools: Dict[str, PoolSpec]
    agents: List[AgentSpec]

    @property
    def realigned_tokens(self) -> int:
        return sum(s.length for a in self.agents for s in a.segments if s.kind != "p0")

    @property
    def token_bytes(self) -> int:
        """Bytes of one token's K+V over all layers/heads in bf16: 2*L*H*d*2."""
        return 2 * self.L * self.H * self.d * 2


def five_agent_workload(L: int = 32, H: int = 8, d: int = 128, D_e: int = 4096,
                        n_agents: int = 5, user_len: int = 1024, resp_len: int = 512,
                        prefix_total: int = 512, slot_prefix: int = 32,
                        capacity: int = 20) -> Workload:
    """PAPER.md Table 2 workload: fully-connected agents, 1K user input,
    512 prefix tokens per agent, 512-token responses shared downstream.

    Agent m's prompt (Eq. 1):
      p_(m,0) [prefix_total - slot_prefix*m] | user_question [user_len] | p_(m,1) [slot_prefix]
      | agent_1_current [resp_len] | p_(m,2) | ... | agent_{m-1}_current | p_(m,m)
    Placeholder bases sit at position 0; prefix bases right after p_(m,0) (A11).
    """
    pools: Dict[str, PoolSpec] = {}
    pools["user_question"] = PoolSpec("user_question", user_len, list(range(1, n_agents + 1)),
                                      [slot_prefix] * n_agents)
    for j in range(1, n_agents):
        cons = list(range(j + 1, n_agents + 1))
        pools[f"agent_{j}_current"] = PoolSpec(f"agent_{j}_current", resp_len, cons,
                                                [slot_prefix] * len(cons))
    agents: List[AgentSpec] = []
    for m in range(1, n_agents + 1):
        p0 = prefix_total - slot_prefix * m
        segs = [SegmentSpec(m, "p0", None, -1, p0, 0, 0)]
        pos = p0
        names = ["user_question"] + [f"agent_{j}_current" for j in range(1, m)]
        for name in names:
            ps = pools[name]
            c = ps.consumers.index(m)
            segs.append(SegmentSpec(m, "placeholder", name, c, ps.L_phi, 0, pos))
            pos += ps.L_phi
            segs.append(SegmentSpec(m, "prefix", name, c, ps.prefix_len[c], p0, pos))
            pos += ps.prefix_len[c]
        agents.append(AgentSpec(m, pos, p0, segs))
    return Workload("llama3-8b-5agent", L, H, d, D_e, capacity, pools, agents)


def shared_segment_workload(L: int = 80, H: int = 8, d: int = 128, D_e: int = 8192, seg_len: int = 3072,
                            prefix_len: int = 32, p0: int = 200, capacity: int = 256) -> Workload:
    """BASELINE.json configs[3]: Llama-3-70B shape, one 3K-token
    shared segment re-prefixed for one consumer agent with a 256-anchor pool, k = 256.
    The agent's prompt: p_(1,0) [p0] | segment [seg_len] | p_(1,1) [prefix_len]; the
    placeholder base at 0, the prefix base right after p_(1,0) (reading A11)."""
    pools = {"segment": PoolSpec("segment", seg_len, [1], [prefix_len])}
    segs = [SegmentSpec(1, "p0", None, -1, p0, 0, 0),
            SegmentSpec(1, "placeholder", "segment", 0, seg_len, 0, p0),
            SegmentSpec(1, "prefix", "segment", 0, prefix_len, p0, p0 + seg_len)]
    return Workload("llama3-70b-shared-segment", L, H, d, D_e, capacity, pools,
                    [AgentSpec(1, p0 + seg_len + prefix_len, p0, segs)])


# ----------------------------------------------------------------------------
# Request streams and a synthetic "dense prefill" (stand-in for the model) for the
# online pool maintenance of Algorithm 1.  Inputs only: the
# "true" in-context caches a model would produce, which both the oracle and the
# CUDA path receive; no KVComm arithmetic.
# ----------------------------------------------------------------------------


@dataclass
class StreamSpec:
    L: int = 2
    H: int = 2
    d: int = 32
    D_e: int = 32
    n_vocab: int = 64
    consumers: int = 2
    p0: Tuple[int, ...] = (12, 20)          # |p_(c,0)| per consumer (placeholder target position)
    prefix: Tuple[int, ...] = (4, 6)        # |p_(c,1)| per consumer
    lengths: Tuple[int, ...] = (16, 20, 24, 28, 32, 36, 40)  # sample lengths drawn per request
    n_clusters: int = 3
    p_swap: float = 0.15


def clustered_stream(spec: StreamSpec, n_requests: int, seed: int = 0) -> List[torch.Tensor]:
    """Token-id sequences: each request picks a cluster (a fixed id sequence), a length,
    and re-draws each position with probability p_swap."""
    g = make_gen(seed)
    Lmax = max(spec.lengths)
    centers = [torch.randint(0, spec.n_vocab, (Lmax,), generator=g) for _ in range(spec.n_clusters)]
    out = []
    for _ in range(n_requests):
        c = int(torch.randint(0, spec.n_clusters, (1,), generator=g))
        L = spec.lengths[int(torch.randint(0, len(spec.lengths), (1,), generator=g))]
        ids = centers[c][:L].clone()
        swap = torch.rand(L, generator=g) < spec.p_swap
        ids = torch.where(swap, torch.randint(0, spec.n_vocab, (L,), generator=g), ids)
        out.append(ids)
    return out


class SyntheticPrefill:
    """Deterministic stand-in for the model's caches (CPU, float64 -> bf16):
      base (standalone) cache of a sample: K_b, V_b = E·Wk_b, E·Wv_b (+ RoPE at its own positions
      is irrelevant: the base frame is position 0 for both sides)
      in-context cache for consumer c: base + a context offset tanh(E·A_c)·0.15 that varies
      smoothly with the token embedding (Prop. 2's premise), keys rotated to the target
      positions by RoPE with the given inv_freq.
    Everything is an INPUT to both the oracle and the CUDA path."""

    def __init__(self, spec: StreamSpec, inv_freq: np.ndarray, seed: int = 0):
        g = make_gen(seed + 4242)
        s = spec
        self.spec, self.inv = s, np.asarray(inv_freq, np.float64)
        self.table = vocab_table(s.n_vocab, s.D_e, g).double()
        sc = 1.0 / math.sqrt(s.D_e)
        self.Wk = torch.randn(s.L, s.H, s.D_e, s.d, generator=g, dtype=torch.float64) * sc * 4
        self.Wv = torch.randn(s.L, s.H, s.D_e, s.d, generator=g, dtype=torch.float64) * sc * 4
        self.A = torch.randn(s.consumers, 2, s.L, s.H, s.D_e, s.d, generator=g, dtype=torch.float64) * sc * 4
        self.B = torch.randn(s.consumers, 2, s.L, s.H, s.D_e, s.d, generator=g, dtype=torch.float64) * sc * 4
        self.pf_base = [[randn_bf16((s.L, s.H, P, s.d), g) for _ in range(2)] for P in s.prefix]

    def emb(self, ids: torch.Tensor) -> torch.Tensor:
        return self.table[ids].to(torch.bfloat16)

    def _rot(self, x: torch.Tensor, pos0: int, per_row: bool = True) -> torch.Tensor:
        """The model's RoPE (rotate_half): row i of the token axis goes to absolute position
        pos0 + i (per_row) or every row is moved by pos0 (a uniform shift)."""
        n, d = x.shape[-2], x.shape[-1]
        pos = torch.arange(pos0, pos0 + n, dtype=torch.float64) if per_row else torch.full((n,), float(pos0),
                                                                                            dtype=torch.float64)
        ang = pos[:, None] * torch.from_numpy(self.inv)[None, :]
        c, s_ = torch.cos(ang), torch.sin(ang)
        x1, x2 = x[..., : d // 2], x[..., d // 2:]
        return torch.cat([x1 * c - x2 * s_, x2 * c + x1 * s_], dim=-1)

    def base(self, ids: torch.Tensor):
        """Standalone prefill of the sample at positions 0..L-1 (the anchor/base cache)."""
        E = self.table[ids]
        k = self._rot(torch.einsum("ie,lhed->lhid", E, self.Wk), 0)
        v = torch.einsum("ie,lhed->lhid", E, self.Wv)
        return k.to(torch.bfloat16).contiguous(), v.to(torch.bfloat16).contiguous()

    def real(self, ids: torch.Tensor, c: int):
        """(placeholder K, V, prefix K, V) of the sample inside consumer c's prompt: the
        sample at positions p0_c.., its context deviation a smooth function of the token
        embeddings; the prefix p_(c,1) right after it, shifted by L from its base position."""
        s = self.spec
        E = self.table[ids]
        L = len(ids)
        ok = 0.15 * torch.tanh(torch.einsum("ie,lhed->lhid", E, self.A[c, 0]))
        ov = 0.15 * torch.tanh(torch.einsum("ie,lhed->lhid", E, self.A[c, 1]))
        t0 = s.p0[c]
        kph = self._rot(torch.einsum("ie,lhed->lhid", E, self.Wk) + ok, t0).to(torch.bfloat16)
        vph = (torch.einsum("ie,lhed->lhid", E, self.Wv) + ov).to(torch.bfloat16)
        m = E.mean(0, keepdim=True)
        P = s.prefix[c]
        pk = 0.15 * torch.tanh(torch.einsum("ie,lhed->lhid", m.expand(P, -1), self.B[c, 0]))
        pv = 0.15 * torch.tanh(torch.einsum("ie,lhed->lhid", m.expand(P, -1), self.B[c, 1]))
        pbk, pbv = self.pf_base[c]
        kpf = self._rot(pbk.double() + pk, L, per_row=False).to(torch.bfloat16)
        vpf = (pbv.double() + pv).to(torch.bfloat16)
        return tuple(x.contiguous() for x in (kph, vph, kpf, vpf))
