"""KVComm CPU oracle — plain, slow, float64 NumPy, written from PAPER.md.

*** TEST INFRASTRUCTURE ONLY. ***  Only `tests/`, `__graft_entry__.smoke()` and
`bench.py` (its `cpu_baseline` leg and `--impl reference`) may import this module.
The product path (`paper_2510_12872_b200/`) never imports, links or executes it,
and this module imports nothing from the product path: the two share no code.

Every intermediate is float64.  bf16 inputs are widened exactly (callers pass
float64 arrays holding bf16 values); results that the product stores in bf16 are
rounded once, round-to-nearest-even, by `bf16_round` (reading A14).

Citations: "P:n" = /root/reference/PAPER.md line n (with the section / equation),
"S:n" = SPEC.md line n.  DESIGN.md lists every reading (A1..A21) taken where the
paper is silent, ambiguous or garbled.

Notation (§3.3-3.4):
  φ        the new placeholder sample (query), length L_φ
  ψ ∈ 𝒜    anchors of the placeholder's pool; 𝒜_φ ⊆ 𝒜 the candidates (Eq. 5)
  h        token embeddings [L, D_e]                      (reading A1)
  w        softmax(-‖h_φ - h_ψ‖) over anchors              (Eq. 5/6)
  Δk/Δv    stored offsets in the base frame                (reading A10)
  δ        target_start - base_start (RoPE position delta)

Parity status per function: every function below is
pinned by tests/test_oracle_pins.py except where "parity unpinned" is written.
The sample-level distance of reading A4 (`scalar_weights`: Frobenius by default,
SPEC's mean-of-ℓ2 as a switch) and the Eq. 7 weight reading A3 are pinned only by
closed forms / library routines of the chosen reading: no printed value in the
paper separates the readings, so with respect to the paper's intended (unstated)
definition they are "parity unpinned".
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

# ---------------------------------------------------------------------------
# bf16 rounding (reading A14: one RNE rounding at the output)
# ---------------------------------------------------------------------------

BF16_MANT_BITS = 7          # stored mantissa bits of bfloat16
BF16_MIN_EXP = -126         # smallest normal exponent (same range as fp32)
BF16_MAX = (2.0 - 2.0 ** -7) * 2.0 ** 127


def bf16_round(x) -> np.ndarray:
    """Round float64 values to the nearest bfloat16 value, ties to even.

    Definition: with |x| in [2^e, 2^(e+1)), the bf16 spacing is 2^(e-7) (or 2^(-133)
    in the subnormal range); x is rounded to the nearest multiple of the spacing,
    ties to even (np.rint), scaling by powers of two being exact in float64.
    Values beyond the largest finite bf16 after rounding become ±inf.
    """
    x = np.asarray(x, dtype=np.float64)
    out = np.zeros_like(x)
    nz = (x != 0) & np.isfinite(x)
    m, e = np.frexp(x[nz])                       # x = m * 2^e, 0.5 <= |m| < 1
    # |x| in [2^(e-1), 2^e): spacing = 2^(e-1-7); subnormal floor 2^(-126-7)
    spacing_exp = np.maximum(e - 1 - BF16_MANT_BITS, BF16_MIN_EXP - BF16_MANT_BITS)
    q = np.rint(np.ldexp(x[nz], -spacing_exp))
    r = np.ldexp(q, spacing_exp)
    r = np.where(np.abs(r) > BF16_MAX, np.sign(r) * np.inf, r)
    out[nz] = r
    out[~np.isfinite(x)] = x[~np.isfinite(x)]
    return out


# ---------------------------------------------------------------------------
# RoPE (§3.1 P:116-121 "k_n = R_n W_K h_n"; alignment P:145-148)
# ---------------------------------------------------------------------------


HALF, INTERLEAVED = "half", "interleaved"  # RoPE pairings (reading A12)


def rope_rotate(x: np.ndarray, delta: int, inv_freq: np.ndarray, layout: str = HALF) -> np.ndarray:
    """Apply R_δ to key vectors x[..., d] (reading A12).

    For f < d/2 with angle a_f = δ · inv_freq[f] (float64, reading A13), pair f is
    (f, f + d/2) for HF `rotate_half` (default) or (2f, 2f + 1) for the interleaved
    (GPT-J) layout; with (u, w) the pair:
        u' = u cos a_f - w sin a_f
        w' = w cos a_f + u sin a_f
    R_0 = I exactly; R_a R_b = R_{a+b}; R_δ is orthogonal ("orthogonal rotation").
    """
    x = np.asarray(x, dtype=np.float64)
    d = x.shape[-1]
    assert d % 2 == 0 and inv_freq.shape == (d // 2,)
    if delta == 0:
        return x.copy()
    a = float(delta) * np.asarray(inv_freq, dtype=np.float64)
    c, s = np.cos(a), np.sin(a)
    if layout == HALF:
        x1, x2 = x[..., : d // 2], x[..., d // 2:]
        return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1)
    if layout == INTERLEAVED:
        u, w = x[..., 0::2], x[..., 1::2]
        y = np.empty_like(x)
        y[..., 0::2] = u * c - w * s
        y[..., 1::2] = w * c + u * s
        return y
    raise ValueError(layout)


# ---------------------------------------------------------------------------
# Offset measurement — insert path (Algorithm 1)
# ---------------------------------------------------------------------------


def measure_offset(k_real, v_real, s_real: int, k_base, v_base, s_base: int,
                   inv_freq: np.ndarray, layout: str = HALF) -> Tuple[np.ndarray, np.ndarray]:
    """Δk = R_{-(s_real - s_base)} k_real - k_base ;  Δv = v_real - v_base.

    Keys are de-rotated into the base frame before differencing ("always
    de-rotates the stored key by R_{-Δ}", reading A10).  Returns float64; the
    stored pool value is bf16_round of it.
    """
    dk = rope_rotate(k_real, -(s_real - s_base), inv_freq, layout) - np.asarray(k_base, np.float64)
    dv = np.asarray(v_real, np.float64) - np.asarray(v_base, np.float64)
    return dk, dv


# ---------------------------------------------------------------------------
# Anchor prediction (Eq. 5)
# ---------------------------------------------------------------------------


def candidate_slots(anchor_len: Dict[int, int], offsets_present: Dict[int, bool],
                    L_phi: int) -> List[int]:
    """𝒜_φ: anchors at least as long as φ (reading A6: L_ψ >= L_φ) that hold the
    consumer's offsets (reading A9), in ascending slot order."""
    return sorted(s for s, L in anchor_len.items() if L >= L_phi and offsets_present.get(s, False))


def distances(h_phi: np.ndarray, h_anchor: Sequence[np.ndarray]) -> np.ndarray:
    """d[i, j] = ‖h_φ[i] - h_ψj[i]‖₂ for i < L_φ (Eq. 5/6 "‖h_φ - h_ψ‖").

    Anchors longer than φ are truncated to their first L_φ rows (reading A8).
    Returns float64 [L_φ, |𝒜_φ|].
    """
    h_phi = np.asarray(h_phi, dtype=np.float64)
    L_phi = h_phi.shape[0]
    cols = []
    for h in h_anchor:
        diff = h_phi - np.asarray(h, dtype=np.float64)[:L_phi]
        cols.append(np.sqrt(np.sum(diff * diff, axis=1)))
    if not cols:
        return np.zeros((L_phi, 0))
    return np.stack(cols, axis=1)


L2, COSINE = "l2", "cosine"


def cosine_distances(h_phi: np.ndarray, h_anchor: Sequence[np.ndarray]) -> np.ndarray:
    """Table A.4's "Cosine Similarity" variant: per position
    d[i, j] = 1 - cos(h_φ[i], h_ψj[i]) (cos = 0 for a zero row), so that
    softmax(-d) = softmax(cos).  Anchors truncated to the first L_φ rows (A8)."""
    h_phi = np.asarray(h_phi, dtype=np.float64)
    L_phi = h_phi.shape[0]
    cols = []
    for h in h_anchor:
        a = np.asarray(h, dtype=np.float64)[:L_phi]
        num = np.sum(h_phi * a, axis=1)
        den = np.sqrt(np.sum(h_phi * h_phi, axis=1) * np.sum(a * a, axis=1))
        cols.append(1.0 - np.where(den > 0, num / np.where(den > 0, den, 1.0), 0.0))
    if not cols:
        return np.zeros((L_phi, 0))
    return np.stack(cols, axis=1)


def cosine_scalar(h_phi: np.ndarray, h_anchor: Sequence[np.ndarray]) -> np.ndarray:
    """Sample-level cosine distance 1 - <h_φ, h_ψ>_F / (‖h_φ‖_F ‖h_ψ‖_F) (A4 analogue)."""
    h_phi = np.asarray(h_phi, dtype=np.float64)
    L_phi = h_phi.shape[0]
    out = []
    for h in h_anchor:
        a = np.asarray(h, dtype=np.float64)[:L_phi]
        den = np.sqrt(np.sum(h_phi * h_phi) * np.sum(a * a))
        out.append(1.0 - (np.sum(h_phi * a) / den if den > 0 else 0.0))
    return np.array(out)


def softmax_neg(dist: np.ndarray, axis: int = -1) -> np.ndarray:
    """softmax(-dist) along `axis`, temperature 1, max-subtracted (reading A15)."""
    z = -np.asarray(dist, dtype=np.float64)
    z = z - np.max(z, axis=axis, keepdims=True)
    e = np.exp(z)
    return e / np.sum(e, axis=axis, keepdims=True)


def position_weights(dist: np.ndarray, top_k: int = 0,
                     slots: Optional[Sequence[int]] = None) -> Tuple[np.ndarray, Optional[np.ndarray]]:
    """Per-position weights W[i, j] = softmax_j(-d[i, j]) (Eq. 6 "softmax mapping of
    -‖h_φ - h_ψ‖ across the anchor dimension"; per position: reading A2).

    top_k > 0 (reading A16, not in the paper): keep the k anchors with the smallest
    distance per position (ties broken by the smaller slot id), softmax over those,
    zero elsewhere.  Returns (W [L_φ, n], idx [L_φ, k] of slot ids or None).
    """
    n = dist.shape[1]
    if top_k <= 0 or top_k >= n:
        W = softmax_neg(dist, axis=1) if n else np.zeros_like(dist)
        return W, None
    slots = list(range(n)) if slots is None else list(slots)
    W = np.zeros_like(dist, dtype=np.float64)
    idx = np.zeros((dist.shape[0], top_k), dtype=np.int64)
    for i in range(dist.shape[0]):
        order = sorted(range(n), key=lambda j: (dist[i, j], slots[j]))[:top_k]
        W[i, order] = softmax_neg(dist[i, order])
        idx[i] = [slots[j] for j in order]
    return W, idx


FROBENIUS, MEAN_L2 = "frobenius", "mean_l2"


def scalar_weights(dist: np.ndarray, mode: str = FROBENIUS) -> Tuple[np.ndarray, np.ndarray]:
    """Sample-level distance and weight of Eq. 5 / Eq. 7:
    w̄ = softmax(-d̄) with d̄_j = ‖h_φ - h_ψj‖ over the whole sample (reading A4):

      FROBENIUS (default): d̄_j = ‖h_φ - h_ψj[:L_φ]‖_F = sqrt(Σ_i d[i, j]²)
      MEAN_L2: d̄_j = mean_i d[i, j]
    """
    dist = np.asarray(dist, np.float64)
    if mode == FROBENIUS:
        dbar = np.sqrt(np.sum(dist * dist, axis=0))
    elif mode == MEAN_L2:
        dbar = np.mean(dist, axis=0)
    else:
        raise ValueError(mode)
    return dbar, softmax_neg(dbar)


def entropy(w: np.ndarray) -> float:
    """H = -Σ w log w with 0 log 0 = 0 (Eq. 5, sign per reading A5)."""
    w = np.asarray(w, dtype=np.float64)
    nz = w > 0
    return float(-np.sum(w[nz] * np.log(w[nz])))


SHAREABLE, NEW_ANCHOR = 0, 1
R_OK, R_EMPTY_POOL, R_TOO_LONG, R_NO_CANDIDATES, R_HIGH_ENTROPY = 0, 1, 2, 3, 4


@dataclass
class MatchResult:
    verdict: int
    reason: int
    candidates: List[int]
    W: Optional[np.ndarray] = None         # [L_φ, |𝒜_φ|]
    idx: Optional[np.ndarray] = None
    dist: Optional[np.ndarray] = None
    dbar: Optional[np.ndarray] = None
    wbar: Optional[np.ndarray] = None
    H: float = 0.0
    threshold: float = 0.0


def predict(h_phi: np.ndarray, anchor_len: Dict[int, int], anchor_emb: Dict[int, np.ndarray],
            offsets_present: Dict[int, bool], gamma: float, top_k: int = 0,
            scalar: str = FROBENIUS, similarity: str = L2) -> MatchResult:
    """Eq. 5:  NewAnchor ⇔ (L_φ > max_{ψ∈𝒜} L_ψ) ∪ (H_{φ|𝒜} > γ log|𝒜_φ|).

    Readings: the max runs over the whole pool (A7); an empty pool or an empty 𝒜_φ
    is NewAnchor (A19); |𝒜_φ| = 1 gives H = 0 = threshold → Shareable for γ > 0;
    γ = 0 is the no-sharing method of Table 6 → always NewAnchor (A19).
    Weights for Eq. 6/7 are returned alongside (Alg. 1).
    """
    if not (0.0 <= gamma <= 1.0):
        raise ValueError("gamma must lie in [0, 1] (S:237)")
    L_phi = int(np.asarray(h_phi).shape[0])
    if not anchor_len:
        return MatchResult(NEW_ANCHOR, R_EMPTY_POOL, [])
    if L_phi > max(anchor_len.values()):
        return MatchResult(NEW_ANCHOR, R_TOO_LONG, [])
    cand = candidate_slots(anchor_len, offsets_present, L_phi)
    if not cand:
        return MatchResult(NEW_ANCHOR, R_NO_CANDIDATES, [])
    if similarity == L2:
        dist = distances(h_phi, [anchor_emb[s] for s in cand])
        W, idx = position_weights(dist, top_k, cand)
        dbar, wbar = scalar_weights(dist, scalar)
    elif similarity == COSINE:
        dist = cosine_distances(h_phi, [anchor_emb[s] for s in cand])
        W, idx = position_weights(dist, top_k, cand)
        dbar = cosine_scalar(h_phi, [anchor_emb[s] for s in cand])
        wbar = softmax_neg(dbar)
    else:
        raise ValueError(similarity)
    H = entropy(wbar)
    thr = gamma * math.log(len(cand))
    # γ = 0 "refers to the original no-cache-sharing method" (Table 6; reading A19):
    # NewAnchor even for |𝒜_φ| = 1, where Eq. 5 alone gives H = 0 = threshold
    verdict = NEW_ANCHOR if (H > thr or gamma == 0.0) else SHAREABLE
    return MatchResult(verdict, R_HIGH_ENTROPY if verdict == NEW_ANCHOR else R_OK, cand,
                       W, idx, dist, dbar, wbar, H, thr)


# ---------------------------------------------------------------------------
# Offset approximation (Eq. 6, Eq. 7) and alignment
# ---------------------------------------------------------------------------


def blend_placeholder(W: np.ndarray, offsets: Sequence[np.ndarray]) -> np.ndarray:
    """Eq. 6 offset term: Δ̂[..., i, :] = Σ_j W[i, j] · Δ_j[..., i, :].

    offsets[j]: [L, H, ≥L_φ, d] (the anchor's stored placeholder offset, truncated
    to the first L_φ tokens, reading A8).  W: [L_φ, n].
    """
    L_phi = W.shape[0]
    acc = None
    for j, off in enumerate(offsets):
        term = W[:, j][:, None] * np.asarray(off, np.float64)[..., :L_phi, :]
        acc = term if acc is None else acc + term
    return acc


def blend_prefix(wbar: np.ndarray, offsets: Sequence[np.ndarray]) -> np.ndarray:
    """Eq. 7 offset term with one weight per anchor (reading A3):
    Δ̂^p = Σ_j w̄_j · Δ^p_j."""
    acc = None
    for j, off in enumerate(offsets):
        term = float(wbar[j]) * np.asarray(off, np.float64)
        acc = term if acc is None else acc + term
    return acc


def apply_offset(k_base, v_base, dk_hat, dv_hat, delta: int,
                 inv_freq: np.ndarray, layout: str = HALF) -> Tuple[np.ndarray, np.ndarray]:
    """K̂ = R_δ(K_base + Δ̂K),  V̂ = V_base + Δ̂V   (reading A10).

    Offsets live in the base frame, so the sum is re-rotated by δ = target_start -
    base_start (workflow step 3, "aligning Key positions via RoPE
    de-rotation/re-rotation, adding the estimated Key/Value offsets").
    Returns float64 (caller rounds with bf16_round).
    """
    k = rope_rotate(np.asarray(k_base, np.float64) + dk_hat, delta, inv_freq, layout)
    v = np.asarray(v_base, np.float64) + dv_hat
    return k, v


def realign_segment(weights: np.ndarray, k_base, v_base, dk: Sequence[np.ndarray],
                    dv: Sequence[np.ndarray], base_start: int, target_start: int,
                    inv_freq: np.ndarray, kind: str = "placeholder", layout: str = HALF):
    """One segment of Algorithm 1's reuse branch.

    kind = "placeholder": weights is W [L_seg, n] and Eq. 6 applies;
    kind = "prefix":      weights is w̄ [n] and Eq. 7 applies.
    Returns dict with float64 blended offsets and bf16-rounded outputs.
    """
    if kind == "placeholder":
        dk_hat = blend_placeholder(weights, dk)
        dv_hat = blend_placeholder(weights, dv)
    elif kind == "prefix":
        dk_hat = blend_prefix(weights, dk)
        dv_hat = blend_prefix(weights, dv)
    else:
        raise ValueError(kind)
    k, v = apply_offset(k_base, v_base, dk_hat, dv_hat, target_start - base_start, inv_freq, layout)
    return {"dk_hat": dk_hat, "dv_hat": dv_hat, "k": bf16_round(k), "v": bf16_round(v),
            "k64": k, "v64": v}


# ---------------------------------------------------------------------------
# Concatenation and ledger ("updated caches are concatenated")
# ---------------------------------------------------------------------------


class LedgerError(ValueError):
    def __init__(self, kind: str, where: int):
        super().__init__(f"{kind} at position {where}")
        self.kind = kind
        self.where = where


def check_ledger(spans: Sequence[Tuple[int, int]], N: int) -> None:
    """Segments (start, length) must tile [0, N) exactly, in order.
    Raises LedgerError('gap'|'overlap'|'short'|'long', position)."""
    pos = 0
    for start, length in spans:
        if start > pos:
            raise LedgerError("gap", pos)
        if start < pos:
            raise LedgerError("overlap", start)
        pos = start + length
    if pos < N:
        raise LedgerError("gap", pos)
    if pos > N:
        raise LedgerError("long", N)


def concat(parts: Sequence[Tuple[int, np.ndarray]], N: int, axis: int = -2) -> np.ndarray:
    """Concatenate (start, tensor) parts along the token axis after the ledger check."""
    check_ledger([(s, p.shape[axis]) for s, p in parts], N)
    return np.concatenate([p for _, p in parts], axis=axis)


# ---------------------------------------------------------------------------
# Anchor pool metadata: insertion and pruning (§3.3 "Anchor Update", P:273-274;
# Alg. 1)
# ---------------------------------------------------------------------------


@dataclass
class PoolModel:
    """Host metadata of one anchor pool of capacity 𝒱.

    Pruning reading A17: when an insert finds the pool full, the existing anchor
    with the smallest access count is discarded, ties going to the earliest
    inserted ("least frequently accessed anchor among the earliest-added
    entries").  The incoming anchor is never its own victim.
    Slots are reused lowest-free-first.
    """
    capacity: int
    slot_len: Dict[int, int] = field(default_factory=dict)
    access: Dict[int, int] = field(default_factory=dict)
    inserted: Dict[int, int] = field(default_factory=dict)
    next_index: int = 0

    def victim(self) -> int:
        return min(self.slot_len, key=lambda s: (self.access[s], self.inserted[s]))

    def insert(self, L_psi: int) -> Tuple[int, int]:
        evicted = -1
        if len(self.slot_len) >= self.capacity:
            evicted = self.victim()
            self.evict(evicted)
        slot = min(set(range(self.capacity)) - set(self.slot_len))
        self.slot_len[slot] = L_psi
        self.access[slot] = 0
        self.inserted[slot] = self.next_index
        self.next_index += 1
        return slot, evicted

    def evict(self, slot: int) -> None:
        if slot not in self.slot_len:
            raise KeyError(slot)
        del self.slot_len[slot], self.access[slot], self.inserted[slot]

    def record_access(self, slots: Sequence[int]) -> None:
        for s in slots:
            if s not in self.slot_len:
                raise KeyError(s)
            self.access[s] += 1


# ---------------------------------------------------------------------------
# Online pool maintenance over a request stream (Algorithm 1; SURVEY
# §8(f) f1): one placeholder pool shared by several consumers (agents).
# ---------------------------------------------------------------------------


@dataclass
class ConsumerLayout:
    """Where the placeholder and its following prefix sit in consumer c's prompt."""
    t0: int                      # placeholder target start = |p_(c,0)|
    pf_base_k: np.ndarray        # prefix base [L, H, P_c, d], at base position pf_base_start
    pf_base_v: np.ndarray
    pf_base_start: int           # = |p_(c,0)| (reading A11)


class OnlinePoolOracle:
    """Algorithm 1 for one placeholder pool, step by step in the paper's order.

    step(): Eq. 5 prediction; if Shareable, the reuse branch realigns the
    placeholder (Eq. 6) and its neighbouring prefix (Eq. 7) for every consumer
     and counts an access for every candidate (reading A18); otherwise the
    fallback branch takes the dense ("real") caches, measures placeholder and prefix
    offsets against the bases, stores them in bf16 (reading A14) and
    inserts the sample as a new anchor with LFU pruning (reading A17).
    """

    def __init__(self, capacity: int, layouts: Sequence[ConsumerLayout], inv_freq: np.ndarray, gamma: float,
                 scalar: str = FROBENIUS):
        self.pool = PoolModel(capacity)
        self.layouts = list(layouts)
        self.inv = inv_freq
        self.gamma = gamma
        self.scalar = scalar
        self.emb: Dict[int, np.ndarray] = {}
        self.off: Dict[int, list] = {}        # slot -> per consumer (dk_ph, dv_ph, dk_pf, dv_pf)

    def step(self, h_phi, base_k, base_v, real):
        """real(c) -> (k_ph, v_ph, k_pf, v_pf): the dense prefill of consumer c (fallback only).
        Returns (MatchResult, outputs per consumer [(k_ph, v_ph, k_pf, v_pf)], (slot, evicted) or None)."""
        L = h_phi.shape[0]
        r = predict(h_phi, dict(self.pool.slot_len), self.emb, {s: True for s in self.pool.slot_len},
                    self.gamma, 0, self.scalar)
        outs = []
        if r.verdict == SHAREABLE:
            for c, lay in enumerate(self.layouts):
                ph = realign_segment(r.W, base_k, base_v, [self.off[s][c][0] for s in r.candidates],
                                     [self.off[s][c][1] for s in r.candidates], 0, lay.t0, self.inv)
                pf = realign_segment(r.wbar, lay.pf_base_k, lay.pf_base_v,
                                     [self.off[s][c][2] for s in r.candidates],
                                     [self.off[s][c][3] for s in r.candidates], lay.pf_base_start, lay.t0 + L,
                                     self.inv, kind="prefix")
                outs.append((ph["k"], ph["v"], pf["k"], pf["v"]))
            self.pool.record_access(r.candidates)
            return r, outs, None
        slot, ev = self.pool.insert(L)
        if ev >= 0:
            del self.emb[ev], self.off[ev]
        self.emb[slot] = np.asarray(h_phi, np.float64)
        offs = []
        for c, lay in enumerate(self.layouts):
            kph, vph, kpf, vpf = [np.asarray(x, np.float64) for x in real(c)]
            dkp, dvp = measure_offset(kph, vph, lay.t0, base_k, base_v, 0, self.inv)
            dkf, dvf = measure_offset(kpf, vpf, lay.t0 + L, lay.pf_base_k, lay.pf_base_v, lay.pf_base_start,
                                      self.inv)
            offs.append((bf16_round(dkp), bf16_round(dvp), bf16_round(dkf), bf16_round(dvf)))
            outs.append((kph, vph, kpf, vpf))
        self.off[slot] = offs
        return r, outs, (slot, ev)


# ---------------------------------------------------------------------------
# fp8 (e4m3) offset storage — SURVEY §8(f) f3 (~50 % of offset elements have
# |x| < 0.1, "substantial headroom for compression", left to future work).  Not part
# of the paper's method: a storage format for the offsets, defined here so the
# device's codes can be checked bit for bit.
# ---------------------------------------------------------------------------

E4M3_MAX = 448.0
E4M3_MANT_BITS = 3
E4M3_MIN_EXP = -6        # smallest normal exponent; subnormal spacing 2^-9


def e4m3_round(x) -> np.ndarray:
    """Round to the nearest OCP e4m3 ("fn", no inf) value, ties to even, saturating
    to ±448 (the satfinite conversion)."""
    x = np.asarray(x, dtype=np.float64)
    out = np.zeros_like(x)
    nz = x != 0
    m, e = np.frexp(x[nz])                       # |x| in [2^(e-1), 2^e)
    spacing_exp = np.maximum(e - 1 - E4M3_MANT_BITS, E4M3_MIN_EXP - E4M3_MANT_BITS)
    r = np.ldexp(np.rint(np.ldexp(x[nz], -spacing_exp)), spacing_exp)
    out[nz] = np.clip(r, -E4M3_MAX, E4M3_MAX)
    return out


def quantize_rows_fp8(x) -> Tuple[np.ndarray, np.ndarray]:
    """Per row (last axis): scale = max|x| / 448 in float32 (1 for an all-zero row);
    code = e4m3_round(float32(x) / scale) with IEEE float32 division.
    Returns (codes as float64 values of the e4m3 grid, scales float32)."""
    x32 = np.asarray(x, dtype=np.float32)
    amax = np.max(np.abs(x32), axis=-1)
    scale = np.where(amax > 0, amax / np.float32(E4M3_MAX), np.float32(1.0)).astype(np.float32)
    q = e4m3_round((x32 / scale[..., None]).astype(np.float32).astype(np.float64))
    return q, scale


def dequantize_rows_fp8(q, scale) -> np.ndarray:
    """x̂ = code x scale (float64, exact)."""
    return np.asarray(q, np.float64) * np.asarray(scale, np.float64)[..., None]
