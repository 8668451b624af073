"""Thin Python binding of libkvcomm (include/kvcomm.h): argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels; this module turns
torch tensors into (pointer, shape, stride) arguments, allocates output buffers with
torch (device-memory plumbing) and raises KVCommError on a non-OK status.  There is
no CPU fallback.

Tensor conventions: K/V of one model shard are bf16 CUDA tensors shaped
[Ls, Hs, T, d] whose last two dims are dense (a token slice of a bigger cache is
fine: the (layer, head) row stride is read from the tensor's strides).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np
import torch

from . import _lib as L
from ._lib import (ALL_CONSUMERS, COPY, NEW_ANCHOR, OFFSET_GIVEN, OFFSET_MEASURE, PLACEHOLDER, PREFIX,
                   SHAREABLE, KVCommError)

__all__ = ["AnchorPool", "OffsetGiven", "OffsetMeasure", "Match", "Segment", "realign_segments",
           "realign_segment", "prepare_segments", "realign_prepared", "concat_prefill_cache", "kernel_launch_count", "KVCommError", "ALL_CONSUMERS",
           "SHAREABLE", "NEW_ANCHOR", "PLACEHOLDER", "PREFIX", "COPY", "match_many", "Plan", "PlanSegment"]


def _stream_handle(stream: Optional[torch.cuda.Stream]) -> int:
    s = torch.cuda.current_stream() if stream is None else stream
    return int(s.cuda_stream)


def _rows_ld(t: torch.Tensor, what: str) -> int:
    """Row stride (in rows) between (layer, head) blocks of a [Ls, Hs, T, d] tensor."""
    if t.dim() != 4:
        raise ValueError(f"{what}: expected [Ls, Hs, T, d], got {tuple(t.shape)}")
    if not t.is_cuda or t.dtype != torch.bfloat16:
        raise ValueError(f"{what}: expected a bf16 CUDA tensor")
    Ls, Hs, T, d = t.shape
    s0, s1, s2, s3 = t.stride()
    if s3 != 1 or (T > 1 and s2 != d) or s1 % d != 0 or (Ls > 1 and s0 != Hs * s1):
        raise ValueError(f"{what}: strides {t.stride()} are not [Ls,Hs,ld,d] row-major")
    return s1 // d


def _dst_layout(t, what: str) -> Tuple[int, int]:
    """(row stride between heads, heads per layer) of a destination [Ls, Hs, N, d]: a
    row-major tensor, or a head slice full[l0:l1, h0:h1] of a consumer's [L, H, N, d]
    cache (layer stride = H heads; kvcomm_realign_desc.dst_heads)."""
    if t.dim() != 4:
        raise ValueError(f"{what}: expected [Ls, Hs, N, d], got {tuple(t.shape)}")
    if not t.is_cuda or t.dtype != torch.bfloat16:
        raise ValueError(f"{what}: expected a bf16 CUDA tensor")
    Ls, Hs, N, d = t.shape
    s0, s1, s2, s3 = t.stride()
    if s3 != 1 or (N > 1 and s2 != d) or s1 % d != 0 or s1 < N * d:
        raise ValueError(f"{what}: strides {t.stride()} are not [Ls,Hs,ld,d] row-major")
    if Ls == 1:
        return s1 // d, Hs
    if s0 % s1 != 0 or s0 // s1 < Hs:
        raise ValueError(f"{what}: layer stride {s0} is not a whole number (>= {Hs}) of head blocks of {s1}")
    return s1 // d, s0 // s1


def _view(k: Optional[torch.Tensor], v: Optional[torch.Tensor], start: int = 0, what: str = "kv") -> L.KVView:
    if k is None:
        return L.KVView()
    ld = _rows_ld(k, what + ".k")
    if v.shape != k.shape or _rows_ld(v, what + ".v") != ld:
        raise ValueError(f"{what}: k and v differ in shape/stride")
    return L.KVView(k.data_ptr(), v.data_ptr(), ld, int(start), 0)


def kernel_launch_count() -> int:
    return int(L.lib().kvcomm_kernel_launch_count())


@dataclass
class OffsetGiven:
    """Precomputed offsets of one consumer, base frame (reading A10)."""
    consumer: int
    dk_ph: Optional[torch.Tensor] = None   # [Ls, Hs, L_psi, d]
    dv_ph: Optional[torch.Tensor] = None
    dk_pf: Optional[torch.Tensor] = None   # [Ls, Hs, P_c, d]
    dv_pf: Optional[torch.Tensor] = None

    def desc(self) -> L.OffsetDesc:
        return L.OffsetDesc(self.consumer, OFFSET_GIVEN, _view(self.dk_ph, self.dv_ph, what="dk_ph"),
                            _view(self.dk_pf, self.dv_pf, what="dk_pf"))


@dataclass
class OffsetMeasure:
    """Offsets measured on device from real (in-context) and base caches (Alg. 1).
    Each cache is (K, V, absolute start position)."""
    consumer: int
    ph_real: Optional[Tuple[torch.Tensor, torch.Tensor, int]] = None
    ph_base: Optional[Tuple[torch.Tensor, torch.Tensor, int]] = None
    pf_real: Optional[Tuple[torch.Tensor, torch.Tensor, int]] = None
    pf_base: Optional[Tuple[torch.Tensor, torch.Tensor, int]] = None

    def desc(self) -> L.OffsetDesc:
        d = L.OffsetDesc()
        d.consumer = self.consumer
        d.mode = OFFSET_MEASURE
        if self.ph_real is not None:
            d.ph_real = _view(*self.ph_real, what="ph_real")
            d.ph_base = _view(*self.ph_base, what="ph_base")
        if self.pf_real is not None:
            d.pf_real = _view(*self.pf_real, what="pf_real")
            d.pf_base = _view(*self.pf_base, what="pf_base")
        return d


@dataclass
class Match:
    verdict: int
    reason: str
    candidates: List[int]
    top_k: int
    entropy: float
    threshold: float
    verdict_in_tie_band: bool
    tie_band_count: int
    W: Optional[torch.Tensor] = None        # [capacity, ld_w] fp32, slot-major
    wbar: Optional[torch.Tensor] = None     # [capacity] fp32
    idx: Optional[torch.Tensor] = None      # [L_phi, top_k] int32
    dist: Optional[torch.Tensor] = None     # [capacity, ld_w] fp64

    @property
    def shareable(self) -> bool:
        return self.verdict == SHAREABLE


class _DevView:
    """__cuda_array_interface__ wrapper to view library-owned device memory."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"data": (int(ptr), False), "shape": tuple(shape), "typestr": typestr,
                                         "version": 3, "strides": None}


class AnchorPool:
    """Device-resident anchor pool of one placeholder (§3.3, Table A.1)."""

    def __init__(self, *, num_layers: int, num_kv_heads: int, head_dim: int, emb_dim: int, capacity: int,
                 max_anchor_len: int, prefix_len: Sequence[int], inv_freq, device: int = 0,
                 layer_range: Optional[Tuple[int, int]] = None, head_range: Optional[Tuple[int, int]] = None,
                 scalar_distance: str = "frobenius", similarity: str = "l2", offset_format: str = "bf16",
                 placement: str = "device", rope_layout: str = "half",
                 emb_shard: Optional[Tuple[int, int]] = None):
        """emb_shard = (rank, world): hold only the embedding rows of the position blocks
        this rank matches under sharded matching (1/world of them)."""
        lb, le = layer_range or (0, num_layers)
        hb, he = head_range or (0, num_kv_heads)
        self.Ls, self.Hs, self.d, self.De = le - lb, he - hb, head_dim, emb_dim
        self.capacity, self.max_anchor_len = capacity, max_anchor_len
        self.prefix_len = [int(x) for x in prefix_len]
        self.device = torch.device("cuda", device)
        self.offset_format = offset_format
        self.rope_layout = rope_layout
        pl = (C.c_int32 * len(self.prefix_len))(*self.prefix_len)
        inv = np.ascontiguousarray(np.asarray(inv_freq, dtype=np.float64))
        cfg = L.PoolConfig(device, num_layers, lb, le, num_kv_heads, hb, he, head_dim, emb_dim, capacity,
                           max_anchor_len, len(self.prefix_len),
                           {"frobenius": L.SCALAR_FROBENIUS, "mean_l2": L.SCALAR_MEAN_L2}[scalar_distance],
                           {"l2": L.SIM_L2, "cosine": L.SIM_COSINE}[similarity],
                           {"bf16": L.OFFSET_BF16, "fp8": L.OFFSET_FP8_E4M3}[offset_format],
                           {"device": L.PLACE_DEVICE, "host": L.PLACE_HOST}[placement],
                           {"half": L.ROPE_HALF, "interleaved": L.ROPE_INTERLEAVED}[rope_layout],
                           emb_shard[0] if emb_shard else 0, emb_shard[1] if emb_shard else 0, pl,
                           inv.ctypes.data_as(C.POINTER(C.c_double)))
        self.emb_shard = tuple(emb_shard) if emb_shard else None
        h = C.c_void_p()
        L.check(L.lib().kvcomm_anchor_pool_create(C.byref(cfg), C.byref(h)))
        self._h = h

    @property
    def handle(self) -> int:
        if self._h is None:
            raise RuntimeError("pool destroyed")
        return self._h.value

    # -- checkpoint ------------------------------------------------------------
    def save(self, path: str, stream=None) -> None:
        """Write the pool (configuration, LFU metadata, every stored anchor) to `path`
        (kvcomm_anchor_pool_save)."""
        L.check(L.lib().kvcomm_anchor_pool_save(self.handle, os.fsencode(path), _stream_handle(stream)))

    @classmethod
    def load(cls, path: str, device: int = 0) -> "AnchorPool":
        """Recreate a saved pool on `device`, slot for slot (kvcomm_anchor_pool_load)."""
        h = C.c_void_p()
        L.check(L.lib().kvcomm_anchor_pool_load(os.fsencode(path), device, C.byref(h)))
        self = cls.__new__(cls)
        self._h = h
        cfg = L.PoolConfig()
        L.check(L.lib().kvcomm_anchor_pool_get_config(h, C.byref(cfg), None, None))
        pl = (C.c_int32 * cfg.num_consumers)()
        inv = (C.c_double * (cfg.head_dim // 2))()
        L.check(L.lib().kvcomm_anchor_pool_get_config(h, C.byref(cfg), pl, inv))
        self.Ls, self.Hs = cfg.layer_end - cfg.layer_begin, cfg.head_end - cfg.head_begin
        self.d, self.De = cfg.head_dim, cfg.emb_dim
        self.capacity, self.max_anchor_len = cfg.capacity, cfg.max_anchor_len
        self.prefix_len = list(pl)
        self.device = torch.device("cuda", device)
        self.offset_format = {L.OFFSET_BF16: "bf16", L.OFFSET_FP8_E4M3: "fp8"}[cfg.offset_format]
        self.rope_layout = {L.ROPE_HALF: "half", L.ROPE_INTERLEAVED: "interleaved"}[cfg.rope_layout]
        self.inv_freq = list(inv)
        self.emb_shard = (cfg.emb_shard_rank, cfg.emb_shard_world) if cfg.emb_shard_world > 1 else None
        return self

    def destroy(self) -> None:
        if self._h is not None:
            L.check(L.lib().kvcomm_anchor_pool_destroy(self._h))
            self._h = None

    def __del__(self):
        try:
            if getattr(self, "_h", None) is not None:
                L.lib().kvcomm_anchor_pool_destroy(self._h)
                self._h = None
        except Exception:
            pass

    def nbytes(self) -> int:
        b = C.c_int64()
        L.check(L.lib().kvcomm_anchor_pool_bytes(self.handle, C.byref(b)))
        return b.value

    # -- a0 ------------------------------------------------------------------
    def insert(self, emb: torch.Tensor, offsets: Sequence = (), stream=None) -> Tuple[int, int]:
        if emb.dim() != 2 or emb.shape[1] != self.De or emb.dtype != torch.bfloat16 or not emb.is_contiguous():
            raise ValueError("emb must be a contiguous bf16 [L_psi, D_e] tensor")
        descs = (L.OffsetDesc * max(len(offsets), 1))(*[o.desc() for o in offsets])
        slot, ev = C.c_int32(), C.c_int32()
        L.check(L.lib().kvcomm_anchor_pool_insert(self.handle, emb.shape[0], emb.data_ptr(), descs, len(offsets),
                                                  _stream_handle(stream), C.byref(slot), C.byref(ev)))
        return slot.value, ev.value

    def set_offsets(self, slot: int, offsets: Sequence, stream=None) -> None:
        descs = (L.OffsetDesc * max(len(offsets), 1))(*[o.desc() for o in offsets])
        L.check(L.lib().kvcomm_anchor_pool_set_offsets(self.handle, slot, descs, len(offsets),
                                                       _stream_handle(stream)))

    def evict(self, slot: int) -> None:
        L.check(L.lib().kvcomm_anchor_pool_evict(self.handle, slot))

    def record_access(self, slots: Sequence[int]) -> None:
        arr = (C.c_int32 * max(len(slots), 1))(*slots)
        L.check(L.lib().kvcomm_anchor_pool_record_access(self.handle, arr, len(slots)))

    def slot_info(self, slot: int) -> dict:
        s = L.SlotInfo()
        L.check(L.lib().kvcomm_anchor_pool_slot_info(self.handle, slot, C.byref(s)))
        return {"occupied": bool(s.occupied), "length": s.length, "access_count": s.access_count,
                "insertion_index": s.insertion_index, "ph_present_mask": s.ph_present_mask,
                "pf_present_mask": s.pf_present_mask}

    def offset_view(self, slot: int, consumer: int, which: str = "ph", rows: Optional[int] = None):
        """bf16 pools: (ΔK, ΔV) stored for (slot, consumer) as [Ls, Hs, rows, d] views of pool memory."""
        k, v, ld = C.c_void_p(), C.c_void_p(), C.c_int64()
        L.check(L.lib().kvcomm_anchor_pool_offset_view(self.handle, slot, consumer, 0 if which == "ph" else 1,
                                                       C.byref(k), C.byref(v), C.byref(ld)))
        rows = ld.value if rows is None else rows
        out = []
        for p in (k.value, v.value):
            flat = torch.as_tensor(_DevView(p, (self.Ls * self.Hs * ld.value * self.d,), "<i2"), device=self.device)
            out.append(flat.view(torch.bfloat16).view(self.Ls, self.Hs, ld.value, self.d)[:, :, :rows])
        return tuple(out)

    def read_offsets(self, slot: int, consumer: int, which: str, rows: int, stream=None):
        """Copies of the stored offsets: bf16 pools -> (ΔK, ΔV) bf16 [Ls, Hs, rows, d];
        fp8 pools -> (codes_K, codes_V uint8 [Ls, Hs, rows, d], scales_K, scales_V fp32 [Ls, Hs, rows])."""
        shape = (self.Ls, self.Hs, rows, self.d)
        if self.offset_format == "fp8":
            k = torch.empty(shape, dtype=torch.uint8, device=self.device)
            v = torch.empty_like(k)
            sk = torch.empty(shape[:3], dtype=torch.float32, device=self.device)
            sv = torch.empty_like(sk)
            L.check(L.lib().kvcomm_anchor_pool_read_offsets(self.handle, slot, consumer, 0 if which == "ph" else 1,
                                                            rows, k.data_ptr(), v.data_ptr(), sk.data_ptr(),
                                                            sv.data_ptr(), _stream_handle(stream)))
            return k, v, sk, sv
        k = torch.empty(shape, dtype=torch.bfloat16, device=self.device)
        v = torch.empty_like(k)
        L.check(L.lib().kvcomm_anchor_pool_read_offsets(self.handle, slot, consumer, 0 if which == "ph" else 1, rows,
                                                        k.data_ptr(), v.data_ptr(), None, None,
                                                        _stream_handle(stream)))
        return k, v

    # -- a1-a3 ---------------------------------------------------------------
    def _match_request(self, query_emb: torch.Tensor, consumer: int, gamma: float, top_k: int, want_dist: bool,
                       ld_w: Optional[int], out: Optional[Match]):
        if query_emb.dim() != 2 or query_emb.shape[1] != self.De or query_emb.dtype != torch.bfloat16 \
                or not query_emb.is_contiguous():
            raise ValueError("query_emb must be a contiguous bf16 [L_phi, D_e] tensor")
        L_phi = query_emb.shape[0]
        if out is not None and out.W is not None and out.W.shape[1] >= L_phi:
            W, wbar, idx, dist = out.W, out.wbar, out.idx, out.dist
            ld_w = W.shape[1]
        else:
            ld_w = ld_w or ((L_phi + 3) // 4 * 4)
            W = torch.zeros(self.capacity, ld_w, dtype=torch.float32, device=self.device)
            wbar = torch.zeros(self.capacity, dtype=torch.float32, device=self.device)
            idx = torch.zeros(L_phi, max(top_k, 1), dtype=torch.int32, device=self.device) if top_k else None
            dist = torch.zeros(self.capacity, ld_w, dtype=torch.float64, device=self.device) if want_dist else None
        info = L.MatchInfo()
        req = L.MatchRequest(self.handle, query_emb.data_ptr(), L_phi, consumer, float(gamma), int(top_k),
                             W.data_ptr(), ld_w, idx.data_ptr() if idx is not None else None, wbar.data_ptr(),
                             dist.data_ptr() if dist is not None else None, C.pointer(info))
        return req, info, (L_phi, W, wbar, idx, dist)

    @staticmethod
    def _match_result(info, bufs) -> Match:
        L_phi, W, wbar, idx, dist = bufs
        cands = list(info.candidates[: info.n_candidates])
        if idx is not None and info.top_k < idx.shape[1] and info.n_candidates > 0:
            idx = idx.view(-1)[: L_phi * info.top_k].view(L_phi, info.top_k)
        return Match(info.verdict, L.REASONS[info.reason], cands, info.top_k, info.entropy, info.threshold,
                     bool(info.verdict_in_tie_band), info.tie_band_count, W, wbar, idx, dist)

    def match(self, query_emb: torch.Tensor, consumer: int = ALL_CONSUMERS, gamma: float = 0.3, top_k: int = 0,
              want_dist: bool = False, ld_w: Optional[int] = None, out: Optional[Match] = None,
              stream=None) -> Match:
        req, info, bufs = self._match_request(query_emb, consumer, gamma, top_k, want_dist, ld_w, out)
        L.check(L.lib().kvcomm_match_anchors(req.pool, req.query_emb, req.L_phi, req.consumer, req.gamma,
                                             req.top_k, req.W, req.ld_w, req.idx, req.wbar, req.dist,
                                             C.byref(info), _stream_handle(stream)))
        return self._match_result(info, bufs)


def match_many(items: Sequence[Tuple["AnchorPool", torch.Tensor]], consumer: int = ALL_CONSUMERS,
               gamma: float = 0.3, top_k: int = 0, outs: Optional[Sequence[Optional[Match]]] = None,
               want_dist: bool = False, stream=None) -> List[Match]:
    """Match several (pool, query) pairs with one device synchronisation
    (kvcomm_match_anchors_batch); each pool at most once."""
    outs = outs or [None] * len(items)
    reqs, infos, bufs = [], [], []
    for (pool, q), o in zip(items, outs):
        r, i, b = pool._match_request(q, consumer, gamma, top_k, want_dist, None, o)
        reqs.append(r)
        infos.append(i)
        bufs.append(b)
    arr = (L.MatchRequest * max(len(reqs), 1))(*reqs)
    L.check(L.lib().kvcomm_match_anchors_batch(arr, len(reqs), _stream_handle(stream)))
    return [AnchorPool._match_result(i, b) for i, b in zip(infos, bufs)]


@dataclass
class Segment:
    """One segment to realign (Eq. 6 placeholder / Eq. 7 prefix + RoPE δ)."""
    pool: AnchorPool
    consumer: int
    kind: int                         # PLACEHOLDER | PREFIX | COPY
    weights: Optional[torch.Tensor]   # PLACEHOLDER: Match.W [capacity, ld_w]; PREFIX: Match.wbar; COPY: None
    candidates: Sequence[int]
    base_k: torch.Tensor              # [Ls, Hs, >=L_seg, d]
    base_v: torch.Tensor
    base_start: int
    target_start: int
    dst_k: torch.Tensor               # [Ls, Hs, N, d]
    dst_v: torch.Tensor
    L_seg: Optional[int] = None
    debug_k: Optional[torch.Tensor] = None   # fp32 [Ls, Hs, L_seg, d]
    debug_v: Optional[torch.Tensor] = None

    def desc(self, keep: list) -> L.RealignDesc:
        L_seg = self.base_k.shape[2] if self.L_seg is None else self.L_seg
        cand = (C.c_int32 * max(len(self.candidates), 1))(*self.candidates)
        keep.append(cand)
        if self.kind != COPY and (self.weights is None or self.weights.dtype != torch.float32
                                  or not self.weights.is_cuda):
            raise ValueError("weights must be fp32 CUDA")
        ld_w = self.weights.shape[1] if self.kind == PLACEHOLDER else 0
        wptr = self.weights.data_ptr() if self.weights is not None else None
        dst_ld, dst_heads = _dst_layout(self.dst_k, "dst_k")
        if _dst_layout(self.dst_v, "dst_v") != (dst_ld, dst_heads):
            raise ValueError("dst_k/dst_v strides differ")
        for t in (self.debug_k, self.debug_v):
            if t is not None and (t.dtype != torch.float32 or not t.is_contiguous()):
                raise ValueError("debug buffers must be contiguous fp32")
        return L.RealignDesc(self.pool.handle, self.consumer, self.kind, wptr, ld_w, cand,
                             len(self.candidates), L_seg, _view(self.base_k, self.base_v, what="base"),
                             self.base_start, self.target_start, self.dst_k.data_ptr(), self.dst_v.data_ptr(),
                             dst_ld, self.debug_k.data_ptr() if self.debug_k is not None else None,
                             self.debug_v.data_ptr() if self.debug_v is not None else None, dst_heads, 0)


@dataclass
class PreparedSegments:
    """Marshalled descriptor array (host work done ahead of the launch)."""
    arr: object
    n: int
    keep: list


def prepare_segments(segs: Sequence[Segment]) -> PreparedSegments:
    keep: list = []
    arr = (L.RealignDesc * max(len(segs), 1))(*[s.desc(keep) for s in segs])
    return PreparedSegments(arr, len(segs), keep)


def realign_prepared(prep: PreparedSegments, stream=None) -> None:
    L.check(L.lib().kvcomm_realign_segments(prep.arr, prep.n, _stream_handle(stream)))


def realign_segments(segs: Sequence[Segment], stream=None) -> None:
    """All segments in one persistent-kernel launch (kvcomm_realign_segments)."""
    realign_prepared(prepare_segments(segs), stream)


def realign_segment(seg: Segment, stream=None) -> None:
    keep: list = []
    d = seg.desc(keep)
    L.check(L.lib().kvcomm_realign_segment(C.byref(d), _stream_handle(stream)))


def concat_prefill_cache(parts: Sequence[Tuple[int, int, Optional[torch.Tensor], Optional[torch.Tensor]]],
                         N_total: int, dst_k: torch.Tensor, dst_v: torch.Tensor, stream=None) -> None:
    """parts: (start, length, src_k, src_v); src None = rows already in place (realigned)."""
    Ls, Hs, _, d = dst_k.shape
    dst_ld = _rows_ld(dst_k, "dst_k")
    refs = (L.SegmentRef * max(len(parts), 1))()
    for i, (start, length, sk, sv) in enumerate(parts):
        refs[i] = L.SegmentRef(int(start), int(length), _view(sk, sv, what="concat src"))
    L.check(L.lib().kvcomm_concat_prefill_cache(refs, len(parts), N_total, Ls, Hs, d, dst_k.data_ptr(),
                                                dst_v.data_ptr(), dst_ld, dst_k.device.index or 0,
                                                _stream_handle(stream)))


@dataclass
class PlanSegment:
    agent: int
    match: int                        # index of the pool in the plan's match list (ignored for COPY)
    kind: int                         # PLACEHOLDER | PREFIX | COPY
    consumer: int
    base_k: torch.Tensor              # [Ls, Hs, L_seg, d]
    base_v: torch.Tensor
    base_start: int
    target_start: int


class Plan:
    """Native executor of Algorithm 1's reuse branch for a fixed multi-agent layout
    (kvcomm_plan_*): per run, one batched match launch and one realign launch with
    the Shareable/NewAnchor branch taken on the device; no host synchronisation
    unless requested."""

    def __init__(self, matches: Sequence[Tuple[AnchorPool, int, float, int]], segments: Sequence[PlanSegment],
                 agents: Sequence[Tuple[int, torch.Tensor, torch.Tensor]], consumer: int = ALL_CONSUMERS):
        """matches: (pool, L_phi, gamma, top_k); agents: (N, dst_k, dst_v)."""
        self.pools = [m[0] for m in matches]
        self._keep = [segments, agents]
        ms = (L.PlanMatch * len(matches))(*[L.PlanMatch(p.handle, int(Lp), consumer, float(g), int(k))
                                            for p, Lp, g, k in matches])
        ss = (L.PlanSegment * max(len(segments), 1))()
        for i, s in enumerate(segments):
            ss[i] = L.PlanSegment(s.agent, s.match, s.kind, s.consumer, _view(s.base_k, s.base_v, what="base"),
                                  s.base_k.shape[2], s.base_start, s.target_start, 0)
        ags = (L.PlanAgent * len(agents))()
        for i, (N, dk, dv) in enumerate(agents):
            ld, heads = _dst_layout(dk, "dst_k")
            if _dst_layout(dv, "dst_v") != (ld, heads):
                raise ValueError("dst_k/dst_v strides differ")
            ags[i] = L.PlanAgent(int(N), heads, dk.data_ptr(), dv.data_ptr(), ld)
        h = C.c_void_p()
        L.check(L.lib().kvcomm_plan_create(ms, len(matches), ss, len(segments), ags, len(agents), C.byref(h)))
        self._h = h
        self.n_matches, self.n_agents = len(matches), len(agents)
        self._events = None

    def _queries(self, queries: Sequence[torch.Tensor]):
        for q in queries:
            if q.dtype != torch.bfloat16 or not q.is_cuda or not q.is_contiguous():
                raise ValueError("queries must be contiguous bf16 CUDA tensors")
        return (C.c_void_p * self.n_matches)(*[q.data_ptr() for q in queries])

    def run(self, queries: Sequence[torch.Tensor], sync: bool = False, stream=None) -> None:
        L.check(L.lib().kvcomm_plan_run(self._h, self._queries(queries), 1 if sync else 0, _stream_handle(stream)))

    def run_begin(self, queries: Sequence[torch.Tensor], stream=None) -> None:
        """First half of a run (candidate filter, table upload, distance kernel); a
        sharded plan needs a cross-rank barrier before run_end."""
        L.check(L.lib().kvcomm_plan_run_begin(self._h, self._queries(queries), _stream_handle(stream)))

    def run_end(self, sync: bool = False, stream=None) -> None:
        L.check(L.lib().kvcomm_plan_run_end(self._h, 1 if sync else 0, _stream_handle(stream)))

    def match_handle(self) -> Tuple[bytes, int]:
        """(64-byte IPC handle, size) of the plan's match buffers, for kvcomm_plan_match_shard."""
        h, n = L.IpcHandle(), C.c_int64()
        L.check(L.lib().kvcomm_plan_match_handle(self._h, C.byref(h), C.byref(n)))
        return C.string_at(C.addressof(h), 64), n.value

    def match_shard(self, rank: int, world: int, handles: Sequence[bytes] = ()) -> None:
        """Shard matching over `world` ranks (handles: every rank's match_handle()[0])."""
        arr = None
        if world > 1:
            if len(handles) != world:
                raise ValueError("one handle per rank")
            arr = (L.IpcHandle * world)()
            for r, hb in enumerate(handles):
                assert len(hb) == 64
                C.memmove(C.addressof(arr[r]), hb, 64)
        L.check(L.lib().kvcomm_plan_match_shard(self._h, int(rank), int(world), arr))

    def set_events(self, before: Optional[torch.cuda.Event], after: Optional[torch.cuda.Event]) -> None:
        """Record `before`/`after` around the realign launch of later runs (kernel timing)."""
        self._events = (before, after)
        for e in (before, after):   # torch creates the CUDA event lazily at its first record
            if e is not None and not e.cuda_event:
                e.record()
        L.check(L.lib().kvcomm_plan_set_events(self._h, before.cuda_event if before is not None else None,
                                               after.cuda_event if after is not None else None))

    def set_realign_stream(self, stream) -> None:
        """Pipelined runs: later runs put their realign kernel on `stream` (a
        torch.cuda.Stream; None restores single-stream runs), so the next run's matching,
        issued on the run stream, overlaps this run's realign (kvcomm_plan_set_realign_stream)."""
        self._rstream = stream
        L.check(L.lib().kvcomm_plan_set_realign_stream(self._h, _stream_handle(stream) if stream is not None else None,
                                                       1 if stream is not None else 0))

    def set_match_events(self, before: Optional[torch.cuda.Event], after: Optional[torch.cuda.Event]) -> None:
        """Record `before`/`after` around the distance kernel (match_dist_kernel) of later runs."""
        self._mevents = (before, after)
        for e in (before, after):
            if e is not None and not e.cuda_event:
                e.record()
        L.check(L.lib().kvcomm_plan_set_match_events(self._h, before.cuda_event if before is not None else None,
                                                     after.cuda_event if after is not None else None))

    def results(self):
        """(list of Match without tensors, list of agent_reused flags) of the last run."""
        infos = (L.MatchInfo * self.n_matches)()
        reused = (C.c_int32 * self.n_agents)()
        L.check(L.lib().kvcomm_plan_results(self._h, infos, reused))
        out = []
        for i in range(self.n_matches):
            W, ldw, wb = self.weights(i)
            inf = infos[i]
            out.append(Match(inf.verdict, L.REASONS[inf.reason], list(inf.candidates[: inf.n_candidates]), inf.top_k,
                             inf.entropy, inf.threshold, bool(inf.verdict_in_tie_band), inf.tie_band_count, W, wb))
        return out, [bool(x) for x in reused]

    def weights(self, match: int):
        W, ld, wb = C.c_void_p(), C.c_int64(), C.c_void_p()
        L.check(L.lib().kvcomm_plan_weights(self._h, match, C.byref(W), C.byref(ld), C.byref(wb)))
        cap = self.pools[match].capacity
        dev = self.pools[match].device
        Wt = torch.as_tensor(_DevView(W.value, (cap * ld.value,), "<f4"), device=dev).view(cap, ld.value)
        wbt = torch.as_tensor(_DevView(wb.value, (cap,), "<f4"), device=dev)
        return Wt, ld.value, wbt

    def destroy(self) -> None:
        if getattr(self, "_h", None) is not None:
            L.check(L.lib().kvcomm_plan_destroy(self._h))
            self._h = None

    def __del__(self):
        try:
            if getattr(self, "_h", None) is not None:
                L.lib().kvcomm_plan_destroy(self._h)
                self._h = None
        except Exception:
            pass
