"""ctypes mirror of include/kvcomm.h and the loader of lib/libkvcomm.so.

There is no fallback: if the shared library is missing the import fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os
import re

HERE = os.path.dirname(os.path.abspath(__file__))
# KVCOMM_LIB: probe builds of the same library (scripts/tune_realign.sh); default in-tree
LIB_PATH = os.environ.get("KVCOMM_LIB") or os.path.join(HERE, "lib", "libkvcomm.so")
HEADER_PATH = os.path.join(os.path.dirname(HERE), "include", "kvcomm.h")

MAX_CAPACITY = 1024
MAX_CONSUMERS = 64
MAX_TOPK = 32
ALL_CONSUMERS = -1

OK = 0
STATUS_NAMES = ["OK", "INVALID_ARGUMENT", "SHAPE_MISMATCH", "NO_CANDIDATES", "MISSING_OFFSET",
                "POSITION_GAP", "POSITION_OVERLAP", "NOT_FOUND", "OUT_OF_MEMORY", "CUDA", "NCCL", "IO"]
SHAREABLE, NEW_ANCHOR = 0, 1
REASONS = ["OK", "EMPTY_POOL", "TOO_LONG", "NO_CANDIDATES", "HIGH_ENTROPY", "SHARD_MISMATCH"]
PLACEHOLDER, PREFIX, COPY = 0, 1, 2
OFFSET_GIVEN, OFFSET_MEASURE = 0, 1
SCALAR_FROBENIUS, SCALAR_MEAN_L2 = 0, 1
SIM_L2, SIM_COSINE = 0, 1
OFFSET_BF16, OFFSET_FP8_E4M3 = 0, 1
PLACE_DEVICE, PLACE_HOST = 0, 1
ROPE_HALF, ROPE_INTERLEAVED = 0, 1


class PoolConfig(C.Structure):
    _fields_ = [("device", C.c_int32), ("num_layers", C.c_int32), ("layer_begin", C.c_int32),
                ("layer_end", C.c_int32), ("num_kv_heads", C.c_int32), ("head_begin", C.c_int32),
                ("head_end", C.c_int32), ("head_dim", C.c_int32), ("emb_dim", C.c_int32),
                ("capacity", C.c_int32), ("max_anchor_len", C.c_int32), ("num_consumers", C.c_int32),
                ("scalar_distance", C.c_int32), ("similarity", C.c_int32),
                ("offset_format", C.c_int32), ("placement", C.c_int32), ("rope_layout", C.c_int32),
                ("emb_shard_rank", C.c_int16), ("emb_shard_world", C.c_int16), ("prefix_len", C.POINTER(C.c_int32)), ("inv_freq", C.POINTER(C.c_double))]


class KVView(C.Structure):
    _fields_ = [("k", C.c_void_p), ("v", C.c_void_p), ("ld", C.c_int64), ("start", C.c_int32),
                ("_pad", C.c_int32)]


class OffsetDesc(C.Structure):
    _fields_ = [("consumer", C.c_int32), ("mode", C.c_int32), ("ph_delta", KVView), ("pf_delta", KVView),
                ("ph_real", KVView), ("ph_base", KVView), ("pf_real", KVView), ("pf_base", KVView)]


class SlotInfo(C.Structure):
    _fields_ = [("occupied", C.c_int32), ("length", C.c_int32), ("access_count", C.c_int64),
                ("insertion_index", C.c_int64), ("ph_present_mask", C.c_uint64),
                ("pf_present_mask", C.c_uint64)]


class MatchInfo(C.Structure):
    _fields_ = [("verdict", C.c_int32), ("reason", C.c_int32), ("n_candidates", C.c_int32),
                ("top_k", C.c_int32), ("candidates", C.c_int32 * MAX_CAPACITY), ("entropy", C.c_double),
                ("threshold", C.c_double), ("verdict_in_tie_band", C.c_int32), ("tie_band_count", C.c_int32)]


class RealignDesc(C.Structure):
    _fields_ = [("pool", C.c_void_p), ("consumer", C.c_int32), ("kind", C.c_int32), ("weights", C.c_void_p),
                ("ld_w", C.c_int64), ("candidates", C.POINTER(C.c_int32)), ("n_candidates", C.c_int32),
                ("L_seg", C.c_int32), ("base", KVView), ("base_start", C.c_int32), ("target_start", C.c_int32),
                ("dst_k", C.c_void_p), ("dst_v", C.c_void_p), ("dst_ld", C.c_int64),
                ("debug_delta_k", C.c_void_p), ("debug_delta_v", C.c_void_p), ("dst_heads", C.c_int32),
                ("_pad", C.c_int32)]


class MatchRequest(C.Structure):
    _fields_ = [("pool", C.c_void_p), ("query_emb", C.c_void_p), ("L_phi", C.c_int32), ("consumer", C.c_int32),
                ("gamma", C.c_float), ("top_k", C.c_int32), ("W", C.c_void_p), ("ld_w", C.c_int64),
                ("idx", C.c_void_p), ("wbar", C.c_void_p), ("dist", C.c_void_p), ("info", C.POINTER(MatchInfo))]


class PlanMatch(C.Structure):
    _fields_ = [("pool", C.c_void_p), ("L_phi", C.c_int32), ("consumer", C.c_int32), ("gamma", C.c_float),
                ("top_k", C.c_int32)]


class PlanSegment(C.Structure):
    _fields_ = [("agent", C.c_int32), ("match", C.c_int32), ("kind", C.c_int32), ("consumer", C.c_int32),
                ("base", KVView), ("L_seg", C.c_int32), ("base_start", C.c_int32), ("target_start", C.c_int32),
                ("_pad", C.c_int32)]


class PlanAgent(C.Structure):
    _fields_ = [("N", C.c_int32), ("dst_heads", C.c_int32), ("dst_k", C.c_void_p), ("dst_v", C.c_void_p),
                ("dst_ld", C.c_int64)]


class IpcHandle(C.Structure):
    _fields_ = [("bytes", C.c_char * 64)]


class SegmentRef(C.Structure):
    _fields_ = [("start", C.c_int32), ("length", C.c_int32), ("src", KVView)]


_SIGS = {
    "kvcomm_status_string": (C.c_char_p, [C.c_int]),
    "kvcomm_last_error_message": (C.c_char_p, []),
    "kvcomm_version": (C.c_int32, []),
    "kvcomm_kernel_launch_count": (C.c_int64, []),
    "kvcomm_anchor_pool_create": (C.c_int, [C.POINTER(PoolConfig), C.POINTER(C.c_void_p)]),
    "kvcomm_anchor_pool_destroy": (C.c_int, [C.c_void_p]),
    "kvcomm_anchor_pool_bytes": (C.c_int, [C.c_void_p, C.POINTER(C.c_int64)]),
    "kvcomm_anchor_pool_insert": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.POINTER(OffsetDesc), C.c_int32,
                                            C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "kvcomm_anchor_pool_set_offsets": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(OffsetDesc), C.c_int32,
                                                 C.c_void_p]),
    "kvcomm_anchor_pool_evict": (C.c_int, [C.c_void_p, C.c_int32]),
    "kvcomm_anchor_pool_record_access": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32), C.c_int32]),
    "kvcomm_anchor_pool_slot_info": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(SlotInfo)]),
    "kvcomm_anchor_pool_offset_view": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                                 C.POINTER(C.c_void_p), C.POINTER(C.c_void_p),
                                                 C.POINTER(C.c_int64)]),
    "kvcomm_anchor_pool_read_offsets": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                                  C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
    "kvcomm_match_anchors": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_float, C.c_int32,
                                       C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p,
                                       C.POINTER(MatchInfo), C.c_void_p]),
    "kvcomm_match_anchors_batch": (C.c_int, [C.POINTER(MatchRequest), C.c_int32, C.c_void_p]),
    "kvcomm_realign_segment": (C.c_int, [C.POINTER(RealignDesc), C.c_void_p]),
    "kvcomm_realign_segments": (C.c_int, [C.POINTER(RealignDesc), C.c_int32, C.c_void_p]),
    "kvcomm_concat_prefill_cache": (C.c_int, [C.POINTER(SegmentRef), C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                              C.c_int32, C.c_void_p, C.c_void_p, C.c_int64, C.c_int32,
                                              C.c_void_p]),
    "kvcomm_plan_create": (C.c_int, [C.POINTER(PlanMatch), C.c_int32, C.POINTER(PlanSegment), C.c_int32,
                                     C.POINTER(PlanAgent), C.c_int32, C.POINTER(C.c_void_p)]),
    "kvcomm_plan_destroy": (C.c_int, [C.c_void_p]),
    "kvcomm_plan_run": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p), C.c_int32, C.c_void_p]),
    "kvcomm_plan_results": (C.c_int, [C.c_void_p, C.POINTER(MatchInfo), C.POINTER(C.c_int32)]),
    "kvcomm_plan_set_events": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "kvcomm_plan_set_match_events": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "kvcomm_plan_set_realign_stream": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32]),
    "kvcomm_plan_weights": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(C.c_void_p), C.POINTER(C.c_int64),
                                      C.POINTER(C.c_void_p)]),
    "kvcomm_plan_match_handle": (C.c_int, [C.c_void_p, C.POINTER(IpcHandle), C.POINTER(C.c_int64)]),
    "kvcomm_plan_match_shard": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.POINTER(IpcHandle)]),
    "kvcomm_plan_run_begin": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p), C.c_void_p]),
    "kvcomm_plan_run_end": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p]),
    "kvcomm_anchor_pool_save": (C.c_int, [C.c_void_p, C.c_char_p, C.c_void_p]),
    "kvcomm_anchor_pool_load": (C.c_int, [C.c_char_p, C.c_int32, C.POINTER(C.c_void_p)]),
    "kvcomm_anchor_pool_get_config": (C.c_int, [C.c_void_p, C.POINTER(PoolConfig), C.POINTER(C.c_int32),
                                                C.POINTER(C.c_double)]),
    "kvcomm_ipc_alloc": (C.c_int, [C.c_int32, C.c_int64, C.POINTER(C.c_void_p), C.POINTER(IpcHandle)]),
    "kvcomm_ipc_free": (C.c_int, [C.c_void_p]),
    "kvcomm_ipc_open": (C.c_int, [C.c_int32, C.POINTER(IpcHandle), C.POINTER(C.c_void_p)]),
    "kvcomm_ipc_close": (C.c_int, [C.c_void_p]),
}


def header_symbols(path: str = HEADER_PATH):
    """Names of every KVCOMM_API function declared in include/kvcomm.h."""
    text = open(path).read()
    return re.findall(r"KVCOMM_API\s+[\w\s\*]+?\b(kvcomm_\w+)\s*\(", text)


def load(path: str = LIB_PATH) -> C.CDLL:
    if not os.path.exists(path):
        raise RuntimeError(f"libkvcomm.so not found at {path}: build it with "
                           "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback exists)")
    lib = C.CDLL(path)
    probe = os.environ.get("KVCOMM_LIB") is not None  # probe builds of older revisions may lack symbols
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name, None)
        if fn is None and probe:
            continue
        if fn is None:
            raise RuntimeError(f"{path} does not export {name}: stale build")
        fn.restype = res
        fn.argtypes = args
    return lib


class KVCommError(RuntimeError):
    def __init__(self, status: int, message: str):
        name = STATUS_NAMES[status] if 0 <= status < len(STATUS_NAMES) else str(status)
        super().__init__(f"{name}: {message}")
        self.status = status
        self.status_name = name


_LIB = None


def lib() -> C.CDLL:
    global _LIB
    if _LIB is None:
        _LIB = load()
    return _LIB


def check(status: int) -> None:
    if status != OK:
        raise KVCommError(status, lib().kvcomm_last_error_message().decode())
