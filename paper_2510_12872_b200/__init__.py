"""B200-native KVComm anchor-realignment hot path (arXiv 2510.12872).

The compute lives in lib/libkvcomm.so (hand-written sm_100a CUDA behind the C ABI
in include/kvcomm.h); `kvcomm` is the thin ctypes binding.  Importing this package
fails loudly if the library has not been built.
"""
from .kvcomm import (ALL_CONSUMERS, COPY, NEW_ANCHOR, PLACEHOLDER, PREFIX, SHAREABLE, AnchorPool,  # noqa
                     KVCommError, Match, OffsetGiven, OffsetMeasure, Segment, concat_prefill_cache,
                     kernel_launch_count, match_many, prepare_segments, realign_prepared, realign_segment,
                     realign_segments, Plan, PlanSegment)
from ._lib import LIB_PATH, lib as _load_lib  # noqa: F401

_load_lib()  # load now: no silent fallback path exists
