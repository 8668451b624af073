"""The C-ABI library loads on a CPU-only box and exports every symbol include/kvcomm.h
declares; the ctypes mirror matches the C layout; host-side contract checks that
return before any device work behave as documented.  (-m "not gpu")"""
import ctypes as C
import os
import subprocess
import tempfile

import pytest

from paper_2510_12872_b200 import _lib as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    lib = L.load()
    names = L.header_symbols()
    assert len(names) >= 17
    for n in names:
        assert hasattr(lib, n), n
    assert lib.kvcomm_version() == 1
    out = subprocess.run(["nm", "-D", "--defined-only", L.LIB_PATH], capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    assert set(names) <= exported
    # nothing but the C ABI leaks out of the shared object
    assert all(e.startswith("kvcomm_") or e.startswith("_") for e in exported), exported


def test_ctypes_layout_matches_c_header():
    prog = r"""
#include <stdio.h>
#include <stddef.h>
#include "kvcomm.h"
#define S(T) printf(#T " %zu\n", sizeof(T));
#define O(T, f) printf(#T "." #f " %zu\n", offsetof(T, f));
int main(void) {
  S(kvcomm_pool_config) S(kvcomm_kv_view) S(kvcomm_offset_desc) S(kvcomm_slot_info)
  S(kvcomm_match_info) S(kvcomm_realign_desc) S(kvcomm_segment_ref) S(kvcomm_match_request)
  S(kvcomm_plan_match) S(kvcomm_plan_segment) S(kvcomm_plan_agent) S(kvcomm_ipc_handle)
  O(kvcomm_plan_segment, base) O(kvcomm_plan_segment, target_start) O(kvcomm_plan_agent, dst_ld)
  O(kvcomm_pool_config, prefix_len) O(kvcomm_pool_config, inv_freq)
  O(kvcomm_match_info, entropy) O(kvcomm_match_info, tie_band_count)
  O(kvcomm_realign_desc, base) O(kvcomm_realign_desc, dst_k) O(kvcomm_realign_desc, debug_delta_v)
  O(kvcomm_offset_desc, pf_base) O(kvcomm_segment_ref, src)
  return 0;
}
"""
    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "l.c")
        exe = os.path.join(d, "l")
        open(src, "w").write(prog)
        subprocess.run(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), src, "-o", exe], check=True)
        lines = subprocess.run([exe], capture_output=True, text=True, check=True).stdout.split("\n")
    got = dict(l.split() for l in lines if l.strip())
    py = {"kvcomm_pool_config": L.PoolConfig, "kvcomm_kv_view": L.KVView, "kvcomm_offset_desc": L.OffsetDesc,
          "kvcomm_slot_info": L.SlotInfo, "kvcomm_match_info": L.MatchInfo, "kvcomm_realign_desc": L.RealignDesc,
          "kvcomm_segment_ref": L.SegmentRef, "kvcomm_match_request": L.MatchRequest,
          "kvcomm_plan_match": L.PlanMatch, "kvcomm_plan_segment": L.PlanSegment, "kvcomm_plan_agent": L.PlanAgent,
          "kvcomm_ipc_handle": L.IpcHandle}
    for k, T in py.items():
        assert int(got[k]) == C.sizeof(T), k
    for key, v in got.items():
        if "." in key:
            t, f = key.split(".")
            assert getattr(py[t], {"debug_delta_v": "debug_delta_v"}.get(f, f)).offset == int(v), key


def test_status_strings_and_error_message():
    lib = L.load()
    assert lib.kvcomm_status_string(0) == b"OK"
    assert lib.kvcomm_status_string(5) == b"POSITION_GAP"
    assert lib.kvcomm_status_string(6) == b"POSITION_OVERLAP"


def test_concat_ledger_errors_before_any_device_work():
    lib = L.load()
    refs = (L.SegmentRef * 2)(L.SegmentRef(0, 3, L.KVView()), L.SegmentRef(4, 6, L.KVView()))
    st = lib.kvcomm_concat_prefill_cache(refs, 2, 10, 2, 2, 16, None, None, 10, 0, None)
    assert L.STATUS_NAMES[st] == "POSITION_GAP"
    assert b"gap at position 3" in lib.kvcomm_last_error_message()
    refs = (L.SegmentRef * 2)(L.SegmentRef(0, 4, L.KVView()), L.SegmentRef(3, 7, L.KVView()))
    st = lib.kvcomm_concat_prefill_cache(refs, 2, 10, 2, 2, 16, None, None, 10, 0, None)
    assert L.STATUS_NAMES[st] == "POSITION_OVERLAP"
    refs = (L.SegmentRef * 1)(L.SegmentRef(0, 4, L.KVView()))
    st = lib.kvcomm_concat_prefill_cache(refs, 1, 10, 2, 2, 16, None, None, 10, 0, None)
    assert L.STATUS_NAMES[st] == "POSITION_GAP"


def test_pool_create_rejects_bad_geometry_before_touching_a_device():
    lib = L.load()
    pl = (C.c_int32 * 1)(4)
    inv = (C.c_double * 8)(*([1.0] * 8))
    h = C.c_void_p()
    for bad in [dict(head_dim=17), dict(head_dim=0), dict(emb_dim=12), dict(capacity=0),
                dict(capacity=2048), dict(layer_end=3), dict(num_consumers=0),
                dict(emb_shard_world=9), dict(emb_shard_rank=2, emb_shard_world=2),
                dict(emb_shard_rank=-1, emb_shard_world=2), dict(emb_shard_rank=1)]:
        cfg = dict(device=0, num_layers=2, layer_begin=0, layer_end=2, num_kv_heads=2, head_begin=0,
                   head_end=2, head_dim=16, emb_dim=32, capacity=4, max_anchor_len=48, num_consumers=1)
        cfg.update(bad)
        c = L.PoolConfig(**cfg, prefix_len=pl, inv_freq=inv)
        st = lib.kvcomm_anchor_pool_create(C.byref(c), C.byref(h))
        assert L.STATUS_NAMES[st] == "INVALID_ARGUMENT", bad
    assert lib.kvcomm_anchor_pool_create(None, C.byref(h)) == 1


def test_binding_fails_loudly_without_library(tmp_path):
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        L.load(str(tmp_path / "missing.so"))


def test_ipc_calls_validate_arguments_before_any_device_work():
    """The fused-gather handle calls reject null/size errors with a status (no crash)."""
    lib = L.load()
    ptr = C.c_void_p()
    h = L.IpcHandle()
    assert lib.kvcomm_ipc_alloc(0, 0, C.byref(ptr), C.byref(h)) == 1            # INVALID_ARGUMENT: size
    assert lib.kvcomm_ipc_alloc(0, 64, None, C.byref(h)) == 1                   # null out pointer
    assert lib.kvcomm_ipc_open(0, None, C.byref(ptr)) == 1
    assert lib.kvcomm_ipc_free(None) == 0 and lib.kvcomm_ipc_close(None) == 0   # no-ops


def test_pool_checkpoint_errors_before_any_device_work(tmp_path):
    """kvcomm_anchor_pool_load: a missing file, a foreign file and a wrong version are
    IO errors raised before any CUDA call; save/load validate their arguments."""
    lib = L.load()
    out = C.c_void_p()
    missing = str(tmp_path / "none.kvc").encode()
    assert lib.kvcomm_anchor_pool_load(missing, 0, C.byref(out)) == L.STATUS_NAMES.index("IO")
    assert b"cannot open" in lib.kvcomm_last_error_message()
    junk = tmp_path / "junk.kvc"
    junk.write_bytes(b"not a checkpoint at all")
    assert lib.kvcomm_anchor_pool_load(str(junk).encode(), 0, C.byref(out)) == L.STATUS_NAMES.index("IO")
    assert b"not a pool checkpoint" in lib.kvcomm_last_error_message()
    old = tmp_path / "old.kvc"
    old.write_bytes(b"KVCPOOL1" + (7).to_bytes(4, "little"))
    assert lib.kvcomm_anchor_pool_load(str(old).encode(), 0, C.byref(out)) == L.STATUS_NAMES.index("IO")
    assert b"version" in lib.kvcomm_last_error_message()
    assert out.value is None
    assert lib.kvcomm_anchor_pool_load(None, 0, C.byref(out)) == L.STATUS_NAMES.index("INVALID_ARGUMENT")
    assert lib.kvcomm_anchor_pool_save(None, b"x", None) == L.STATUS_NAMES.index("INVALID_ARGUMENT")
    assert lib.kvcomm_status_string(L.STATUS_NAMES.index("IO")) == b"IO"
