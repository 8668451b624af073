#!/bin/bash
# compute-sanitizer over smoke() and a few small parity tests that reach the other
# realign paths (fp8 blocks, weight chunks of a large pool, host-resident pool,
# interleaved RoPE, measured inserts), 12 random configurations of the fuzz sweep, and
# the pool checkpoint + plan tests (split runs), the request plan (grouped / gated) and
# the opt-in TMA match kernel.
# Run on the GPU box; prints one summary line per (tool, target).
T1='python -c "import __graft_entry__ as g; g.smoke()"'
T2='python -m pytest -q -x -m gpu tests/test_gpu_parity.py -k "test_weight_block_fallback or test_fp8_offsets_codes_and_realign or test_host_resident_pool or test_interleaved_rope_layout or test_measure_insert" -p no:cacheprovider'
T3='env KVCOMM_FUZZ_CASES=12 python -m pytest -q -x -m gpu tests/test_gpu_fuzz.py -p no:cacheprovider'
T4='python -m pytest -q -x -m gpu tests/test_gpu_checkpoint.py tests/test_gpu_plan.py -p no:cacheprovider'
# round 2: the bench's grouped/gated plan launch at small sizes, and the opt-in TMA match kernel
T5='python -m pytest -q -x -m gpu tests/test_gpu_request_parity.py -p no:cacheprovider'
T6='env KVCOMM_MATCH_TMA=1 python -c "import __graft_entry__ as g; g.smoke()"'
# round 2 (later): the row-ring match kernel; the plan tests include pipelined runs (realign stream)
T7='env KVCOMM_MATCH_TMA=2 python -c "import __graft_entry__ as g; g.smoke()"'
for tool in memcheck racecheck synccheck initcheck; do
  for t in "$T1" "$T2" "$T3" "$T4" "$T5" "$T6" "$T7"; do
    out=$(eval compute-sanitizer --tool $tool --error-exitcode 9 $t 2>&1)
    rc=$?
    echo "== $tool rc=$rc :: ${t:0:60} :: $(echo "$out" | grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|passed|failed' | tr '\n' ' ')"
  done
done
