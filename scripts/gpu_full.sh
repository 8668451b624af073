#!/bin/bash
# Round-end style GPU pass: smoke, pytest -m gpu, bench (bf16 + fp8), launch lists and
# full ncu captures (bf16 + fp8).  Outputs under gpurun_out/.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo gputest rc=$?
tail -3 gpurun_out/gputest.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
timeout 600 python bench.py --offsets fp8 > gpurun_out/bench_fp8.json 2> gpurun_out/bench_fp8.err; echo bench8 rc=$?
[ -n "$NO_PROFILE" ] || { bash scripts/profile_box.sh > gpurun_out/profile_box.log 2>&1; TAG=_fp8 bash scripts/profile_box.sh --offsets fp8 > gpurun_out/profile_box_fp8.log 2>&1; }
ls gpurun_out
