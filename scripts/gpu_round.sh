#!/bin/bash
# One GPU pass: smoke, pytest -m gpu, bench (bf16 + fp8).  Outputs under gpurun_out/.
set -x
mkdir -p gpurun_out
nproc; lscpu | grep 'Model name'
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo gputest rc=$?
tail -5 gpurun_out/gputest.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
timeout 600 python bench.py --offsets fp8 > gpurun_out/bench_fp8.json 2> gpurun_out/bench_fp8.err; echo bench8 rc=$?
cat gpurun_out/bench.json gpurun_out/bench_fp8.json
