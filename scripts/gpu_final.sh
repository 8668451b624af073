#!/bin/bash
# Final pass of a round on one B200: full ncu captures + launch lists (bf16, fp8), the GPU
# test suite and smoke(), bench lines (bf16, fp8, sustained 300 steps, the reference arm).
mkdir -p gpurun_out
bash scripts/profile_box.sh > gpurun_out/pb.log 2>&1
TAG=_fp8 bash scripts/profile_box.sh --offsets fp8 > gpurun_out/pb8.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gputest.log 2>&1; echo gputest rc=$?
tail -2 gpurun_out/gputest.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
python bench.py --offsets fp8 > gpurun_out/bench_fp8.json 2> gpurun_out/bench_fp8.err; echo bench8 rc=$?
python bench.py --steps 300 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/bench_sustained.json 2>&1; echo sustained rc=$?
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/reference.json 2>&1; echo ref rc=$?
python scripts/config4_bench.py > gpurun_out/config4.json 2>&1; echo c4 rc=$?
