#!/bin/bash
# Run on the GPU box (via gpurun): launch list of one bench step + full ncu captures
# of the realign and match kernels.  Outputs land in gpurun_out/.
set -x
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/launches.csv python bench.py --profile --steps 2 --warmup 3 > gpurun_out/launches.log 2>&1
ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:realign_kernel -c 1 -o gpurun_out/prof_realign -f python bench.py --profile --steps 1 --warmup 3 \
    > gpurun_out/prof_realign.log 2>&1
ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:match_dist_kernel -c 2 -o gpurun_out/prof_match -f python bench.py --profile --steps 1 --warmup 3 \
    > gpurun_out/prof_match.log 2>&1
ls -la gpurun_out
