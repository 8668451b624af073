#!/bin/bash
# Run on the GPU box (via gpurun): launch list of one bench step + full ncu captures
# of the realign and match kernels.  Outputs land in gpurun_out/.  Extra arguments are
# passed to bench.py (e.g. --offsets fp8); set TAG to suffix the output names.
set -x
mkdir -p gpurun_out
T=${TAG:-}
ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/launches$T.csv python bench.py --profile --steps 2 --warmup 3 "$@" > gpurun_out/launches$T.log 2>&1
ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:realign_kernel -c 1 -o gpurun_out/prof_realign$T -f python bench.py --profile --steps 1 --warmup 3 "$@" \
    > gpurun_out/prof_realign$T.log 2>&1
if [ -z "$T" ]; then
ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:match_dist_kernel -c 2 -o gpurun_out/prof_match$T -f python bench.py --profile --steps 1 --warmup 3 "$@" \
    > gpurun_out/prof_match$T.log 2>&1
fi
ls -la gpurun_out
