#!/bin/bash
# Full ncu capture of one realign launch (and optionally match_dist) of the bench step.
# usage: TAG=_fp8 bash scripts/ncu_realign.sh --offsets fp8     (outputs in gpurun_out/)
mkdir -p gpurun_out
T=${TAG:-}
ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:realign_kernel -c 1 -o gpurun_out/prof_realign$T -f python bench.py --profile --steps 1 --warmup 3 "$@" \
    > gpurun_out/prof_realign$T.log 2>&1
if [ -n "$MATCH" ]; then
ncu --set full --clock-control none --import-source on --profile-from-start off \
    -k regex:match_dist_kernel -c 1 -o gpurun_out/prof_match$T -f python bench.py --profile --steps 1 --warmup 3 "$@" \
    > gpurun_out/prof_match$T.log 2>&1
fi
