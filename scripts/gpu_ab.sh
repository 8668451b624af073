#!/bin/bash
# A/B of realign builds on one box: each KVCOMM_LIB probe vs the in-tree library,
# bf16 and fp8 offsets, alternating so drift hits every build alike.  Probe builds:
#   make -C paper_2510_12872_b200/csrc OUT=../lib/probe_X/libkvcomm.so OBJDIR=../lib/probe_X/obj EXTRA=...
# usage: bash scripts/gpu_ab.sh probe_a probe_b ...   (REPS=2, OFFS="bf16 fp8")
mkdir -p gpurun_out
for rep in $(seq ${REPS:-2}); do
  for off in ${OFFS:-bf16 fp8}; do
    BENCH_ARGS="--offsets $off" bash scripts/tune_realign.sh "X=main" \
      $(for p in "$@"; do echo "KVCOMM_LIB=paper_2510_12872_b200/lib/$p/libkvcomm.so"; done)
  done
done
