#!/bin/bash
# Realign-kernel variant sweep on the GPU box: prints achieved GB/s per setting.
run() {
  out=$(env "$@" python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1)
  echo "$* :: $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(f"realign {r["launch_ms"]:.3f} ms {r["achieved"]:.0f} GB/s frac {r["frac"]:.3f} | step {d["ms_per_step"]:.3f} ms value {d["value"]:.0f}")' 2>&1 | tail -1)"
}
for v in ${VARIANTS:-0 2 4 8}; do run KVCOMM_REALIGN_VARIANT=$v; done
