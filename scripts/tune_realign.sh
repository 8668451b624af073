#!/bin/bash
# Realign-kernel variant sweep on the GPU box: prints achieved GB/s per setting.
# usage: bash scripts/tune_realign.sh "ENV=.. ENV2=.." "ENV=.." ...   (extra bench args in BENCH_ARGS)
run() {
  out=$(env $1 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline $BENCH_ARGS 2>&1 | tail -1)
  echo "$1 $BENCH_ARGS :: $(echo "$out" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; m=r.get("match") or {}; print(f"realign {r["launch_ms"]:.3f} ms {r["achieved"]:.0f} GB/s frac {r["frac"]:.3f} | match {m.get("launch_ms",0)*1e3:.1f} us {m.get("achieved",0):.0f} GB/s | step {d["ms_per_step"]:.3f} ms value {d["value"]:.0f}")' 2>&1 | tail -1)"
}
for cfg in "$@"; do run "$cfg"; done
