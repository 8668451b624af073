#!/usr/bin/env python
"""Format scripts/sweep.py JSON lines as the markdown table kept under profiles/.

  python scripts/sweep_md.py <tag> < sweep.jsonl > profiles/<tag>_sweep.md
"""
import json
import sys

tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
rows = [json.loads(l) for l in sys.stdin if l.strip()]
print(f"# {tag} realign sweep on 1 B200 (8B shape, one consumer, K+V all layers/heads)\n")
print("`python scripts/sweep.py` — CUDA events, median of 5 batches of 10 back-to-back `kvcomm_realign_segment` launches; "
      "bytes = (m+2) x T x 128 KiB.\n")
print("| anchors m | tokens T | ms | tokens/s | GB/s | PAPER Table A.5 H100 'softmax' ms | B200 speedup |")
print("|---:|---:|---:|---:|---:|---:|---:|")
for r in rows:
    if r.get("status") == "OOM":
        print(f"| {r['anchors']} | {r['tokens']} | OOM ({r.get('need_GiB', r.get('need_GiB_per_gpu', 0)):.0f} GiB of offsets{' per GPU' if 'need_GiB_per_gpu' in r else ''}) | | | | |")
        continue
    p = r.get("paper_h100_softmax_ms")
    sp = r.get("speedup_vs_paper")
    print(f"| {r['anchors']} | {r['tokens']} | {r['ms']:.3f} | {r['tokens_per_s']:.3g} | {r['GBps']:.0f} | "
          f"{p if p else ''} | {f'{sp:.1f}x' if sp else ''} |")
