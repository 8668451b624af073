#!/usr/bin/env python
"""Step a0 (insert path, Algorithm 1's fallback branch P:786-796) on one B200 at the
config-2 shape: one anchor of the user_question pool (1024 tokens, 5 consumers,
32-token prefixes), Llama-3-8B shape.

  measure: offsets measured on device from real/base K,V (kvcomm_anchor_pool_insert
           with OFFSET_MEASURE: ΔK = R_{-Δs} K_real - K_base, ΔV = V_real - V_base)
  given:   precomputed offsets copied into the slab
Prints one JSON line per mode: device time per insert (CUDA events, median of 5
batches of 10 inserts into a full pool, LFU eviction included) and algorithmic GB/s
(measure: 4 reads + 2 writes per element; given: 2 reads + 2 writes... per plane).

  python scripts/insert_bench.py [--offsets bf16|fp8]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch

import synth

L, H, D, DE, T, P, C, CAP = 32, 8, 128, 4096, 1024, 32, 5, 20


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--offsets", default="bf16", choices=["bf16", "fp8"])
    args = ap.parse_args()
    import paper_2510_12872_b200 as kv
    inv = synth.llama3_inv_freq(D)
    pool = kv.AnchorPool(num_layers=L, num_kv_heads=H, head_dim=D, emb_dim=DE, capacity=CAP, max_anchor_len=T,
                         prefix_len=[P] * C, inv_freq=inv, offset_format=args.offsets)
    g = torch.Generator(device="cuda").manual_seed(0)
    r = lambda n: torch.randn(L, H, n, D, generator=g, device="cuda").to(torch.bfloat16)
    emb = torch.randn(T, DE, generator=g, device="cuda").to(torch.bfloat16)
    real = [(r(T), r(T), r(P), r(P)) for _ in range(C)]
    base = (r(T), r(T), r(P), r(P))
    meas = [kv.OffsetMeasure(c, ph_real=(real[c][0], real[c][1], 480 + 64 * c), ph_base=(base[0], base[1], 0),
                             pf_real=(real[c][2], real[c][3], 1504 + 64 * c), pf_base=(base[2], base[3], 480))
            for c in range(C)]
    given = [kv.OffsetGiven(c, real[c][0], real[c][1], real[c][2], real[c][3]) for c in range(C)]
    row = H * D * 2 * L  # one token of one plane, all layers/heads
    elems_rows = C * (T + P) * 2  # (consumer, token, plane) rows written
    out_row = row if args.offsets == "bf16" else L * H * (D + 4)
    for mode, offs, reads in (("measure", meas, 2), ("given", given, 1)):
        for _ in range(CAP + 3):  # fill the pool, then every insert evicts (LFU)
            pool.insert(emb, offs)
        batches = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(10):
                pool.insert(emb, offs)
            e1.record()
            torch.cuda.synchronize()
            batches.append(e0.elapsed_time(e1) / 10)
        ms = sorted(batches)[2]
        # measure: real + base rows read per (consumer, plane) row (base re-read per consumer),
        # one offset row written; given: one row read, one written; + the embedding copy
        alg = elems_rows * (reads * row + out_row) + 2 * T * DE * 2
        print(json.dumps({"step": "a0 insert", "mode": mode, "offsets": args.offsets, "ms_per_insert": ms,
                          "alg_bytes": alg, "GBps": alg / (ms / 1e3) / 1e9,
                          "shape": f"8B shape, {T}-token anchor, {C} consumers x ({T} placeholder + {P} prefix) rows"}))
    pool.destroy()


if __name__ == "__main__":
    main()
