#!/usr/bin/env python
"""Anchor-count x segment-length sweep of the realign kernel (BASELINE.json configs[4],
8B shape, 1 GPU) plus PAPER.md Table A.5's grid (5-25 anchors x 1K-4K tokens,
P:1456-1469) for a like-for-like comparison with the paper's H100 numbers.

For each point one placeholder segment of T tokens is realigned against m anchors
(all layers/heads, K and V) through kvcomm_realign_segment; device time by CUDA
events: median of 5 batches of 10 back-to-back launches after 5 warm-ups.  Prints JSON lines.
Grid points that do not fit one GPU's HBM are reported as OOM.

  python scripts/sweep.py [--quick]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch

import synth
import paper_2510_12872_b200 as kv

L, H, D, DE = 32, 8, 128, 4096
TOKEN_BYTES = 2 * L * H * D * 2  # K+V, all layers/heads, bf16: 128 KiB

TABLE_A5 = {5: (0.894, 1.719, 3.552), 10: (1.773, 3.576, 7.128), 15: (2.620, 5.332, 10.766),
            20: (3.933, 7.859, 15.624), 25: (4.435, 9.614, 18.113)}


def build_pool(cap, maxlen, placement="device", offsets="bf16"):
    inv = synth.llama3_inv_freq(D)
    pool = kv.AnchorPool(num_layers=L, num_kv_heads=H, head_dim=D, emb_dim=DE, capacity=cap, max_anchor_len=maxlen,
                         prefix_len=[0], inv_freq=inv, placement=placement, offset_format=offsets)
    g = torch.Generator(device="cuda").manual_seed(0)
    src_k = (torch.randn(L, H, maxlen, D, generator=g, device="cuda") * synth.OFFSET_STD).to(torch.bfloat16)
    src_v = (torch.randn(L, H, maxlen, D, generator=g, device="cuda") * synth.OFFSET_STD).to(torch.bfloat16)
    emb = torch.zeros(maxlen, DE, dtype=torch.bfloat16, device="cuda")
    z = src_k[:, :, :0]
    for _ in range(cap):
        pool.insert(emb, [kv.OffsetGiven(0, src_k, src_v, z, z)])
    del src_k, src_v
    torch.cuda.synchronize()
    return pool


def time_point(pool, m, T, reps=10, offsets="bf16"):
    g = torch.Generator(device="cuda").manual_seed(m * 7 + T)
    base_k = torch.randn(L, H, T, D, generator=g, device="cuda").to(torch.bfloat16)
    base_v = torch.randn(L, H, T, D, generator=g, device="cuda").to(torch.bfloat16)
    dst_k = torch.empty(L, H, T + 512, D, dtype=torch.bfloat16, device="cuda")
    dst_v = torch.empty_like(dst_k)
    ldw = (T + 3) // 4 * 4
    W = torch.full((pool.capacity, ldw), 1.0 / m, dtype=torch.float32, device="cuda")
    seg = kv.Segment(pool, 0, kv.PLACEHOLDER, W, list(range(m)), base_k, base_v, 0, 512, dst_k, dst_v)
    prep = kv.prepare_segments([seg])
    for _ in range(5):
        kv.realign_prepared(prep)
    # median of 5 batches: the first launches over freshly allocated buffers are
    # sometimes 2-10x slower (seen with old and new kernels alike), a warm-up effect
    batches = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps):
            kv.realign_prepared(prep)
        e1.record()
        torch.cuda.synchronize()
        batches.append(e0.elapsed_time(e1) / reps)
    ms = sorted(batches)[len(batches) // 2]
    off_tok = TOKEN_BYTES if offsets == "bf16" else L * H * (D + 4) * 2  # e4m3 codes + row scale, K+V
    byts = m * T * off_tok + 2 * T * TOKEN_BYTES
    return {"anchors": m, "tokens": T, "ms": ms, "ms_batches": [round(b, 4) for b in batches], "tokens_per_s": T / (ms / 1e3), "GBps": byts / (ms / 1e3) / 1e9,
            "alg_bytes": byts}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--placement", default="device", choices=["device", "host"],
                    help="host: offset slabs in pinned host memory (f4), a few points only")
    ap.add_argument("--offsets", default="bf16", choices=["bf16", "fp8"])
    args = ap.parse_args()
    free = torch.cuda.mem_get_info()[0]
    plans = [  # (capacity, maxlen, points)
        (25, 4096, [(m, T) for m in (5, 10, 15, 20, 25) for T in (1024, 2048, 4096)]),
        (1024, 1024, [(m, T) for m in (16, 64, 256, 1024) for T in (512, 1024)]),
        (256, 4096, [(m, T) for m in (16, 64, 256) for T in (2048, 4096)]),
        (64, 8192, [(m, 8192) for m in (16, 64)]),
    ]
    if args.quick:
        plans = plans[:1]
    if args.placement == "host":  # offsets stream over the host link: a few small points
        plans = [(16, 1024, [(4, 1024), (16, 1024)])]
    for cap, maxlen, pts in plans:
        need = cap * maxlen * TOKEN_BYTES * 1.02 + 6e9
        if need > free:
            for m, T in pts:
                print(json.dumps({"anchors": m, "tokens": T, "status": "OOM",
                                  "need_GiB": round(cap * maxlen * TOKEN_BYTES / 2**30, 1)}))
            continue
        pool = build_pool(cap, maxlen, args.placement, args.offsets)
        for m, T in pts:
            r = time_point(pool, m, T, offsets=args.offsets)
            r.update(placement=args.placement, offsets=args.offsets)
            if m in TABLE_A5 and T in (1024, 2048, 4096):
                h100 = TABLE_A5[m][(1024, 2048, 4096).index(T)]
                r["paper_h100_softmax_ms"] = h100
                r["speedup_vs_paper"] = h100 / r["ms"]
            print(json.dumps(r), flush=True)
        pool.destroy()
        torch.cuda.empty_cache()
    # infeasible corners of the full grid on one GPU (1024 anchors x >= 2K, 256 x 8K)
    if args.placement == "host":
        return
    for m, T in [(1024, 2048), (1024, 4096), (1024, 8192), (256, 8192)]:
        print(json.dumps({"anchors": m, "tokens": T, "status": "OOM",
                          "need_GiB": round(m * T * TOKEN_BYTES / 2**30, 1)}))


if __name__ == "__main__":
    main()
