#!/usr/bin/env python
"""Anchor-count x segment-length sweep of the realign kernel (BASELINE.json configs[4],
8B shape, 1/2/4/8 GPUs) plus PAPER.md Table A.5's grid (5-25 anchors x 1K-4K tokens,
P:1456-1469) for a like-for-like comparison with the paper's H100 numbers.

For each point one placeholder segment of T tokens is realigned against m anchors
(all layers/heads, K and V) through kvcomm_realign_segment; device time by CUDA
events: median of 5 batches of 10 back-to-back launches after 5 warm-ups.  Prints JSON lines.
Grid points that do not fit one GPU's HBM are reported as OOM.

Under torchrun with G ranks (one per GPU) every rank holds its layer block (32/G
layers, shard.layer_shard) of the pool, with only its 1/G of the embedding rows
(sharded embeddings) — what makes the 1024-anchor x 8K corner fit at G = 8 —
and realigns it; a point's time is the max over ranks (all-reduce MAX of the CUDA-event
medians), tokens/s counts the whole segment.

  python scripts/sweep.py [--quick]
  python -m torch.distributed.run --nproc-per-node G --master-addr 127.0.0.1 scripts/sweep.py
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


RANK = int(os.environ.get("RANK", "0"))
WORLD = int(os.environ.get("WORLD_SIZE", "1"))


def allreduce_max(v: float) -> float:
    if WORLD == 1:
        return v
    import torch.distributed as dist
    dev = "cpu" if dist.get_backend() == "gloo" else "cuda"
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def layer_block():
    from paper_2510_12872_b200 import shard
    return shard.layer_shard(L, RANK, WORLD)


def build_pool(cap, maxlen, placement="device", offsets="bf16"):
    inv = synth.llama3_inv_freq(D)
    lb, le = layer_block()
    pool = kv.AnchorPool(num_layers=L, num_kv_heads=H, head_dim=D, emb_dim=DE, capacity=cap, max_anchor_len=maxlen,
                         prefix_len=[0], inv_freq=inv, placement=placement, offset_format=offsets,
                         layer_range=(lb, le), emb_shard=(RANK, WORLD) if WORLD > 1 else None)
    g = torch.Generator(device="cuda").manual_seed(0)
    src_k = (torch.randn(le - lb, H, maxlen, D, generator=g, device="cuda") * synth.OFFSET_STD).to(torch.bfloat16)
    src_v = (torch.randn(le - lb, H, maxlen, D, generator=g, device="cuda") * synth.OFFSET_STD).to(torch.bfloat16)
    emb = torch.zeros(maxlen, DE, dtype=torch.bfloat16, device="cuda")
    z = src_k[:, :, :0]
    for _ in range(cap):
        pool.insert(emb, [kv.OffsetGiven(0, src_k, src_v, z, z)])
    del src_k, src_v
    torch.cuda.synchronize()
    return pool


def time_point(pool, m, T, reps=10, offsets="bf16"):
    g = torch.Generator(device="cuda").manual_seed(m * 7 + T)
    Ls = pool.Ls
    base_k = torch.randn(Ls, H, T, D, generator=g, device="cuda").to(torch.bfloat16)
    base_v = torch.randn(Ls, H, T, D, generator=g, device="cuda").to(torch.bfloat16)
    dst_k = torch.empty(Ls, H, T + 512, D, dtype=torch.bfloat16, device="cuda")
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
    ms = allreduce_max(ms)   # the point takes as long as the slowest rank
    off_tok = TOKEN_BYTES if offsets == "bf16" else L * H * (D + 4) * 2  # e4m3 codes + row scale, K+V
    byts = m * T * off_tok + 2 * T * TOKEN_BYTES   # whole segment, all ranks together
    return {"anchors": m, "tokens": T, "gpus": WORLD, "ms": ms, "ms_batches": [round(b, 4) for b in batches],
            "tokens_per_s": T / (ms / 1e3), "GBps": byts / (ms / 1e3) / 1e9, "GBps_per_gpu": byts / WORLD / (ms / 1e3) / 1e9,
            "alg_bytes": byts}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--placement", default="device", choices=["device", "host"],
                    help="host: offset slabs in pinned host memory (f4), a few points only")
    ap.add_argument("--offsets", default="bf16", choices=["bf16", "fp8"])
    ap.add_argument("--grid", default="paper", choices=["paper", "full"],
                    help="full: SURVEY §8(d) config 5, m in {16,64,256,1024} x T in {512..8K}, OOM where it cannot fit")
    args = ap.parse_args()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("KVCOMM_BENCH_SAME_GPU") == "1":   # test-only: every rank on cuda:0
        local = 0
    torch.cuda.set_device(local)
    if WORLD > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo" if os.environ.get("KVCOMM_BENCH_SAME_GPU") == "1" else "nccl")
    free = torch.cuda.mem_get_info()[0]
    emit = (lambda r: print(json.dumps(r), flush=True)) if RANK == 0 else (lambda r: None)
    plans = [  # (capacity, maxlen, points)
        (25, 4096, [(m, T) for m in (5, 10, 15, 20, 25) for T in (1024, 2048, 4096)]),
        (1024, 1024, [(m, T) for m in (16, 64, 256, 1024) for T in (512, 1024)]),
        (256, 4096, [(m, T) for m in (16, 64, 256) for T in (2048, 4096)]),
        (64, 8192, [(m, 8192) for m in (16, 64)]),
    ]
    if args.grid == "full":   # config 5: every (m, T) of the grid; pools sized per row of T
        plans = [(m, T, [(m, T)]) for m in (16, 64, 256, 1024) for T in (512, 1024, 2048, 4096, 8192)]
    if args.quick:
        plans = plans[:1]
    if args.placement == "host":  # offsets stream over the host link: a few small points
        plans = [(16, 1024, [(4, 1024), (16, 1024)])]
    Ls = layer_block()[1] - layer_block()[0]
    for cap, maxlen, pts in plans:
        # per GPU: this rank's layers of the offsets + its embedding rows (all of them at G = 1)
        need = cap * maxlen * (TOKEN_BYTES * Ls / L + DE * 2 / WORLD) * 1.02 + 6e9
        ok = allreduce_max(0.0 if need <= free else 1.0) == 0.0   # every rank must fit
        if not ok:
            for m, T in pts:
                emit({"anchors": m, "tokens": T, "gpus": WORLD, "status": "OOM",
                      "need_GiB_per_gpu": round(need / 2**30, 1)})
            continue
        pool = build_pool(cap, maxlen, args.placement, args.offsets)
        for m, T in pts:
            r = time_point(pool, m, T, offsets=args.offsets)
            r.update(placement=args.placement, offsets=args.offsets)
            if m in TABLE_A5 and T in (1024, 2048, 4096):
                h100 = TABLE_A5[m][(1024, 2048, 4096).index(T)]
                r["paper_h100_softmax_ms"] = h100
                r["speedup_vs_paper"] = h100 / r["ms"]
            emit(r)
        pool.destroy()
        torch.cuda.empty_cache()
    # infeasible corners of the full grid on one GPU (1024 anchors x >= 2K, 256 x 8K)
    if not (args.placement == "host" or args.grid == "full" or WORLD > 1):
        for m, T in [(1024, 2048), (1024, 4096), (1024, 8192), (256, 8192)]:
            emit({"anchors": m, "tokens": T, "status": "OOM", "need_GiB": round(m * T * TOKEN_BYTES / 2**30, 1)})
    if WORLD > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
