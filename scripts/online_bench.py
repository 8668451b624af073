#!/usr/bin/env python
"""SURVEY §8(f) f1 at the config-2 shape: Algorithm 1's online loop (OnlinePool.step)
over a clustered request stream for one user_question-like pool (1,024-token samples,
5 consumers with 32-token prefixes, capacity 20, γ = 0.3), Llama-3-8B shape.

Reuse steps match + realign all consumers (Eq. 5-7); fallback steps copy the dense
caches and insert the sample with device-measured offsets, LFU-pruned.
The dense "prefill" caches are fixed synthetic tensors (the model is out of scope),
so only the pool/kernel work is timed.  Prints one JSON line: reuse rate and device
time per reuse and per fallback step (CUDA events around each step, host
synchronisation of the match verdict included).

  python scripts/online_bench.py [--requests 60] [--p-swap 0.15]
"""
import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch

import synth

L, H, D, DE, T, P, C, CAP, V = 32, 8, 128, 4096, 1024, 32, 5, 20, 128256


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--requests", type=int, default=60)
    ap.add_argument("--p-swap", type=float, default=0.15)
    ap.add_argument("--clusters", type=int, default=4)
    ap.add_argument("--gamma", type=float, default=0.3)
    ap.add_argument("--capacity", type=int, default=CAP, help="pool capacity V (Table 6 P:507-515 sweeps 5-25)")
    ap.add_argument("--warm", type=int, default=None,
                    help="samples of the stream's clusters inserted (measured offsets) before the stream "
                         "(an empty pool accepts every sample once it holds one anchor: |A| = 1 -> H = 0, A19); "
                         "default: the capacity")
    args = ap.parse_args()
    if args.warm is None:
        args.warm = args.capacity
    import paper_2510_12872_b200 as kv
    from paper_2510_12872_b200.online import ConsumerSlot, OnlinePool
    dev = "cuda"
    g = torch.Generator(device=dev).manual_seed(0)
    vocab = (torch.randn(V, DE, generator=g, device=dev) / math.sqrt(DE)).to(torch.bfloat16)
    r = lambda n: torch.randn(L, H, n, D, generator=g, device=dev).to(torch.bfloat16)
    inv = synth.llama3_inv_freq(D)
    pool = kv.AnchorPool(num_layers=L, num_kv_heads=H, head_dim=D, emb_dim=DE, capacity=args.capacity, max_anchor_len=T,
                         prefix_len=[P] * C, inv_freq=inv)
    p0 = [480 - 32 * c for c in range(C)]
    cons = [ConsumerSlot(p0[c], r(P), r(P), 480, torch.empty(L, H, p0[c] + T + P, D, dtype=torch.bfloat16, device=dev),
                         torch.empty(L, H, p0[c] + T + P, D, dtype=torch.bfloat16, device=dev)) for c in range(C)]
    online = OnlinePool(pool, cons, gamma=args.gamma)
    base_k, base_v = r(T), r(T)
    dense = [(r(T), r(T), r(P), r(P)) for _ in range(C)]
    spec = synth.StreamSpec(n_vocab=V, lengths=(T,), n_clusters=args.clusters, p_swap=args.p_swap)
    all_ids = synth.clustered_stream(spec, args.warm + args.requests, seed=1)  # one set of cluster centers
    stream_ids = all_ids[args.warm:]
    for ids in all_ids[:args.warm]:
        emb = vocab[ids.to(dev)].contiguous()
        offs = [kv.OffsetMeasure(c, ph_real=(dense[c][0], dense[c][1], p0[c]), ph_base=(base_k, base_v, 0),
                                 pf_real=(dense[c][2], dense[c][3], p0[c] + T), pf_base=(cons[c].pf_base_k,
                                 cons[c].pf_base_v, 480)) for c in range(C)]
        pool.insert(emb, offs)
    times = {"reuse": [], "fallback": []}
    entropies = []
    for ids in stream_ids:
        emb = vocab[ids.to(dev)].contiguous()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        res = online.step(emb, base_k, base_v, lambda c: dense[c])
        e1.record()
        torch.cuda.synchronize()
        times["reuse" if res.verdict == kv.SHAREABLE else "fallback"].append(e0.elapsed_time(e1))
        entropies.append((round(res.entropy, 3), res.reason, len(res.candidates)))
    med = lambda xs: sorted(xs)[len(xs) // 2] if xs else None
    reuse_ms = med(times["reuse"][2:] or times["reuse"])
    print(json.dumps({
        "step": "f1 online pool (Alg. 1)", "requests": args.requests, "reuse_rate": online.reuse_rate,
        "reuse_steps": len(times["reuse"]), "fallback_steps": len(times["fallback"]),
        "ms_reuse_step_median": reuse_ms, "ms_fallback_step_median": med(times["fallback"][1:] or times["fallback"]),
        "realigned_tokens_per_reuse_step": C * (T + P),
        "entropy_reason_ncand_first10": entropies[:10],
        "reuse_tokens_per_s": C * (T + P) / (reuse_ms / 1e3) if reuse_ms else None,
        "gamma": args.gamma, "capacity": args.capacity,
        "shape": f"8B shape, {T}-token samples, {C} consumers x {P}-token prefixes, capacity {args.capacity}, gamma {args.gamma}, "
                 f"{args.clusters} clusters, p_swap {args.p_swap}, {args.warm} warm anchors"}))
    pool.destroy()


if __name__ == "__main__":
    main()
