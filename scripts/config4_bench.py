#!/usr/bin/env python
"""BASELINE.json configs[3] on one B200: one 1/8 shard of the Llama-3-70B-shape request
(layers [0,20) x KV heads [0,4) of 80 x 8; a 3072-token shared segment + 32-token
prefix + 200-token p_(m,0) copy; 256-anchor pool, k = 256) through the plan, the same
launch configuration tests/test_gpu_config4.py checks against the oracle.

Prints one JSON line: per-request-shard device time (CUDA events, median of batches),
the realign kernel alone, its algorithmic bytes and GB/s.  The 8-GPU aggregate is not
measured here (one GPU per gpurun call): each of the 8 shards does the same work with
no communication before the delivery of the realigned blocks.

  python scripts/config4_bench.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import synth
from synth.state import keyed_gen

L, H, D, DE = 80, 8, 128, 8192
LAYERS, HEADS = (0, 20), (0, 4)
T, P, M, P0, N_VOCAB = 3072, 32, int(os.environ.get("C4_ANCHORS", "256")), 200, 128256
SEED = 70


def main():
    import paper_2510_12872_b200 as kv
    Ls, Hs = LAYERS[1] - LAYERS[0], HEADS[1] - HEADS[0]
    g = keyed_gen(SEED, "c4vocab")
    vocab = (torch.randn(N_VOCAB, DE, generator=g, device="cuda") / np.sqrt(DE)).to(torch.bfloat16)
    pool = kv.AnchorPool(num_layers=L, num_kv_heads=H, head_dim=D, emb_dim=DE, capacity=M, max_anchor_len=T,
                         prefix_len=[P], inv_freq=synth.llama3_inv_freq(D), layer_range=LAYERS, head_range=HEADS)
    go = keyed_gen(SEED, "c4off-bench")
    rnd = lambda n: (torch.randn(Ls, Hs, n, D, generator=go, device="cuda") * synth.OFFSET_STD).to(torch.bfloat16)
    ids0 = None
    for s in range(M):
        ids = torch.randint(0, N_VOCAB, (T,), generator=keyed_gen(SEED, "c4ids", s), device="cuda")
        ids0 = ids if s == 0 else ids0
        pool.insert(vocab[ids], [kv.OffsetGiven(0, rnd(T), rnd(T), rnd(P), rnd(P))])
    gq = keyed_gen(SEED, "c4query")
    swap = torch.rand(T, generator=gq, device="cuda") < 0.3
    query = vocab[torch.where(swap, torch.randint(0, N_VOCAB, (T,), generator=gq, device="cuda"), ids0)].contiguous()
    del vocab
    gb = keyed_gen(SEED, "c4base")
    base = [torch.randn(Ls, Hs, T, D, generator=gb, device="cuda").to(torch.bfloat16) for _ in range(2)]
    pfb = [torch.randn(Ls, Hs, P, D, generator=gb, device="cuda").to(torch.bfloat16) for _ in range(2)]
    p0 = [torch.randn(Ls, Hs, P0, D, generator=gb, device="cuda").to(torch.bfloat16) for _ in range(2)]
    N = P0 + T + P
    dst = [torch.empty(Ls, Hs, N, D, dtype=torch.bfloat16, device="cuda") for _ in range(2)]
    segs = [kv.PlanSegment(0, 0, kv.PLACEHOLDER, 0, base[0], base[1], 0, P0),
            kv.PlanSegment(0, 0, kv.PREFIX, 0, pfb[0], pfb[1], P0, P0 + T),
            kv.PlanSegment(0, 0, kv.COPY, 0, p0[0], p0[1], 0, 0)]
    plan = kv.Plan([(pool, T, 0.3, 0)], segs, [(N, dst[0], dst[1])])
    stream = torch.cuda.current_stream()
    for _ in range(5):
        plan.run([query], stream=stream)
    torch.cuda.synchronize()
    _, reused = plan.results()
    if not all(reused):
        raise SystemExit("request fell back: the timing needs the reuse branch")
    ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    plan.set_events(*ev)
    steps, realign = [], []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ks = []
        e0.record(stream)
        for _ in range(4):
            plan.run([query], stream=stream)
            ev[1].synchronize()
            ks.append(ev[0].elapsed_time(ev[1]))
        e1.record(stream)
        torch.cuda.synchronize()
        steps.append(e0.elapsed_time(e1) / 4)
        realign.extend(ks)
    step_ms = sorted(steps)[len(steps) // 2]
    plan.set_events(None, None)

    # Requests pipelined (the bench's schedule, kvcomm_plan_set_realign_stream): the next
    # request's matching (replicated here: all 3,072 positions x 256 anchors, 12.9 GB) runs
    # beside this request's realign; both streams share HBM
    rs = torch.cuda.Stream()
    plan.set_realign_stream(rs)
    for _ in range(3):
        plan.run([query], stream=stream)
    stream.wait_stream(rs)
    torch.cuda.synchronize()
    piped = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(8):
            plan.run([query], stream=stream)
        stream.wait_stream(rs)
        e1.record(stream)
        torch.cuda.synchronize()
        piped.append(e0.elapsed_time(e1) / 8)
    plan.set_realign_stream(None)
    _, reused = plan.results()
    if not all(reused):
        raise SystemExit("pipelined request fell back")
    step_ms_piped = sorted(piped)[len(piped) // 2]

    # Sharded matching: with G ranks each computes T/G positions of the match.
    # One rank's share is timed here as a match-only plan over the first T/G positions of
    # the same query and pool (one 1-token COPY segment keeps the plan well-formed), with
    # the device kept busy while the host prepares the run so that the events see device
    # time only.  The peer stores of the W columns and partials (7/G of ~M*T*12 B) and the
    # cross-rank barrier are not in this number (no second GPU here).
    match_ms = {}
    one = [torch.zeros(Ls, Hs, 1, D, dtype=torch.bfloat16, device="cuda") for _ in range(2)]
    tiny = [torch.empty(Ls, Hs, 1, D, dtype=torch.bfloat16, device="cuda") for _ in range(2)]
    for G in (1, 2, 4, 8):
        Tg = T // G
        mp = kv.Plan([(pool, Tg, 0.3, 0)], [kv.PlanSegment(0, 0, kv.COPY, 0, one[0], one[1], 0, 0)],
                     [(1, tiny[0], tiny[1])])
        qg = query[:Tg].contiguous()
        for _ in range(3):
            mp.run([qg], stream=stream)
        ts = []
        for _ in range(7):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda._sleep(2_000_000)       # ~1 ms of device work hides the host-side preparation
            e0.record(stream)
            mp.run([qg], stream=stream)
            e1.record(stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        match_ms[G] = sorted(ts)[len(ts) // 2]
        mp.destroy()
    # embedding memory per GPU: every row (replicated) vs emb_shard=(0, 8) (sharded matching)
    emb_bytes = {}
    for name, es in (("replicated", None), ("sharded_G8", (0, 8))):
        q = kv.AnchorPool(num_layers=L, num_kv_heads=H, head_dim=D, emb_dim=DE, capacity=M, max_anchor_len=T,
                          prefix_len=[P], inv_freq=synth.llama3_inv_freq(D), layer_range=(0, 1), head_range=(0, 1),
                          emb_shard=es)
        emb_bytes[name] = q.nbytes()
        q.destroy()
    emb_note = ("pool bytes of a 1-layer x 1-head pool of the same capacity/length (offsets identical, so the "
                "difference is the embedding slab: 256 anchors x 3072 rows x 8192 x 2 B, or 1/8 of the rows)")
    rl_ms = sorted(realign)[len(realign) // 2]
    tok = Ls * Hs * D * 2 * 2  # one token row, K+V, this shard
    alg = ((M + 2) * T + (M + 2) * P + 2 * P0) * tok
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs") \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else None
    print(json.dumps({
        "workload": "BASELINE configs[3] shard: llama3-70b-shape layers [0,20) x kv heads [0,4), 3072-token "
                    "segment + 32-token prefix + 200-token p0, 256-anchor pool, k=256",
        "realigned_tokens": T + P, "step_ms": step_ms, "realign_ms": rl_ms,
        "step_ms_pipelined": step_ms_piped,
        "pipelined_note": "requests back to back, realign on its own stream, the next request's replicated "
                          "match beside it (40-register match build)",
        "shard_tokens_per_s": (T + P) / (step_ms / 1e3),
        "realign_alg_bytes": alg, "realign_GBps": alg / (rl_ms / 1e3) / 1e9,
        "frac_of_measured_peak": (alg / (rl_ms / 1e3) / 1e9 / peak) if peak else None,
        "match_only_ms_by_G": match_ms,
        "match_note": "match-only plan over T/G positions (+1-token copy): one rank's share of sharded "
                      "matching, without its NVLink stores and the barrier",
        "step_ms_sharded_match_G8_est": step_ms - match_ms[1] + match_ms[8],
        "pool_bytes_small_shard": emb_bytes, "pool_bytes_note": emb_note,
        "note": "one of 8 shards measured on one B200; the 8-GPU run is not measured here"}))
    plan.destroy()
    pool.destroy()


if __name__ == "__main__":
    main()
