"""Worker for tests/test_gpu_grid.py (launched by torch.distributed.run, not collected by
pytest): the layer x KV-head grid of SURVEY §8(e) (70B: "layer groups x KV-head
groups") on one GPU, every rank over gloo.

Rank r holds layers x heads block grid_shard(L, H, r, LG, HG) of every pool and base
cache and realigns it; the block is delivered to the consumer rank's full [L, H, N, d]
cache either by the realign kernel itself (fused: the destination is the IPC-mapped
full cache viewed at the block, with the full cache's layer stride: plan agent
dst_heads = H) or by the targeted gather (nccl mode: local [Ls, Hs, N, d] shard outputs,
grouped send/recv, staging + local permute into full[l0:l1, h0:h1]).  Every consumer
rank compares its agents' full caches bit for bit with an unsharded single-process run
of the same seeded inputs.

  argv: workload (five|segment) LG HG gather (fused|nccl) match (replicated|shard-match)
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch
import torch.distributed as dist


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    wl, LG, HG, gather, match = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], sys.argv[5]
    assert LG * HG == world
    torch.cuda.set_device(0)
    dist.init_process_group("gloo")
    import synth
    from synth.state import build_five_agent_state
    from paper_2510_12872_b200 import shard
    from paper_2510_12872_b200.request import AgentLayout, ReuseRequest

    if wl == "five":
        w = synth.five_agent_workload(L=4, H=4, d=128, D_e=64, user_len=96, resp_len=40, prefix_total=64,
                                      slot_prefix=8, capacity=4)
    else:   # configs[3]'s structure at a small shape: one segment, one consumer, many anchors
        w = synth.shared_segment_workload(L=4, H=4, d=128, D_e=64, seg_len=150, prefix_len=8, p0=24, capacity=12)
    ref = build_five_agent_state(w, seed=4, device=0, gamma=1.0)
    ref_req = ReuseRequest(ref.pools, ref.agents, gamma=1.0)
    ref_req.plan.run([ref.queries[n] for n in ref_req.names], sync=True)
    ref_ms, reused = ref_req.plan.results()
    assert all(reused), reused

    lr, hr = shard.grid_shard(w.L, w.H, rank, LG, HG)
    st = build_five_agent_state(w, seed=4, device=0, gamma=1.0, layer_range=lr, head_range=hr)
    assert all(a.dst_k.shape[:2] == (lr[1] - lr[0], hr[1] - hr[0]) for a in st.agents)
    peer = None
    if gather == "fused":
        peer = shard.PeerCaches([(a.agent, a.N) for a in st.agents], w.L, w.H, w.d, rank, world, 0)
        agents = [AgentLayout(a.agent, a.N, a.p0_k, a.p0_v, a.segments, *peer.destinations(i, lr, hr))
                  for i, a in enumerate(st.agents)]
        req = ReuseRequest(st.pools, agents, gamma=1.0)
        full = [peer.full(i) for i in range(len(st.agents))]
    else:
        req = st.request
        full = [(torch.zeros(w.L, w.H, a.N, w.d, dtype=torch.bfloat16, device="cuda"),
                 torch.zeros(w.L, w.H, a.N, w.d, dtype=torch.bfloat16, device="cuda"))
                if shard.consumer_rank(a.agent, world) == rank else (None, None) for a in st.agents]
    if match == "shard-match":
        req.shard_matching(rank, world, 0)
    qs = [st.queries[n] for n in req.names]
    for _ in range(2):
        if match == "shard-match":
            req._mshard.run(qs, sync=True)
        else:
            req.plan.run(qs, sync=True)
        if peer is not None:
            peer.sync()
        else:
            shard.gather_to_consumers([a.agent for a in st.agents], [(a.dst_k, a.dst_v) for a in st.agents], full,
                                      w.L, rank, world, head_groups=HG)
    ms, reused = req.plan.results()
    assert all(reused), reused
    for a, b in zip(ms, ref_ms):   # weights bit-identical to the unsharded run
        assert a.candidates == b.candidates and a.verdict == b.verdict and a.entropy == b.entropy
        assert torch.equal(a.W, b.W) and torch.equal(a.wbar, b.wbar), f"rank {rank}: weights differ"
    checked = 0
    for i, a in enumerate(ref.agents):
        fk, fv = full[i]
        if fk is None:
            continue
        assert torch.equal(fk, a.dst_k), f"rank {rank} agent {a.agent} K differs"
        assert torch.equal(fv, a.dst_v), f"rank {rank} agent {a.agent} V differs"
        checked += 1
    dist.barrier()
    if match == "shard-match":
        req._mshard.close()
    if peer is not None:
        peer.close()
    print(f"rank {rank}: {checked} agents bit-exact", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
