"""Worker for tests/test_gpu_peer.py (launched by torch.distributed.run, not collected by
pytest): the fused gather on one GPU with 2 ranks over gloo.

Each rank realigns its layer block of a small 5-agent workload straight into the
consumer rank's IPC-shared full-depth caches (shard.PeerCaches); every consumer rank
then checks its agents' caches bit for bit against an unsharded single-process run of
the same seeded inputs.  On one GPU the IPC mapping is same-device memory, so this
exercises the handle exchange, the layer offsets and the ordering, not NVLink."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch
import torch.distributed as dist


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    fmt = sys.argv[1] if len(sys.argv) > 1 else "bf16"
    shard_match = len(sys.argv) > 2 and sys.argv[2] in ("shard-match", "shard-mismatch", "shard-match-emb",
                                                          "shard-mismatch-empty", "shard-mismatch-replace")
    empty_rank1 = len(sys.argv) > 2 and sys.argv[2] == "shard-mismatch-empty"
    emb_shard = len(sys.argv) > 2 and sys.argv[2] == "shard-match-emb"
    replace_rank1 = len(sys.argv) > 2 and sys.argv[2] == "shard-mismatch-replace"
    mismatch = len(sys.argv) > 2 and sys.argv[2] in ("shard-mismatch", "shard-mismatch-empty",
                                                      "shard-mismatch-replace")
    top_k = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    sim = sys.argv[4] if len(sys.argv) > 4 else "l2"
    scal = sys.argv[5] if len(sys.argv) > 5 else "frobenius"
    # "pipe": the bench's N > 1 schedule — every realign on a second stream
    # (kvcomm_plan_set_realign_stream), runs issued back to back, one delivery sync at the end
    pipe = len(sys.argv) > 6 and sys.argv[6] == "pipe"
    pk = dict(offset_format=fmt, similarity=sim, scalar_distance=scal)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo")
    import synth
    from synth.state import build_five_agent_state
    from paper_2510_12872_b200 import shard
    from paper_2510_12872_b200.request import AgentLayout, ReuseRequest

    w = synth.five_agent_workload(L=5, H=2, d=64, D_e=64, user_len=96, resp_len=40, prefix_total=64,
                                  slot_prefix=8, capacity=4)
    ref = build_five_agent_state(w, seed=3, device=0, gamma=1.0, **pk)
    ref_req = ReuseRequest(ref.pools, ref.agents, gamma=1.0, top_k=top_k)
    ref_req.plan.run([ref.queries[n] for n in ref_req.names], sync=True)
    ref_ms, reused = ref_req.plan.results()
    assert all(reused), reused

    lr = shard.layer_shard(w.L, rank, world)
    st = build_five_agent_state(w, seed=3, device=0, gamma=1.0, layer_range=lr,
                                emb_shard=(rank, world) if emb_shard else None, **pk)
    peer = shard.PeerCaches([(a.agent, a.N) for a in st.agents], w.L, w.H, w.d, rank, world, 0)
    agents = [AgentLayout(a.agent, a.N, a.p0_k, a.p0_v, a.segments, *peer.destinations(i, lr))
              for i, a in enumerate(st.agents)]
    req = ReuseRequest(st.pools, agents, gamma=1.0, top_k=top_k)
    if mismatch:   # the ranks' pools out of step: rank 1 lacks one user_question anchor
        if rank == 1 and replace_rank1:
            # the full pool takes one more anchor: LFU evicts slot 0 and the newcomer reuses
            # that slot id, so both ranks still list candidates 0..3 — but slot 0 now holds a
            # different anchor (same length) on rank 1
            from paper_2510_12872_b200 import kvcomm as K
            inp, name = st.inputs, "user_question"
            emb = inp.vocab()[inp.anchor_ids(name, 1)]
            offs = [K.OffsetGiven(c, inp.offset(name, 1, c, "ph", 0), inp.offset(name, 1, c, "ph", 1),
                                  inp.offset(name, 1, c, "pf", 0), inp.offset(name, 1, c, "pf", 1))
                    for c in range(len(w.pools[name].consumers))]
            slot, ev = st.pools[name].insert(emb, offs)
            assert (slot, ev) == (0, 0), (slot, ev)
        elif rank == 1 and not empty_rank1:
            st.pools["user_question"].evict(0)
        if rank == 1 and empty_rank1:   # every pool empty: rank 1 decides everything on the host
            for pool in st.pools.values():
                for slot in range(pool.capacity):
                    if pool.slot_info(slot)["occupied"]:
                        pool.evict(slot)
        req.shard_matching(rank, world, 0)
        for _ in range(2):
            req._mshard.run([st.queries[n] for n in req.names], sync=True)
            peer.sync()
        from paper_2510_12872_b200._lib import KVCommError
        if empty_rank1 and rank == 1:   # no job here: host verdicts, all agents fall back
            ms, reused = req.plan.results()
            assert not any(reused) and all(m.reason == "EMPTY_POOL" for m in ms), [m.reason for m in ms]
        else:
            try:
                req.plan.results()
                raise AssertionError("out-of-step pools were not detected")
            except KVCommError as e:
                assert e.status_name == "SHAPE_MISMATCH" and "sharded matching" in str(e), e
        checked = 0
        for i, a in enumerate(ref.agents):   # no agent was realigned: the caches stay zero
            fk, fv = peer.full(i)
            if fk is None:
                continue
            assert not fk.any() and not fv.any(), f"rank {rank}: agent {a.agent} written"
            checked += 1
        dist.barrier()
        req._mshard.close()
        peer.close()
        print(f"rank {rank}: {checked} agents untouched, mismatch reported", flush=True)
        dist.destroy_process_group()
        return
    if shard_match:  # each rank computes half the match positions, stored into both ranks' buffers
        req.shard_matching(rank, world, 0)
    rs = torch.cuda.Stream() if pipe else None
    if pipe:
        req.plan.set_realign_stream(rs)
    for _ in range(3):  # the later runs overwrite the same rows (and alternate the match buffers)
        if shard_match:
            req._mshard.run([st.queries[n] for n in req.names], sync=not pipe)
        else:
            req.plan.run([st.queries[n] for n in req.names], sync=not pipe)
        if not pipe:
            peer.sync()
    if pipe:
        torch.cuda.current_stream().wait_stream(rs)
        peer.sync()
    ms, reused = req.plan.results()
    if pipe:
        req.plan.set_realign_stream(None)
    assert all(reused), reused
    for a, b in zip(ms, ref_ms):   # weights and verdicts bit-identical to the unsharded run
        assert a.candidates == b.candidates and a.verdict == b.verdict
        assert a.entropy == b.entropy and a.threshold == b.threshold, (a.entropy, b.entropy)
        assert torch.equal(a.W, b.W) and torch.equal(a.wbar, b.wbar), f"rank {rank}: weights differ"
    checked = 0
    for i, a in enumerate(ref.agents):
        fk, fv = peer.full(i)
        if fk is None:
            continue
        assert torch.equal(fk, a.dst_k), f"rank {rank} agent {a.agent} K differs"
        assert torch.equal(fv, a.dst_v), f"rank {rank} agent {a.agent} V differs"
        checked += 1
    dist.barrier()
    if shard_match:
        req._mshard.close()
    peer.close()
    print(f"rank {rank}: {checked} agents bit-exact", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
