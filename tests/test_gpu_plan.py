"""Native request plan (kvcomm_plan_*) vs the unfused C-ABI calls, and the
device-side Shareable/NewAnchor branch of Algorithm 1 (-m gpu)."""
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu


def _small_state(seed=0, gamma=0.3):
    from synth.state import build_five_agent_state
    w = synth.five_agent_workload(L=3, H=2, d=64, D_e=64, user_len=96, resp_len=40, prefix_total=48,
                                  slot_prefix=4, capacity=4)
    return build_five_agent_state(w, seed=seed, gamma=gamma, anchor_extra=8)


def _snap(st):
    return [(a.dst_k.clone(), a.dst_v.clone()) for a in st.agents]


def test_plan_equals_unfused_bitwise_and_reports_all_reused():
    st = _small_state()
    for a in st.agents:
        a.dst_k.fill_(7.0)
        a.dst_v.fill_(7.0)
    res_u = st.request.run_unfused(st.queries)
    torch.cuda.synchronize()
    ref = _snap(st)
    for a in st.agents:
        a.dst_k.fill_(-3.0)
        a.dst_v.fill_(-3.0)
    res_p = st.request.run(st.queries)           # plan, sync
    assert res_p.reused_agents == res_u.reused_agents == [1, 2, 3, 4, 5]
    assert res_p.realigned_tokens == res_u.realigned_tokens
    for (k, v), a in zip(ref, st.agents):
        assert torch.equal(k, a.dst_k) and torch.equal(v, a.dst_v)
    for n in st.request.names:
        mu, mp = res_u.matches[n], res_p.matches[n]
        assert mu.candidates == mp.candidates and mu.verdict == mp.verdict and mu.entropy == mp.entropy
        assert torch.equal(mu.W, mp.W[:, : mu.W.shape[1]]) and torch.equal(mu.wbar, mp.wbar)


def test_plan_pipelined_runs_match_single_run():
    st = _small_state(seed=3)
    st.request.run(st.queries)
    ref = _snap(st)
    for _ in range(5):                            # several runs in flight, no host sync in between
        st.request.run(st.queries, sync=False)
    res = st.request.results()
    assert res.reused_agents == [1, 2, 3, 4, 5]
    for (k, v), a in zip(ref, st.agents):
        assert torch.equal(k, a.dst_k) and torch.equal(v, a.dst_v)


def test_realign_stream_pipelining_matches_sequential_runs():
    """kvcomm_plan_set_realign_stream (the bench's N = 1 schedule): runs alternate between
    two query sets — B sends agent_2_current's pool NewAnchor, so its agents keep A's rows —
    with every realign on a second stream and no host sync; the caches and verdicts must be
    those of the same runs issued one at a time."""
    st = _small_state(seed=7)
    g = torch.Generator(device="cuda").manual_seed(2)
    qa = dict(st.queries)
    qb = dict(st.queries)
    qb["agent_2_current"] = (torch.randn(qb["agent_2_current"].shape, generator=g, device="cuda") * 0.125
                             ).to(torch.bfloat16)
    for a in st.agents:
        a.dst_k.fill_(1.0)
        a.dst_v.fill_(1.0)
    st.request.run(qa)
    st.request.run(qb)
    ref = _snap(st)
    res_ref = st.request.results()
    for a in st.agents:
        a.dst_k.fill_(1.0)
        a.dst_v.fill_(1.0)
    torch.cuda.synchronize()
    plan = st.request.plan
    rs = torch.cuda.Stream()
    plan.set_realign_stream(rs)
    try:
        for _ in range(3):
            st.request.launch([qa[n] for n in st.request.names])
            st.request.launch([qb[n] for n in st.request.names])
        torch.cuda.current_stream().wait_stream(rs)
        res = st.request.results()
    finally:
        plan.set_realign_stream(None)
    torch.cuda.synchronize()
    assert res.fallback_agents == res_ref.fallback_agents == [3, 4, 5]
    for n in st.request.names:
        assert res.matches[n].verdict == res_ref.matches[n].verdict
        assert res.matches[n].entropy == res_ref.matches[n].entropy
    for (k, v), a in zip(ref, st.agents):
        assert torch.equal(k, a.dst_k) and torch.equal(v, a.dst_v)


def test_device_side_branch_skips_agents_of_a_new_anchor_pool():
    st = _small_state(seed=5)
    g = torch.Generator(device="cuda").manual_seed(1)
    q = dict(st.queries)
    # agent_2_current's sample is far from every anchor -> high entropy -> NewAnchor
    q["agent_2_current"] = (torch.randn(q["agent_2_current"].shape, generator=g, device="cuda") * 0.125
                            ).to(torch.bfloat16)
    for a in st.agents:
        a.dst_k.fill_(5.0)
        a.dst_v.fill_(5.0)
    res_u = st.request.run_unfused(q)
    torch.cuda.synchronize()
    ref = _snap(st)
    for a in st.agents:
        a.dst_k.fill_(5.0)
        a.dst_v.fill_(5.0)
    res_p = st.request.run(q)
    assert res_u.matches["agent_2_current"].verdict == 1 and res_u.matches["agent_2_current"].reason == "HIGH_ENTROPY"
    assert res_p.fallback_agents == res_u.fallback_agents == [3, 4, 5]   # agents that consume agent_2_current
    assert res_p.reused_agents == [1, 2]
    for (k, v), a in zip(ref, st.agents):
        assert torch.equal(k, a.dst_k) and torch.equal(v, a.dst_v)
    for a in st.agents[2:]:
        assert torch.all(a.dst_k == 5.0)          # fallback agents untouched


def test_two_plans_sharing_pools_run_concurrently_on_two_streams():
    """Plans own their match scratch: two requests over the same pools, in flight on
    two streams at once (different queries: one has a NewAnchor pool), each give
    the result of running alone."""
    from paper_2510_12872_b200.request import AgentLayout, ReuseRequest
    st = _small_state(seed=7)
    g = torch.Generator(device="cuda").manual_seed(2)
    q2 = dict(st.queries)
    q2["agent_1_current"] = (torch.randn(q2["agent_1_current"].shape, generator=g, device="cuda") * 0.125
                             ).to(torch.bfloat16)
    agents2 = [AgentLayout(a.agent, a.N, a.p0_k, a.p0_v, a.segments, torch.full_like(a.dst_k, 9.0),
                           torch.full_like(a.dst_v, 9.0)) for a in st.agents]
    req2 = ReuseRequest(st.pools, agents2, gamma=st.request.gamma, top_k=st.request.top_k)
    # references: each alone
    st.request.run(st.queries)
    ref1 = _snap(st)
    req2.run(q2)
    ref2 = [(a.dst_k.clone(), a.dst_v.clone()) for a in agents2]
    for a in list(st.agents) + agents2:
        a.dst_k.fill_(1.0)
        a.dst_v.fill_(1.0)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(4):
        st.request.run(st.queries, sync=False, stream=s1)
        req2.run(q2, sync=False, stream=s2)
    torch.cuda.synchronize()
    assert st.request.results().reused_agents == [1, 2, 3, 4, 5]
    assert req2.results().fallback_agents == [2, 3, 4, 5]
    for (k, v), a in zip(ref1, st.agents):
        assert torch.equal(k, a.dst_k) and torch.equal(v, a.dst_v)
    for (k, v), a in zip(ref2, agents2):
        if a.agent == 1:
            assert torch.equal(k, a.dst_k) and torch.equal(v, a.dst_v)


def test_split_run_and_shard_argument_contracts():
    """kvcomm_plan_run_begin/run_end pair up (begin twice, end without begin:
    INVALID_ARGUMENT), begin+end equals run bit for bit, and kvcomm_plan_match_shard
    validates rank/world before touching any peer."""
    from paper_2510_12872_b200 import kvcomm as K
    st = _small_state(seed=2, gamma=1.0)
    plan, q = st.request.plan, [st.queries[n] for n in st.request.names]
    plan.run(q, sync=True)
    torch.cuda.synchronize()
    ref = _snap(st)
    for a in st.agents:
        a.dst_k.fill_(0.5)
        a.dst_v.fill_(0.5)
    with pytest.raises(K.KVCommError, match="not begun"):
        plan.run_end()
    plan.run_begin(q)
    with pytest.raises(K.KVCommError, match="already begun"):
        plan.run_begin(q)
    plan.run_end(sync=True)
    for (k, v), a in zip(ref, st.agents):
        assert torch.equal(k, a.dst_k) and torch.equal(v, a.dst_v)
    for rank, world in ((0, 9), (2, 2), (-1, 2)):
        with pytest.raises(K.KVCommError, match="INVALID_ARGUMENT"):
            plan.match_shard(rank, world, [b"\0" * 64] * max(world, 1) if world > 0 else [])
    with pytest.raises(ValueError):
        plan.match_shard(0, 2, [b"\0" * 64])     # one handle per rank
    plan.match_shard(0, 1)                         # back to unsharded: runs still work
    plan.run(q, sync=True)

def test_every_pool_new_anchor_launches_nothing_into_the_caches():
    """All five samples far from their pools: every verdict NewAnchor, every segment's
    gate closed in the prep kernel's unit list (segment -1), so the one realign launch
    writes nothing — the caches keep their contents, single-stream and pipelined."""
    st = _small_state(seed=9)
    g = torch.Generator(device="cuda").manual_seed(4)
    q = {n: (torch.randn(x.shape, generator=g, device="cuda") * 0.125).to(torch.bfloat16)
         for n, x in st.queries.items()}
    for pipelined in (False, True):
        for a in st.agents:
            a.dst_k.fill_(3.0)
            a.dst_v.fill_(3.0)
        rs = torch.cuda.Stream() if pipelined else None
        if rs is not None:
            st.request.plan.set_realign_stream(rs)
        try:
            for _ in range(2):
                st.request.launch([q[n] for n in st.request.names])
            if rs is not None:
                torch.cuda.current_stream().wait_stream(rs)
            res = st.request.results()
        finally:
            st.request.plan.set_realign_stream(None)
        torch.cuda.synchronize()
        assert res.reused_agents == [] and res.fallback_agents == [1, 2, 3, 4, 5]
        assert all(not m.shareable for m in res.matches.values())
        for a in st.agents:
            assert torch.all(a.dst_k == 3.0) and torch.all(a.dst_v == 3.0)
