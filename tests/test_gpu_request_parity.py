"""The bench's launch configuration at small sizes, compared with the oracle on every
element (-m gpu).

ReuseRequest.plan is what bench.py times: one batched match over every pool and ONE
gated realign launch in which the consumers of one sample form a shared-base group
(user_question for 5 agents, agent_j_current for 5 - j), with the p_(m,0) COPY
segments in the same launch.  Here the same plan runs on small 5-agent states — d = 128
(the kernel instantiation the bench uses) and d = 64 (the generic one), bf16 and fp8
pools, dense and top-k weights — and every realigned / copied element of every reused
agent is checked against the oracle (tests/state_oracle.py).  The gated case makes one
pool NewAnchor (Algorithm 1's branch): its consumers must be left untouched and
every other agent must still match the oracle element by element.
"""
import numpy as np
import pytest
import torch

import synth
from oracle import kvcomm_oracle as O
from tests import harness, state_oracle

pytestmark = pytest.mark.gpu


def _state(d, fmt, top_k=0, seed=0):
    from synth.state import build_five_agent_state
    w = synth.five_agent_workload(L=2, H=2, d=d, D_e=128, user_len=80, resp_len=40, prefix_total=96,
                                  slot_prefix=8, capacity=5)
    return build_five_agent_state(w, seed=seed, gamma=0.9, anchor_extra=8, offset_format=fmt, top_k=top_k)


def _check_match(gm, om):
    assert gm.candidates == om.candidates
    gW = harness.f64(gm.W)[om.candidates][:, : om.W.shape[0]].T
    assert np.all(np.abs(gW - om.W) <= 1e-5 * np.abs(om.W) + 1e-7)
    assert abs(gm.entropy - om.H) <= 1e-6 * abs(om.H) + 1e-9
    if abs(om.H - om.threshold) > harness.TIE_REL * om.threshold:
        assert gm.verdict == om.verdict


@pytest.mark.parametrize("d,fmt,top_k", [(128, "bf16", 0), (128, "fp8", 0), (64, "bf16", 0), (128, "bf16", 3)])
def test_request_every_element(d, fmt, top_k):
    st = _state(d, fmt, top_k, seed=d + top_k)
    for a in st.agents:
        a.dst_k.fill_(float("nan"))
        a.dst_v.fill_(float("nan"))
    res = st.request.run(st.queries)
    torch.cuda.synchronize()
    assert res.reused_agents == [1, 2, 3, 4, 5]
    matches = {}
    for n in st.w.pools:
        om = state_oracle.oracle_match(st, n, top_k=top_k)
        if om.idx is not None:
            assert not harness.distance_tie_positions(om.dist, om.candidates, top_k).any()
        _check_match(res.matches[n], om)
        matches[n] = om
    counts = state_oracle.check_request(st, matches, res.reused_agents, fp8=fmt == "fp8")
    state_oracle.report(f"request_d{d}_{fmt}_k{top_k}", counts)
    assert counts["segments"] == 30
    assert counts["n"] == st.w.realigned_tokens * st.w.L * st.w.H * d * 2


@pytest.mark.parametrize("fmt", ["bf16", "fp8"])
def test_request_gated_every_element(fmt):
    st = _state(128, fmt, seed=7)
    g = torch.Generator(device="cuda").manual_seed(11)
    q = dict(st.queries)
    # agent_2_current's sample is far from every anchor -> high entropy -> NewAnchor (an input, drawn here)
    q["agent_2_current"] = (torch.randn(q["agent_2_current"].shape, generator=g, device="cuda") * 0.125
                            ).to(torch.bfloat16)
    for a in st.agents:
        a.dst_k.fill_(5.0)
        a.dst_v.fill_(5.0)
    res = st.request.run(q)
    torch.cuda.synchronize()
    matches = {n: state_oracle.oracle_match(st, n, query=q[n]) for n in st.w.pools}
    assert matches["agent_2_current"].verdict == O.NEW_ANCHOR
    for n in st.w.pools:
        _check_match(res.matches[n], matches[n])
    assert res.fallback_agents == [3, 4, 5] and res.reused_agents == [1, 2]
    for a in st.agents[2:]:                       # consumers of the NewAnchor pool: untouched
        assert torch.all(a.dst_k == 5.0) and torch.all(a.dst_v == 5.0)
    counts = state_oracle.check_request(st, matches, res.reused_agents, fp8=fmt == "fp8")
    state_oracle.report(f"request_gated_{fmt}", counts)
    assert counts["segments"] == 2 + 4            # agent 1: 1 placeholder + 1 prefix; agent 2: 2 + 2
