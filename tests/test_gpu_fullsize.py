"""Full-size parity (BASELINE.json configs[1]) in the launch configuration bench.py
times: the 8B-shape 5-agent request through ReuseRequest (5 matches, ONE batched
realign launch over all 30 segments, p_(m,0) copies + ledger), with the bench's
pipelined schedule (realign stream, runs back to back).

Matching outputs (all weights / verdicts of every pool) and every realigned or
copied K/V element of every agent are compared with the oracle (tests/state_oracle.py).  Oracle inputs are regenerated from their keyed seeds (synth.state), never read
back from the CUDA path.
"""
import time

import numpy as np
import pytest
import torch

import synth
from oracle import kvcomm_oracle as O
from tests import harness, state_oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", params=["bf16", "fp8"])
def state(request):
    """The request with bf16 pools (the bench) and with fp8-e4m3 pools (f3; the oracle
    then blends its own quantise/dequantise of the same offsets)."""
    assert torch.cuda.is_available()
    from synth.state import build_five_agent_state
    st = build_five_agent_state(seed=0, gamma=0.3, anchor_extra=16, offset_format=request.param)
    st.offset_format = request.param
    st.oracle_matches = {}
    # the bench's schedule: requests pipelined (each realign on its own stream, the next
    # request's matching beside it), three runs back to back without a host sync
    plan = st.request.plan
    rs = torch.cuda.Stream()
    plan.set_realign_stream(rs)
    for _ in range(3):
        st.request.launch([st.queries[n] for n in st.request.names])
    torch.cuda.current_stream().wait_stream(rs)
    res = st.request.results()
    plan.set_realign_stream(None)
    torch.cuda.synchronize()
    yield st, res
    for p in st.pools.values():
        p.destroy()
    torch.cuda.empty_cache()


def _oracle_match(st, name):
    if name not in st.oracle_matches:
        st.oracle_matches[name] = state_oracle.oracle_match(st, name)
    return st.oracle_matches[name]


@pytest.mark.parametrize("name", ["user_question", "agent_1_current", "agent_4_current"])
def test_fullsize_match_all_positions(state, name):
    st, res = state
    gm = res.matches[name]
    om = _oracle_match(st, name)
    assert gm.candidates == om.candidates == list(range(st.w.capacity))
    L_phi = st.w.pools[name].L_phi
    gW = harness.f64(gm.W)[:, :L_phi]
    assert np.all(np.abs(gW - om.W.T) <= 1e-5 * np.abs(om.W.T) + 1e-7)
    gwb = harness.f64(gm.wbar)
    assert np.all(np.abs(gwb - om.wbar) <= 1e-5 * om.wbar + 1e-7)
    assert abs(gm.entropy - om.H) <= 1e-6 * om.H + 1e-9
    if abs(om.H - om.threshold) > 1e-6 * om.threshold:
        assert gm.verdict == om.verdict
    assert gm.shareable   # the bench workload is all-reuse


def test_fullsize_every_element(state):
    """All 10,720 realigned tokens x 32 layers x 8 heads x 128 x (K, V) of the bench's
    launch, and every copied p_(m,0) row, against the oracle (host threads)."""
    st, res = state
    matches = {n: _oracle_match(st, n) for n in st.w.pools}
    t0 = time.perf_counter()
    counts = state_oracle.check_request(st, matches, res.reused_agents, fp8=st.offset_format == "fp8")
    counts["oracle_s"] = round(time.perf_counter() - t0, 1)
    state_oracle.report(f"fullsize_config2_{st.offset_format}", counts)
    assert counts["segments"] == 30
    assert counts["n"] == 10720 * 32 * 8 * 128 * 2


def test_fullsize_p0_copied_and_every_row_written(state):
    st, res = state
    for a in st.agents:
        p0 = st.w.agents[a.agent - 1].p0
        assert torch.equal(a.dst_k[:, :, :p0], st.inputs.p0(a.agent, 0))
        assert torch.equal(a.dst_v[:, :, :p0], st.inputs.p0(a.agent, 1))
        assert torch.isfinite(a.dst_k.float()).all() and torch.isfinite(a.dst_v.float()).all()
    assert res.realigned_tokens == st.w.realigned_tokens == 10720
    assert res.reused_agents == [1, 2, 3, 4, 5]
